# Re-entry check of HEAD on one B200: GPU tests, smoke, default bench, cfg3/cfg5hh lines.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2j_gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2j_tests.log 2>&1; tail -3 gpurun_out/r2j_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2j_smoke.log 2>&1; tail -1 gpurun_out/r2j_smoke.log
timeout 300 python bench.py > gpurun_out/r2j_cfg2.json 2> gpurun_out/r2j_cfg2.err; tail -c 600 gpurun_out/r2j_cfg2.json
timeout 300 python bench.py --config cfg3 > gpurun_out/r2j_cfg3.json 2> gpurun_out/r2j_cfg3.err
timeout 300 python bench.py --config cfg4 > gpurun_out/r2j_cfg4.json 2> gpurun_out/r2j_cfg4.err
