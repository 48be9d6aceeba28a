# Re-entry check: GPU tests + cfg2 / cfg3 bench on the restored tree.
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r51_tests.log 2>&1; tail -3 gpurun_out/r51_tests.log
timeout 600 python bench.py > gpurun_out/r51_cfg2.json 2> gpurun_out/r51_cfg2.err; python tools/bench_summary.py cfg2 gpurun_out/r51_cfg2.json
timeout 600 python bench.py --config cfg3 > gpurun_out/r51_cfg3.json 2> gpurun_out/r51_cfg3.err; python tools/bench_summary.py cfg3 gpurun_out/r51_cfg3.json
