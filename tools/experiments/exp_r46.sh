cd $GRAFT_REPO_ROOT
echo "== switch every step, no sync"; STEPS=300 SYNC=0 SWITCH=1 timeout 300 python tools/repro_cfg3.py 2>&1 | tail -1
echo "== switch every 7, no sync"; STEPS=300 SYNC=0 SWITCH=7 timeout 300 python tools/repro_cfg3.py 2>&1 | tail -1
timeout 300 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/r46_cfg3.json 2> gpurun_out/r46_cfg3.err; echo rc=$?; python tools/bench_summary.py cfg3 gpurun_out/r46_cfg3.json
timeout 600 python -m pytest tests/test_gpu_cascade.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
