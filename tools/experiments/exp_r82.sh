# prefix kernel: records in the kernel parameters, setup before the wait for the prologue.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_cascade.py tests/test_gpu_scores.py -q -x 2>&1 | tail -2
for i in 1 2 3; do timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-e2e > gpurun_out/r82_$i.json 2>/dev/null; python tools/bench_summary.py "cfg3 #$i" gpurun_out/r82_$i.json; done
timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/r82_cfg4.json 2>/dev/null; python tools/bench_summary.py "cfg4" gpurun_out/r82_cfg4.json
