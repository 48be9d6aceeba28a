# paired cascade partition: GPU cascade tests, cfg3 auto / paired off, cfg4 / cfg2d (K2 chunk mode unchanged?), trace.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_cascade.py -q -x 2>&1 | tail -3
timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-e2e > gpurun_out/r61_auto.json 2>gpurun_out/r61_auto.err; python tools/bench_summary.py "cfg3 auto" gpurun_out/r61_auto.json; tail -1 gpurun_out/r61_auto.err
timeout 300 python bench.py --config cfg3 --prefix-splits 2 --no-cpu-baseline --no-e2e > gpurun_out/r61_s2.json 2>/dev/null; python tools/bench_summary.py "cfg3 S2" gpurun_out/r61_s2.json
timeout 300 python bench.py --config cfg2d --no-cpu-baseline --no-e2e > gpurun_out/r61_cfg2d.json 2>/dev/null; python tools/bench_summary.py "cfg2d" gpurun_out/r61_cfg2d.json
timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/r61_cfg4.json 2>/dev/null; python tools/bench_summary.py "cfg4" gpurun_out/r61_cfg4.json
echo "== auto"; KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/cascade_trace.py 2>&1 | tail -9
