# MULTI instantiation for the paired cascade; single-unit prefix kernels as before.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_cascade.py -q -x 2>&1 | tail -2
timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-e2e > gpurun_out/r62_auto.json 2>/dev/null; python tools/bench_summary.py "cfg3 auto" gpurun_out/r62_auto.json
timeout 300 python bench.py --config cfg3 --prefix-splits 2 --no-cpu-baseline --no-e2e > gpurun_out/r62_s2.json 2>/dev/null; python tools/bench_summary.py "cfg3 S2" gpurun_out/r62_s2.json
echo "== auto"; KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/cascade_trace.py 2>&1 | tail -9
echo "== S2"; SPLITS=2 KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/cascade_trace.py 2>&1 | tail -9
