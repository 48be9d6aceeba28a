# K1: segments handed from the producer through shared memory, one-round-trip unit merges; cfg3 S=2/3/4, cfg2.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_cascade.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for s in 2 3 4; do
  timeout 300 python bench.py --config cfg3 --prefix-splits $s --no-cpu-baseline --no-e2e > gpurun_out/r58_$s.json 2>/dev/null
  python tools/bench_summary.py "cfg3 S$s" gpurun_out/r58_$s.json
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r58_cfg2.json 2>/dev/null; python tools/bench_summary.py cfg2 gpurun_out/r58_cfg2.json
timeout 300 python bench.py --config cfg5 --no-cpu-baseline --no-e2e > gpurun_out/r58_cfg5.json 2>/dev/null; python tools/bench_summary.py cfg5 gpurun_out/r58_cfg5.json
for s in 2 3; do echo "== SPLITS=$s"; SPLITS=$s KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/cascade_trace.py 2>&1 | tail -8; done
