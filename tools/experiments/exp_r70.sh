# host-buffer pred with packed (slot-layout) host buffers: one copy each way; e2e of cfg3 / cfg2.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_host_io.py -q -x 2>&1 | tail -2
for c in cfg3 cfg2 cfg4; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/r70_$c.json 2>/dev/null; python tools/bench_summary.py "$c" gpurun_out/r70_$c.json; done
