# K2 with 3 V stages (JR 3): chunk / cascade parity, cfg4 / cfg2d / cfg3, per-tile trace.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_cascade.py tests/test_gpu_parity.py -q -x -k "chunk or cascade" 2>&1 | tail -2
for c in cfg4 cfg2d cfg3; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r68_$c.json 2>/dev/null; python tools/bench_summary.py "$c" gpurun_out/r68_$c.json; done
CFG=cfg3 KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/k2_trace.py 2>&1 | grep -E "period|M:V|M:PF0|M:PV0|S0:PF arr"
CFG=cfg4 KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/k2_trace.py 2>&1 | grep -E "period|M:V|M:PF0|M:PV0|S0:PF arr"
