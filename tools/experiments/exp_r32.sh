cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_cascade.py tests/test_gpu_parity.py tests/test_gpu_scores.py -x -q 2>&1 | tail -3
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/r32_$label.json 2>gpurun_out/r32_$label.err; python tools/bench_summary.py $label gpurun_out/r32_$label.json; }
run auto --config cfg3
run s2 --config cfg3 --prefix-splits 2
run s3 --config cfg3 --prefix-splits 3
run s4 --config cfg3 --prefix-splits 4
run s6 --config cfg3 --prefix-splits 6
run s8 --config cfg3 --prefix-splits 8
run cfg2 --config cfg2
for sp in 0 3 4; do echo "== SPLITS=$sp"; KVFS_LIB_PATH=build_var/trace/libkvfs.so SPLITS=$sp timeout 300 python tools/cascade_trace.py 2>&1; done
