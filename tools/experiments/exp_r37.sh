cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_cascade.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/r37_$label.json 2>gpurun_out/r37_$label.err; python tools/bench_summary.py $label gpurun_out/r37_$label.json; }
run auto --config cfg3
run s2 --config cfg3 --prefix-splits 2
run s3 --config cfg3 --prefix-splits 3
run s16 --config cfg3 --prefix-splits 16
for cfg in "0 0" "3 0"; do set -- $cfg
echo "== SPLITS=$1 CTAS=$2"
KVFS_LIB_PATH=build_var/trace/libkvfs.so SPLITS=$1 CTAS=$2 timeout 300 python tools/cascade_trace.py 2>&1 | grep -v 'split merge\|phases'
done
