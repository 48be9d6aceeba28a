cd $GRAFT_REPO_ROOT
KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/cascade_trace.py > gpurun_out/r2z_trace.txt 2>&1; cat gpurun_out/r2z_trace.txt
KVFS_LIB_PATH=build_var/trace/libkvfs.so CTAS=592 timeout 300 python tools/cascade_trace.py > gpurun_out/r2z_trace592.txt 2>&1; cat gpurun_out/r2z_trace592.txt
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --no-e2e --config cfg3 "$@" > gpurun_out/r2z_$label.json 2>gpurun_out/r2z_$label.err; python tools/bench_summary.py $label gpurun_out/r2z_$label.json; }
run base
run s8 --prefix-splits 8
run c592 --decode-ctas 592
run s8c592 --prefix-splits 8 --decode-ctas 592
run c1184 --decode-ctas 1184
run s4 --prefix-splits 4
run s2 --prefix-splits 2
