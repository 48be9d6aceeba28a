cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_cascade.py tests/test_gpu_parity.py tests/test_gpu_outliers.py -x -q > gpurun_out/r2l_tests.log 2>&1; tail -3 gpurun_out/r2l_tests.log
export KVFS_LIB_PATH=$PWD/build_var/trace/libkvfs.so
python tools/cascade_trace.py > gpurun_out/r2l_trace.txt 2>&1; cat gpurun_out/r2l_trace.txt
SPLITS=8 python tools/cascade_trace.py > gpurun_out/r2l_trace_s8.txt 2>&1; cat gpurun_out/r2l_trace_s8.txt
unset KVFS_LIB_PATH
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --steps 50 --warmup 10 "$@" > gpurun_out/r2l_$label.json 2>gpurun_out/r2l_$label.err; python tools/bench_summary.py $label gpurun_out/r2l_$label.json; }
run cfg3 --config cfg3
run cfg3s8 --config cfg3 --prefix-splits 8
run cfg2
