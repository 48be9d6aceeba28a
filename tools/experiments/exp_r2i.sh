cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cascade.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2i_tests.log 2>&1; tail -2 gpurun_out/r2i_tests.log
export KVFS_LIB_PATH=$PWD/build_var/trace/libkvfs.so
python tools/cascade_trace.py 2>&1 | tee gpurun_out/r2i_trace_default.txt
unset KVFS_LIB_PATH
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 5 "$@" > gpurun_out/r2i_$label.json 2>gpurun_out/r2i_$label.err; python tools/bench_summary.py $label gpurun_out/r2i_$label.json; }
run cfg2
run cfg3 --config cfg3
run cfg3_dyn1024 --config cfg3 --decode-chunks 1024
run cfg5 --config cfg5
