cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_outliers.py -x -q > gpurun_out/r2k_tests.log 2>&1; tail -15 gpurun_out/r2k_tests.log
export KVFS_LIB_PATH=$PWD/build_var/trace/libkvfs.so
python tools/cascade_trace.py > gpurun_out/r2k_trace.txt 2>&1; cat gpurun_out/r2k_trace.txt
SPLITS=4 python tools/cascade_trace.py > gpurun_out/r2k_trace_s4.txt 2>&1; cat gpurun_out/r2k_trace_s4.txt
