cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_cascade.py -x -q > gpurun_out/r2n_tests.log 2>&1; tail -3 gpurun_out/r2n_tests.log
CFG=cfg3 python tools/host_step_profile.py
CFG=cfg2 python tools/host_step_profile.py
export KVFS_LIB_PATH=$PWD/build_var/trace/libkvfs.so
python tools/cascade_trace.py 2>&1 | tail -9
SPLITS=8 python tools/cascade_trace.py 2>&1 | tail -9
