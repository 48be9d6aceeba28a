cd $GRAFT_REPO_ROOT
export KVFS_LIB_PATH=$PWD/build_var/trace/libkvfs.so
python tools/cascade_trace.py 2>&1 | tail -9
SPLITS=8 python tools/cascade_trace.py 2>&1 | tail -9
