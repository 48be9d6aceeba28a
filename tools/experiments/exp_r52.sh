# cfg3 cascade phase traces at several key-split counts (globaltimer stamps, trace build).
cd $GRAFT_REPO_ROOT
for s in 0 2 3 4 8 16; do echo "== SPLITS=$s"; SPLITS=$s KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/cascade_trace.py 2>&1 | tail -12; done
