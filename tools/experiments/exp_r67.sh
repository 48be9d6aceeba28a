# K2 per-tile pipeline timeline: prefix kernel (cfg3, CTA 0 = a single 14-tile unit) and chunk kernel (cfg4).
cd $GRAFT_REPO_ROOT
CFG=cfg3 KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/k2_trace.py 2>&1 | tail -40
CFG=cfg4 KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/k2_trace.py 2>&1 | tail -34
