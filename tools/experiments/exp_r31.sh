cd $GRAFT_REPO_ROOT
for cfg in "4 464" "2 0" "4 0" "16 0"; do set -- $cfg
echo "== SPLITS=$1 CTAS=$2"
KVFS_LIB_PATH=build_var/trace/libkvfs.so SPLITS=$1 CTAS=$2 timeout 300 python tools/cascade_trace.py 2>&1
done
