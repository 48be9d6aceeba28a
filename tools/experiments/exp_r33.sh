cd $GRAFT_REPO_ROOT
for cfg in "2 528" "2 512" "2 496" "3 512" "16 592" "16 512"; do set -- $cfg
echo "== SPLITS=$1 CTAS=$2"
KVFS_LIB_PATH=build_var/trace/libkvfs.so SPLITS=$1 CTAS=$2 timeout 300 python tools/cascade_trace.py 2>&1 | grep -v 'split merge\|phases'
done
