# cfg3 cascade, fold mode: epilogue with hoisted record addresses; phase trace.
cd $GRAFT_REPO_ROOT
for s in 2 3; do
  KVFS_EXP_PREFIX_FOLD=1 timeout 300 python bench.py --config cfg3 --prefix-splits $s --no-cpu-baseline --no-e2e > gpurun_out/r54_$s.json 2>/dev/null
  python tools/bench_summary.py "fold S$s" gpurun_out/r54_$s.json
  echo "== fold SPLITS=$s"; KVFS_EXP_PREFIX_FOLD=1 SPLITS=$s KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/cascade_trace.py 2>&1 | tail -9
done
echo "== no fold SPLITS=8"; SPLITS=8 KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/cascade_trace.py 2>&1 | tail -12
