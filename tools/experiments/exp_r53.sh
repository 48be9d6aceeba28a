# cfg3 cascade: K1-fold of split records (no in-kernel merge) and L2 prefetch of the prefix range.
cd $GRAFT_REPO_ROOT
KVFS_EXP_PREFIX_FOLD=1 KVFS_EXP_PREFIX_PREFETCH=1 timeout 600 python -m pytest tests/test_gpu_cascade.py -q -x 2>&1 | tail -2
for f in 0 1; do for pf in 0 1; do for s in 2 3 4 8; do
  KVFS_EXP_PREFIX_FOLD=$f KVFS_EXP_PREFIX_PREFETCH=$pf timeout 300 python bench.py --config cfg3 --prefix-splits $s --no-cpu-baseline --no-e2e > gpurun_out/r53_$f$pf$s.json 2>/dev/null
  python tools/bench_summary.py "fold$f pf$pf S$s" gpurun_out/r53_$f$pf$s.json
done; done; done
for s in 2 3 4; do echo "== fold pf SPLITS=$s"; KVFS_EXP_PREFIX_FOLD=1 KVFS_EXP_PREFIX_PREFETCH=1 SPLITS=$s KVFS_LIB_PATH=build_var/trace/libkvfs.so timeout 300 python tools/cascade_trace.py 2>&1 | tail -9; done
