# e2e: host-buffer input copies held until the previous step prologue finished (PCIe read contention test).
cd $GRAFT_REPO_ROOT
for c in cfg2 cfg3; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/r73_${c}_a.json 2>/dev/null; python tools/bench_summary.py "$c as is" gpurun_out/r73_${c}_a.json
  KVFS_EXP_IO_AFTER_PROLOGUE=1 timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/r73_${c}_b.json 2>/dev/null; python tools/bench_summary.py "$c after prologue" gpurun_out/r73_${c}_b.json
done
