# cfg3: host cost per step, and the step with / without the per-layer timing events.
cd $GRAFT_REPO_ROOT
export KVFS_EXP_PREFIX_FOLD=1
CFG=cfg3 timeout 300 python tools/host_step_profile.py 2>&1 | tail -12
for c in cfg3 cfg2; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r55_$c.json 2>/dev/null; python tools/bench_summary.py "$c timed" gpurun_out/r55_$c.json
  BENCH_NO_LAYER_TIMING=1 timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r55_${c}_nt.json 2>/dev/null; python tools/bench_summary.py "$c untimed" gpurun_out/r55_${c}_nt.json
done
