# e2e with the host-buffer call after an untimed slot warm-up.
cd $GRAFT_REPO_ROOT
for c in cfg2 cfg4 cfg5 cfg3; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/r60_$c.json 2>gpurun_out/r60_$c.err; python tools/bench_summary.py "$c" gpurun_out/r60_$c.json; tail -2 gpurun_out/r60_$c.err
done
