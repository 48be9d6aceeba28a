# fold mode (auto) + bench timing pass: cascade tests, cfg3 / cfg2 lines.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_cascade.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for c in cfg3 cfg2; do
  timeout 300 python bench.py --config $c > gpurun_out/r56_$c.json 2>gpurun_out/r56_$c.err; python tools/bench_summary.py "$c" gpurun_out/r56_$c.json
done
