# pred_attn_batch_host: GPU tests, e2e of cfg2 / cfg3 / cfg4 / cfg5.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_host_io.py tests/test_gpu_cascade.py -q -x 2>&1 | tail -3
for c in cfg3 cfg2 cfg4 cfg5; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/r59_$c.json 2>gpurun_out/r59_$c.err; python tools/bench_summary.py "$c" gpurun_out/r59_$c.json; tail -2 gpurun_out/r59_$c.err
done
