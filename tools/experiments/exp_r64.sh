# prologue as a programmatic launch after the previous step's decode kernel (host reads before the wait).
cd $GRAFT_REPO_ROOT
timeout 300 python tools/sanitize_cases.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_cascade.py tests/test_gpu_parity.py tests/test_gpu_host_io.py -q -x 2>&1 | tail -2
for c in cfg3 cfg2 cfg5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r64_$c.json 2>/dev/null; python tools/bench_summary.py "$c" gpurun_out/r64_$c.json
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prologue|decode_attn|chunk_attn" --csv --log-file gpurun_out/r64_launches_cfg3.csv python bench.py --config cfg3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/r64_launches_cfg3.csv
