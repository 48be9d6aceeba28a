# flat table deltas in the step prologue: GPU tests, cfg3 / cfg2 bench, cfg3 launch list.
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r57_tests.log 2>&1; tail -2 gpurun_out/r57_tests.log
for c in cfg3 cfg2; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r57_$c.json 2>gpurun_out/r57_$c.err; python tools/bench_summary.py "$c" gpurun_out/r57_$c.json
done
K="upload|prologue|decode_attn|chunk_attn"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" --csv --log-file gpurun_out/r57_launches_cfg3.csv python bench.py --config cfg3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -c prologue gpurun_out/r57_launches_cfg3.csv
