cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_scores.py tests/test_gpu_outliers.py tests/test_gpu_parity.py -x -q > gpurun_out/r2x_tests.log 2>&1; tail -3 gpurun_out/r2x_tests.log
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/r2x_$label.json 2>gpurun_out/r2x_$label.err; python tools/bench_summary.py $label gpurun_out/r2x_$label.json; python -c "import json,sys; d=json.loads(open('gpurun_out/r2x_$label.json').read().strip().splitlines()[-1]); print(json.dumps(d['extra'].get('scores')))"; }
run cfg2_scores --scores
run cfg2_fused --scores --fused-scores
run cfg5_scores --config cfg5 --scores
run cfg5_fused --config cfg5 --scores --fused-scores
