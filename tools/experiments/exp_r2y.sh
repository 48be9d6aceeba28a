cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2y_tests.log 2>&1; tail -5 gpurun_out/r2y_tests.log
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/r2y_$label.json 2>gpurun_out/r2y_$label.err; python tools/bench_summary.py $label gpurun_out/r2y_$label.json; python -c "import json,sys; d=json.loads(open('gpurun_out/r2y_$label.json').read().strip().splitlines()[-1]); print(json.dumps(d['extra'].get('scores')))"; }
run cfg2 
run cfg2_fused --scores --fused-scores
run cfg2b 
run cfg2_scores --scores
