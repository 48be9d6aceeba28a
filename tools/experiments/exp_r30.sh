cd $GRAFT_REPO_ROOT
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/r30_$label.json 2>gpurun_out/r30_$label.err; python tools/bench_summary.py $label gpurun_out/r30_$label.json; }
run s4c464 --config cfg3 --prefix-splits 4 --decode-ctas 464
run s2c528 --config cfg3 --prefix-splits 2 --decode-ctas 528
run s3c496 --config cfg3 --prefix-splits 3 --decode-ctas 496
run s8c336 --config cfg3 --prefix-splits 8 --decode-ctas 336
run s4c460 --config cfg3 --prefix-splits 4 --decode-ctas 460
run s5c432 --config cfg3 --prefix-splits 5 --decode-ctas 432
run s2 --config cfg3 --prefix-splits 2
run cfg2_fused --scores --fused-scores
python -c "import json,sys; d=json.loads(open('gpurun_out/r30_cfg2_fused.json').read().strip().splitlines()[-1]); print(json.dumps(d['extra'].get('scores')))"
timeout 300 python -m pytest tests/test_gpu_scores.py tests/test_gpu_outliers.py -x -q 2>&1 | tail -2
