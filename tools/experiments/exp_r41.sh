cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_scores.py tests/test_gpu_outliers.py -x -q 2>&1 | tail -2
run() { label=$1; shift; timeout 300 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/r41_$label.json 2>gpurun_out/r41_$label.err; python tools/bench_summary.py $label gpurun_out/r41_$label.json; python -c "import json,sys; d=json.loads(open('gpurun_out/r41_$label.json').read().strip().splitlines()[-1]); print(json.dumps(d['extra'].get('scores')))"; }
run cfg2_fused --scores --fused-scores
run cfg5_fused --config cfg5 --scores --fused-scores
run cfg2_plain
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:'decode_attn|logit_scores' -s 2 -c 6 --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --scores --fused-scores > gpurun_out/r41_ncu.csv 2>/dev/null
