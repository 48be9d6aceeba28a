cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scores.py tests/test_gpu_outliers.py tests/test_gpu_multilayer.py -x -q 2>&1 | tail -3
run() { label=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/r48_$label.json 2>gpurun_out/r48_$label.err; python -c "
import json; d=json.loads(open('gpurun_out/r48_$label.json').read().strip().splitlines()[-1]); e=d['extra']; print('$label', 'holes ms', round(e['decode_ms_holes'],3), 'GB/s', round(e['decode_gbs_holes']), 'compacted ms', round(e['decode_ms_compacted'],3), d['clocks'])" 2>&1 | tail -1; }
run hh_g1 --config cfg5hh --holes-gather 1
run hh_g0 --config cfg5hh --holes-gather 0
