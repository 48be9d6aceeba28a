# K1 software-pipelined sub-blocks (G <= 4): parity subset, holes / cfg3 / cfg2 / cfg5.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scores.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --config cfg5hh --no-cpu-baseline --no-e2e > gpurun_out/r78.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r78.json').read().strip().splitlines()[-1]); e=d['extra']; print('holes ms', round(e['decode_ms_holes'],3), 'compacted', round(e['decode_ms_compacted'],3), d['clocks']['sm_mhz'])"
for c in cfg3 cfg2 cfg5; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r78_$c.json 2>/dev/null; python tools/bench_summary.py $c gpurun_out/r78_$c.json; done
