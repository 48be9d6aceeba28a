# K1 partial sub-blocks walk their retained keys packed: parity (holes / eviction / scores), cfg5hh, cfg2, cfg5.
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scores.py tests/test_gpu_fullsize.py tests/test_gpu_cascade.py -q -x 2>&1 | tail -2
for c in cfg5hh cfg2 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r69_$c.json 2>/dev/null; python tools/bench_summary.py "$c" gpurun_out/r69_$c.json; done
python -c "
import json; d=json.loads(open('gpurun_out/r69_cfg5hh.json').read().strip().splitlines()[-1]); e=d['extra']; print('holes ms', round(e['decode_ms_holes'],3), 'GB/s', round(e['decode_gbs_holes']), 'compacted', round(e['decode_ms_compacted'],3))"
timeout 600 python bench.py --config cfg5hh --hh-drop 0.8 --no-cpu-baseline --no-e2e > gpurun_out/r69_d80.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r69_d80.json').read().strip().splitlines()[-1]); e=d['extra']; print('80% holes ms', round(e['decode_ms_holes'],3), 'compacted', round(e['decode_ms_compacted'],3))"
