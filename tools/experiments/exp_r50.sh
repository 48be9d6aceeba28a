cd $GRAFT_REPO_ROOT
run() { label=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/r50_$label.json 2>gpurun_out/r50_$label.err; python -c "
import json; d=json.loads(open('gpurun_out/r50_$label.json').read().strip().splitlines()[-1]); e=d['extra']; print('$label', 'holes ms', round(e['decode_ms_holes'],3), 'GB/s', round(e['decode_gbs_holes']), 'compacted ms', round(e['decode_ms_compacted'],3), 'compact ms', round(e['compact_ms_device'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
run d80_g1 --config cfg5hh --hh-drop 0.8 --holes-gather 1
run d80_g0 --config cfg5hh --hh-drop 0.8 --holes-gather 0
run d90_g1 --config cfg5hh --hh-drop 0.9 --holes-gather 1
run d90_g0 --config cfg5hh --hh-drop 0.9 --holes-gather 0
