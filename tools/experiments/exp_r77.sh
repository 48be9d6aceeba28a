# K1 with 4 consumer warps per ring (2 rings per CTA) on the consumer-latency-bound workloads.
cd $GRAFT_REPO_ROOT
for lib in paper_2510_25412_b200/libkvfs.so build_var/nw4/libkvfs.so; do
  echo "== $lib"
  KVFS_LIB_PATH=$lib timeout 600 python bench.py --config cfg5hh --no-cpu-baseline --no-e2e > gpurun_out/r77.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r77.json').read().strip().splitlines()[-1]); e=d['extra']; print('holes ms', round(e['decode_ms_holes'],3), 'compacted', round(e['decode_ms_compacted'],3), d['clocks']['sm_mhz'])"
  KVFS_LIB_PATH=$lib timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-e2e > gpurun_out/r77.json 2>/dev/null; python tools/bench_summary.py cfg3 gpurun_out/r77.json
  KVFS_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r77.json 2>/dev/null; python tools/bench_summary.py cfg2 gpurun_out/r77.json
done
