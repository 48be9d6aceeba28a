"""Print the key fields of a set of bench lines (profiles/bench_<tag>_*.json): value, ms per step, kernel time,
roofline, e2e, clocks, plus the workload-specific extras (holes / compaction, scores, copies)."""
import glob
import json
import os
import sys


def main():
    tag = sys.argv[1]
    for f in sorted(glob.glob(f"profiles/bench_{tag}_*.json")):
        c = os.path.basename(f)[len(f"bench_{tag}_"):-5]
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r, e, ex = d.get("roofline") or {}, d.get("e2e") or {}, d.get("extra") or {}
        print(f"{c:16s} value {d.get('value') or 0:12.0f} ms/step {d.get('ms_per_step') or 0:8.4f} kernel "
              f"{r.get('kernel_ms_mean') or 0:8.4f} {r.get('bound')} achieved {r.get('achieved') or 0:7.0f} "
              f"frac {r.get('frac') or 0:5.3f} e2e {e.get('value') or 0:10.0f} clk {(d.get('clocks') or {}).get('sm_mhz')}")
        for k in ("decode_ms_holes", "decode_ms_compacted", "compact_ms_device", "pack_kernel_ms", "offload_kernel_gbs"):
            if k in ex:
                print(f"    {k} {ex[k]:.3f}")
        if "scores" in ex:
            sc = ex["scores"]
            print(f"    scores ms {sc.get('ms_mean', 0):.4f} overhead {sc.get('overhead_vs_attention', 0):.3f}")


if __name__ == "__main__":
    main()
