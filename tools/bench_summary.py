"""One-line summary of a bench.py JSON line (tuning runs): label, step / kernel ms, roofline fraction, clocks."""
import json
import sys

label, path = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(path).read().strip().splitlines()[-1])
except Exception as e:  # noqa: BLE001
    print(label, "FAILED", e)
    sys.exit(0)
r = d.get("roofline", {})
print(f"{label:28s} ms/step {d.get('ms_per_step', 0):.4f} kernel {r.get('kernel_ms_mean', 0):.4f} "
      f"frac {r.get('frac', 0):.3f} {r.get('unit', '')} ach {r.get('achieved', 0):.0f} "
      f"e2e {d.get('e2e', {}).get('value', 0):.0f} clk {d.get('clocks', {}).get('sm_mhz')} "
      f"{d.get('clocks', {}).get('reasons')} ctas {d.get('extra', {}).get('decode_ctas')}")
