"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, mean, share."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
agg = collections.OrderedDict()
for d in data:
    name = d["Kernel Name"].split("(")[0].replace("unnamed>::", "")
    agg.setdefault(name, []).append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
print(f"{len(data)} launches, {tot / 1e3:.1f} us total (cold-cache, serialised)")
for name, v in agg.items():
    print(f"  {name[:60]:60s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.2f} us  share={100 * sum(v) / tot:5.1f}%")
