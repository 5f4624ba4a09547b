"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name:
launch_summary.py launches.csv [skip_fraction]   (skip_fraction 0.5 = last half only)"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"].split("(")[0][-44:], float(d["Metric Value"].replace(",", ""))))
out = out[int(len(out) * frac):]
agg = defaultdict(lambda: [0, 0.0])
for k, v in out:
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot / 1e3:.1f} us over {len(out)} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
    print(f"{v[1] / 1e3:9.1f} us {v[0]:5d}x {v[1] / tot * 100:5.1f}%  {k}")
