"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel totals."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            hdr, start = r, i
            break
    ix = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[ix["Metric Value"]])
        unit = r[ix["Metric Unit"]]
        us = v / 1000 if unit == "ns" else (v if unit == "us" else v * 1000)
        out.append((int(r[ix["ID"]]), r[ix["Kernel Name"]].split("(")[0][-40:], us,
                    r[ix["Grid Size"]], r[ix["Block Size"]]))
    return out


if __name__ == "__main__":
    ks = load(sys.argv[1])
    if "--all" in sys.argv:
        for k in ks:
            print(f"{k[0]:5d} {k[1]:42s} {k[2]:10.1f} us  grid{k[3]} block{k[4]}")
    agg = OrderedDict()
    for k in ks:
        a = agg.setdefault(k[1], [0, 0.0])
        a[0] += 1
        a[1] += k[2]
    tot = sum(a[1] for a in agg.values())
    for name, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:42s} n={c:4d} {us:10.1f} us {100 * us / tot:5.1f}%")
    print(f"total {tot:.1f} us over {len(ks)} launches")
