"""Summarise an ncu report: key metrics per kernel + hottest SASS lines (stall samples)."""
import csv
import io
import subprocess
import sys

REP = sys.argv[1]
KEYS = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Executed Ipc Active",
        "Issue Slots Busy", "Dynamic Shared Memory Per Block", "Waves Per SM",
        "Block Limit Shared Mem", "Block Limit Registers"]


def run(args):
    return subprocess.run(["ncu", "-i", REP] + args, capture_output=True, text=True).stdout


def details():
    rows = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    out = {}
    for r in rows[1:]:
        k = (r[ix["ID"]], r[ix["Kernel Name"]][:60])
        if r[ix["Metric Name"]] in KEYS:
            out.setdefault(k, {})[r[ix["Metric Name"]]] = r[ix["Metric Value"]] + " " + r[ix["Metric Unit"]]
    return out


def hot(kid, top=20):
    txt = run(["--page", "source", "--csv", "--launch-skip", str(kid), "--launch-count", "1"])
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return []
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data, seen = [], set()
    for r in rows[2:]:
        try:
            a = r[ix["Address"]]
            if a in seen:
                continue
            seen.add(a)
            data.append((int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)),
                         int(float(r[ix["Instructions Executed"]] or 0)), r[ix["Source"]][:70]))
        except Exception:
            pass
    tot = sum(d[0] for d in data) or 1
    data.sort(reverse=True)
    return [(round(100 * d[0] / tot, 1), d[1], d[2]) for d in data[:top]]


if __name__ == "__main__":
    det = details()
    for i, ((kid, name), m) in enumerate(det.items()):
        print(f"== [{kid}] {name}")
        for k in KEYS:
            if k in m:
                print(f"   {k:32s} {m[k]}")
        if "--hot" in sys.argv:
            for h in hot(i):
                print("     ", h)
