"""Executed-instruction mix by SASS opcode for one kernel of an ncu report (from the
source page's per-instruction 'Instructions Executed'):
    python tools/ncu_opmix.py REP [launch_index] [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(k),
                      "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = rows[1]
seen, mix, stall = set(), collections.Counter(), collections.Counter()
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if d.get("Address") in seen or not (d.get("Instructions Executed") or "").isdigit():
        continue
    seen.add(d["Address"])
    ins = d["Source"].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1] if " " in ins else ins
    op = ins.split()[0] if ins else "?"
    mix[op] += int(d["Instructions Executed"])
    stall[op] += int(d.get("Warp Stall Sampling (All Samples)") or 0)
tot = sum(mix.values()) or 1
stot = sum(stall.values()) or 1
print(f"warp instructions {tot}")
for op, v in mix.most_common(top):
    print(f"{op:28s} {v:10d} {100*v/tot:5.1f}%   stalls {100*stall[op]/stot:5.1f}%")
