"""Per-CUDA-source-line executed warp instructions and stall samples of one kernel in an ncu
report (from the cuda,sass source page):  python tools/ncu_lines.py REP [launch_index] [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(k),
                      "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = None
fname = ""
agg = {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a source line: its aggregated metrics
        d = dict(zip(hdr[:2] + hdr[4:], r[:2] + r[4:]))
        try:
            ins = int(d["Instructions Executed"])
            st = int(d["Warp Stall Sampling (All Samples)"])
        except ValueError:
            continue
        key = (fname, int(r[0]))
        a = agg.setdefault(key, [0, 0, r[1].strip()[:70]])
        a[0] += ins
        a[1] += st
tot = sum(v[0] for v in agg.values()) or 1
stot = sum(v[1] for v in agg.values()) or 1
print(f"warp instructions {tot}, stall samples {stot}")
for (f, ln), (ins, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f}:{ln:<5d} {100*ins/tot:5.1f}% ins {100*st/stot:5.1f}% stall  {src}")
