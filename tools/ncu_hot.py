"""Top SASS lines by warp-stall samples (and the CUDA source lines they map to) of one
kernel in an ncu report:  python tools/ncu_hot.py REP [launch_index] [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25


def page(kind):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(k),
                          "--launch-count", "1", "--print-source", kind],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[1]
    out = [dict(zip(hdr, r)) for r in rows[2:]]
    key = "Warp Stall Sampling (All Samples)"
    return [r for r in out if (r.get(key) or "0").isdigit()]


sass = page("sass")
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in sass) or 1
print(f"SASS lines {len(sass)}, samples {tot}")
for r in sorted(sass, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]:
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{100*s/tot:5.1f}%  {r['Address'][-5:]}  {r['Source'].strip()[:70]}")
src = page("cuda")
tot2 = sum(int(r.get("Warp Stall Sampling (All Samples)") or 0) for r in src) or 1
print("\nCUDA source lines")
for r in sorted(src, key=lambda r: -int(r.get("Warp Stall Sampling (All Samples)") or 0))[:top]:
    s = int(r.get("Warp Stall Sampling (All Samples)") or 0)
    print(f"{100*s/tot2:5.1f}%  L{r.get('#', r.get('Line', '?'))}  {r['Source'].strip()[:90]}")
