"""Per-kernel efficiency table from ncu --set full reports: duration, tensor-pipe activity,
DRAM bytes and bandwidth vs the measured HBM peak, issue utilisation.
    python tools/kernel_table.py report.ncu-rep [...]"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
FAC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TF = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def rows(rep):
    out = []
    k = 0
    while True:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--launch-skip", str(k),
                              "--launch-count", "1"], capture_output=True, text=True).stdout
        r = list(csv.reader(txt.splitlines()))
        if len(r) < 3:
            break
        hdr, units, vals = r[0], r[1], r[2]
        d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))

        def num(key, table=None):
            try:
                v = float(d[key])
            except (KeyError, ValueError):
                return None
            return v * (table or {}).get(u.get(key, ""), 1.0) if table else v
        dur = num("gpu__time_duration.sum", TF)
        rd = num("dram__bytes_read.sum", FAC) or 0.0
        wr = num("dram__bytes_write.sum", FAC) or 0.0
        tens = None
        for key in d:
            if "pipe_tensor_cycles_active" in key and key.endswith("pct_of_peak_sustained_elapsed"):
                tens = num(key)
                break
        out.append({
            "kernel": d.get("Kernel Name", "?").split("(")[0].replace("void ", "").split("::")[-1],
            "dram_read_bytes": rd, "dram_write_bytes": wr,
            "us": dur * 1e6 if dur else None,
            "dram_MB": (rd + wr) / 1e6,
            "dram_GBps": (rd + wr) / dur / 1e9 if dur else None,
            "hbm_frac": (rd + wr) / dur / 1e9 / PEAKS["hbm_gbs"] if dur else None,
            "tensor_pipe_pct": tens,
            "issue_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "occupancy_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
        })
        k += 1
    return out


if __name__ == "__main__":
    if sys.argv[1] == "--json":  # --json OUT REP: per-launch DRAM traffic for bench.py
        out, rep = sys.argv[2], sys.argv[3]
        ks = {f"{i}:{r['kernel']}": {"dram_read_bytes": r["dram_read_bytes"],
                                    "dram_write_bytes": r["dram_write_bytes"],
                                    "duration_us": r["us"]} for i, r in enumerate(rows(rep))}
        json.dump({"source": f"ncu --set full --clock-control none, tools/prof_search.py C2 "
                             f"({os.path.basename(rep)}); cold caches (ncu flushes between "
                             "replays)", "kernels": ks}, open(out, "w"), indent=1)
        sys.exit(0)
    for rep in sys.argv[1:]:
        print(f"## {os.path.basename(rep)}")
        print("| kernel | time (us) | DRAM MB | DRAM GB/s | of HBM peak | tensor pipe % | issue % | occupancy % |")
        print("|---|---|---|---|---|---|---|---|")
        for r in rows(rep):
            f = lambda v, fmt: (fmt % v) if v is not None else "-"
            print(f"| {r['kernel']} | {f(r['us'], '%.1f')} | {f(r['dram_MB'], '%.1f')} | "
                  f"{f(r['dram_GBps'], '%.0f')} | {f(r['hbm_frac'], '%.2f')} | "
                  f"{f(r['tensor_pipe_pct'], '%.1f')} | {f(r['issue_pct'], '%.1f')} | "
                  f"{f(r['occupancy_pct'], '%.1f')} |")
        print()
