"""profiles/<round>_kernel_traffic.json from an `ncu --set full` report: DRAM bytes read +
written per launch of each captured kernel, keyed by the bench phase it implements (bench.py
puts the dominant phase's figure in roofline.traffic).

    python tools/kernel_traffic.py gpurun_out/r02_c5_full.ncu-rep profiles/r02_kernel_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

# (the kernels of a phase are summed: the two-pass h = 3 R_co is k_rco3_s + k_rco_epi + the
# clipped-column passes; one search is assumed per report)
PHASE = [("k_acg<3, 256, 0, 1>", "autocorr_sec"), ("k_rco3_s", "autocorr_sec"),
         ("k_rco_epi<2", "autocorr_sec"), ("k_rco_epg<2", "autocorr_sec"),
         ("k_rco_epg9<2", "autocorr_sec"),
         ("k_rco3_clip", "autocorr_sec"), ("k_rco5_s", "autocorr_count"),
         ("k_rco5_cnt", "autocorr_count"), ("k_seg_order", "autocorr_count"),
         ("k_acg<5, 128", "autocorr_count"),
         ("k_wstats4", "window_stats"), ("k_tc_corr<1>", "centre_scan"),
         ("k_centre_epi", "centre_scan_epilogue"), ("k_tc_corr<2>", "survivor_eval"),
         ("k_sec_rows_multi", "sec_multi")]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
res = {"source": sys.argv[1].split("/")[-1], "phases": {}, "kernels": {}}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    b = sum(float(d[k].replace(",", "")) * UNIT.get(u[k], 1)
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    name = d["Kernel Name"]
    t_us = float(d["gpu__time_duration.sum"].replace(",", "")) * (
        1e-3 if u["gpu__time_duration.sum"] == "nsecond" else
        1e3 if u["gpu__time_duration.sum"] == "msecond" else 1.0)
    res["kernels"][name[:90]] = {"dram_bytes": b, "time_us": t_us}
    for key, ph in PHASE:
        if key in name:
            res["phases"][ph] = res["phases"].get(ph, 0.0) + b
            break
json.dump(res, open(sys.argv[2], "w"), indent=1)
print(json.dumps(res["phases"], indent=1))
