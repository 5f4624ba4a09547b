import csv,sys,subprocess
rep=sys.argv[1]; k=int(sys.argv[2]) if len(sys.argv)>2 else 0
txt=subprocess.run(["ncu","-i",rep,"--page","raw","--csv","--launch-skip",str(k),"--launch-count","1"],capture_output=True,text=True).stdout
rows=list(csv.reader(txt.splitlines()))
hdr=rows[0]; vals=rows[2] if len(rows)>2 else rows[1]
d=dict(zip(hdr,vals))
print(d.get("Kernel Name","")[:60], d.get("gpu__time_duration.sum"))
st={k:v for k,v in d.items() if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued')}
tot=sum(float(v or 0) for v in st.values()) or 1
for kk,v in sorted(st.items(), key=lambda kv:-float(kv[1] or 0))[:8]:
    print(f"  {kk.replace('smsp__pcsamp_warps_issue_stalled_',''):30s} {100*float(v)/tot:.1f}%")
for key in ["sm__inst_executed.sum","smsp__inst_executed.sum","l1tex__t_sector_hit_rate.pct","lts__t_sector_hit_rate.pct","dram__bytes_read.sum","dram__bytes_write.sum","sm__warps_active.avg.pct_of_peak_sustained_active","smsp__inst_executed_op_global_ld.sum","l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum","l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]:
    if key in d: print(f"  {key:55s} {d[key]}")
