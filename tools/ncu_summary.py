import csv, sys, subprocess
rep = sys.argv[1]
raw = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
r = list(csv.reader(raw.splitlines())); h=r[0]
keys=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','launch__registers_per_thread','launch__grid_size','launch__occupancy_limit_registers','lts__t_sector_hit_rate.pct','smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__throughput.avg.pct_of_peak_sustained_active']
for row in r[2:]:
    print('-----')
    for k in keys:
        if k in h: print(f"  {k:60s} {row[h.index(k)][:60]} {r[1][h.index(k)]}")
    items=[(float(row[i] or 0),h[i]) for i,x in enumerate(h) if x.startswith('smsp__pcsamp_warps_issue_stalled') and not x.endswith('not_issued')]
    tot=sum(a for a,_ in items) or 1
    print('  stalls:', ', '.join(f'{n.replace("smsp__pcsamp_warps_issue_stalled_","")} {v/tot*100:.0f}%' for v,n in sorted(items, reverse=True)[:6]))
