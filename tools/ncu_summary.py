import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = ['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum',
 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.pct_of_peak_sustained_active',
 'launch__registers_per_thread','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','sm__throughput.avg.pct_of_peak_sustained_elapsed',
 'smsp__issue_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','launch__grid_size','launch__block_size',
 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
 'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum','l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum','lts__t_sectors_op_write.sum','lts__t_sectors_op_read.sum']
for r in rows[2:]:
    for w in want:
        if w in hdr: print(f"  {w} = {r[hdr.index(w)]}")
    st = [(h, float(r[i])) for i, h in enumerate(hdr) if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued') and r[i] not in ('', 'n/a')]
    st.sort(key=lambda x: -x[1])
    tot = sum(v for _, v in st) or 1
    print("  stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_','')}={100*v/tot:.0f}%" for h, v in st[:8]))
    print()
