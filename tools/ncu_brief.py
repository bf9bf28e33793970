"""Brief summary of one ncu report: key metrics + warp stall reasons + top stall lines."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
nlines = int(sys.argv[2]) if len(sys.argv) > 2 else 15
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
keys = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum"]
for k in keys:
    if k in h:
        print(f"  {k} = {v[h.index(k)]}")
st = {}
for i, k in enumerate(h):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
        try:
            st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v[i])
        except ValueError:
            pass
tot = sum(st.values()) or 1
print("  stalls: " + ", ".join(f"{k}={100*x/tot:.0f}%" for k, x in sorted(st.items(), key=lambda x: -x[1])[:9]))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
res = collections.Counter(); sl = collections.Counter(); src = {}
f = None; hdr = None
g = lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0
for row in csv.reader(out.splitlines()):
    if not row: continue
    if row[0] == "File Path": f = row[1].split('/')[-1]; continue
    if row[0] == "Line No": hdr = row; continue
    if hdr is None or not row[0].isdigit(): continue
    key = (f, int(row[0])); src[key] = row[1][:80]
    res[key] += g(row[hdr.index("Instructions Executed")]); sl[key] += g(row[hdr.index("Warp Stall Sampling (All Samples)")])
ts = sum(sl.values()) or 1; ti = sum(res.values()) or 1
for key, x in sorted(sl.items(), key=lambda x: -x[1])[:nlines]:
    print(f"  {key[0]}:{key[1]:4d} stall {100*x/ts:5.1f}% inst {100*res[key]/ti:5.1f}%  {src[key]}")
