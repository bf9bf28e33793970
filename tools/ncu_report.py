"""One reader for the ncu outputs this repo keeps under profiles/ (replaces the
round-1 ncu_summary / ncu_brief / ncu_per_kernel / ncu_lines2 / ncu_stall_lines /
ncu_traffic / launch_summary scripts).

    python tools/ncu_report.py launches LAUNCHES.csv        # --metrics launch list: time, share, DRAM per kernel
    python tools/ncu_report.py full REP.ncu-rep [--lines N]  # --set full capture: key counters, stalls, hot lines
    python tools/ncu_report.py traffic REP.ncu-rep [local=N] # DRAM bytes per launch by kernel family (JSON)
    python tools/ncu_report.py steptraffic LAUNCHES.csv SORTS  # DRAM bytes per sort by kernel class (JSON, bench.py)
"""
import collections
import csv
import json
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
SKIP = ("generate", "k_sorted", "k_digest", "elementwise", "copy", "fill")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "launch__cluster_size" ,
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "lts__t_sectors_op_write.sum", "lts__t_sectors_op_read.sum"]


def short(name):
    return name.split("(")[0].replace("void ", "").replace("radsort::", "").replace("<unnamed>::", "").strip()


def launches(path):
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    by = collections.defaultdict(dict)
    for r in rows:
        d = by[int(r["ID"])]
        d["name"] = short(r["Kernel Name"])
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1)
    agg = collections.OrderedDict()
    for _, d in sorted(by.items()):
        if any(x in d["name"] for x in SKIP):
            continue
        a = agg.setdefault(d["name"], [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0)
        a[3] += d.get("dram__bytes_write.sum", 0)
    tot = sum(v[1] for v in agg.values()) or 1
    print(f"{'kernel':58s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'DRAM rd GB':>10s} {'DRAM wr GB':>10s}")
    for k, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:58]:58s} {n:8d} {t * 1e3:9.2f} {100 * t / tot:5.1f}% {rd / 1e9:10.2f} {wr / 1e9:10.2f}")


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def full(rep, nlines=12):
    h, units, rows = raw_rows(rep)
    for v in rows:
        print(short(v[h.index("Kernel Name")]))
        for k in KEYS:
            if k in h:
                print(f"  {k} = {v[h.index(k)]} {units[h.index(k)]}")
        st = {}
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1
        print("  stalls: " + ", ".join(f"{k}={100 * x / tot:.0f}%" for k, x in sorted(st.items(), key=lambda x: -x[1])[:9]))
    if nlines <= 0:
        return
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    ins, sl, src = collections.Counter(), collections.Counter(), {}
    f = hdr = None
    g = lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0  # noqa: E731
    for row in csv.reader(out.splitlines()):
        if not row:
            continue
        if row[0] == "File Path":
            f = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not row[0].isdigit():
            continue
        key = (f, int(row[0]))
        src[key] = row[1][:80]
        ins[key] += g(row[hdr.index("Instructions Executed")])
        sl[key] += g(row[hdr.index("Warp Stall Sampling (All Samples)")])
    ts, ti = sum(sl.values()) or 1, sum(ins.values()) or 1
    print(f"  hot source lines (warp-stall samples, instructions executed; {ti:.3e} warp instructions):")
    for key, x in sorted(sl.items(), key=lambda x: -x[1])[:nlines]:
        print(f"  {key[0]}:{key[1]:4d} stall {100 * x / ts:5.1f}% inst {100 * ins[key] / ti:5.1f}%  {src[key]}")


def traffic(rep, phase):
    h, units, rows = raw_rows(rep)
    ir, iw, ik = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("Kernel Name")
    fam = collections.defaultdict(list)
    for r in rows:
        name = short(r[ik]).split("<")[0]
        b = float(r[ir].replace(",", "")) * UNIT[units[ir]] + float(r[iw].replace(",", "")) * UNIT[units[iw]]
        key = {"k_scatter": "scatter", "k_hist_pre": "hist", "k_local": "local", "k_local_cluster": "local",
               "k_children": "children"}.get(name, name)
        fam[key].append(b)
    out = {k: round(sum(v) / (phase[k] if k in phase else len(v))) for k, v in fam.items()}
    out["_source"] = f"ncu {rep.split('/')[-1]}: mean dram__bytes_read.sum + dram__bytes_write.sum per launch"
    print(json.dumps(out, indent=1))


CLASSES = {"k_scatter": "scatter", "k_hist_pre": "hist", "k_local": "local", "k_local_pipe": "local",
           "k_local_cluster": "local", "k_children": "children"}


def steptraffic(path, sorts):
    """DRAM bytes (read + write) per sort of each kernel class bench.py times, from a
    --metrics launch list of `sorts` sorts (bench.py divides by its launches per step)."""
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    by = collections.defaultdict(dict)
    for r in rows:
        d = by[int(r["ID"])]
        d["name"] = short(r["Kernel Name"]).split("<")[0]
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1)
    fam = collections.defaultdict(float)
    for d in by.values():
        if d["name"] in CLASSES:
            fam[CLASSES[d["name"]]] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    out = {k: round(v / sorts) for k, v in fam.items()}
    out["_per"] = "step"
    out["_source"] = (f"ncu launch list {path.split('/')[-1]} ({sorts} sorts): dram__bytes_read.sum + "
                      "dram__bytes_write.sum summed per kernel class, per sort")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    cmd, arg = sys.argv[1], sys.argv[2]
    if cmd == "launches":
        launches(arg)
    elif cmd == "full":
        full(arg, int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 12)
    elif cmd == "steptraffic":
        steptraffic(arg, int(sys.argv[3]))
    elif cmd == "traffic":
        traffic(arg, {a.split("=")[0]: int(a.split("=")[1]) for a in sys.argv[3:] if "=" in a})
    else:
        raise SystemExit(__doc__)
