"""DRAM traffic per launch by kernel family from an ncu report (dram__bytes_read.sum + dram__bytes_write.sum).

    python tools/ncu_traffic.py gpurun_out/prof/c4_dram.ncu-rep [--phase-launches local=2]

Prints JSON {family: mean bytes per launch}; "local" is the on-chip sort phase
(k_local + k_local_cluster) divided by the phase's launches per level, the way
bench.py counts them (--phase-launches local=N)."""
import collections
import csv
import json
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    rep = sys.argv[1]
    phase = {}
    for a in sys.argv[2:]:
        if a.startswith("--phase-launches"):
            continue
        k, v = a.split("=")
        phase[k] = int(v)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    ir, iw, ik = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("Kernel Name")
    fam = collections.defaultdict(list)
    for r in rows[2:]:
        name = r[ik].split("<")[0].replace("void ", "").strip()
        b = float(r[ir].replace(",", "")) * UNIT[units[ir]] + float(r[iw].replace(",", "")) * UNIT[units[iw]]
        key = {"k_scatter": "scatter", "k_hist_pre": "hist", "k_local": "local", "k_local_cluster": "local",
               "k_children": "children"}.get(name, name)
        fam[key].append((name, b))
    out = {}
    for k, v in fam.items():
        if k == "local" and "local" in phase:
            out[k] = round(sum(b for _, b in v) / phase["local"])
        else:
            out[k] = round(sum(b for _, b in v) / len(v))
    out["_source"] = f"ncu {rep.split('/')[-1]}: mean dram__bytes_read.sum + dram__bytes_write.sum per launch"
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
