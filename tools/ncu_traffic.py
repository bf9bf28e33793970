"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
radsort kernels in an ncu report -> profiles/traffic_<config>.json (read by bench.py)."""
import csv
import json
import subprocess
import sys
from collections import defaultdict

rep, out = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, units = rows[0], rows[1]
ki, ri, wi, ti = (hdr.index(x) for x in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                          "gpu__time_duration.sum"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
acc = defaultdict(list)
for r in rows[2:]:
    name = r[ki]
    cls = "scatter" if "k_scatter" in name else "local" if "k_local" in name else "hist" if "k_hist" in name else None
    if not cls:
        continue
    b = float(r[ri]) * scale.get(units[ri], 1) + float(r[wi]) * scale.get(units[wi], 1)
    acc[cls].append(b)
res = {k: round(sum(v) / len(v)) for k, v in acc.items()}
res["_source"] = f"ncu --set full, {rep.split('/')[-1]}: mean dram__bytes_read.sum + dram__bytes_write.sum per launch"
json.dump(res, open(out, "w"), indent=1)
print(res)
