"""ms per sort for one record layout (device-resident input, CUDA events; diagnostics).

    python tools/layout_bench.py R K n [dist] [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1703_00687_b200 as rs  # noqa: E402
from datagen import device as dd  # noqa: E402

R, K, n = int(sys.argv[1]), int(sys.argv[2]), int(float(sys.argv[3]))
dist = sys.argv[4] if len(sys.argv) > 4 else "uniform"
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
rs.init(0)
a = dd.generate_tensor(n, R, K, dist, "random", 12345)
b = torch.empty_like(a)
t = torch.empty_like(a)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for i in range(steps + 2):
    b.copy_(a)
    torch.cuda.synchronize()
    e0.record()
    rs.sort(b, t, K)
    e1.record()
    torch.cuda.synchronize()
    if i >= 2:
        ms.append(e0.elapsed_time(e1))
st = rs.last_stats()
print(json.dumps({"R": R, "K": K, "n": n, "dist": dist, "ms": round(min(ms), 3), "cluster_env": os.environ.get("RADSORT_CLUSTER"),
                  "levels": st["levels"], "scatter_passes": st["scatter_passes"]}))
