"""One sort of a BASELINE config with per-level logging and the final stats (diagnostics).

    RADSORT_LOG=1 python tools/level_stats.py c3
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1703_00687_b200 as rs  # noqa: E402
from datagen import device as dd  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
rs.init(0)
a = dd.generate_config(cfg)
t = torch.empty_like(a)
K = dd.CONFIGS[cfg]["K"]
for _ in range(2):
    b = a.clone()
    torch.cuda.synchronize()
    rs.sort(b, t, K)
    torch.cuda.synchronize()
st = rs.last_stats()
print(json.dumps({k: v for k, v in st.items() if k not in ("kernel_ms", "kernel_bytes")}, indent=0))
