"""Record-size and key-distribution sweeps (the paper's §4.2 experiments, PAPER.md:262-276:
sorting time against record size / key distribution) on synthetic inputs: ms per sort per
case, device-resident input, CUDA events, every output checked (sorted + multiset digest
unchanged).  One JSON line per case.

    python tools/sweep_bench.py size  [bytes] [steps]    # all built layouts at ~bytes of input, uniform keys
    python tools/sweep_bench.py dist  [n] [steps]        # (8,8) and (16,8), every key distribution of datagen
    python tools/sweep_bench.py case R K n dist [steps]  # one case
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1703_00687_b200 as rs  # noqa: E402
import verify  # noqa: E402
from datagen import device as dd  # noqa: E402

LAYOUTS = [(8, 8), (16, 8), (16, 16), (24, 8), (24, 16), (32, 8), (32, 16), (40, 16)]
DISTS = ["uniform", "uniform40", "zipf", "sorted", "reverse", "few", "equal", "consttop", "bytes"]


def run_case(R, K, n, dist, steps):
    a = dd.generate_tensor(n, R, K, dist, "random", 20260000 + R * 100 + K)
    b = torch.empty_like(a)
    t = torch.empty_like(a)
    dig_in = verify.digest(a.data_ptr(), n, R)
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
    bad, _ = verify.sorted_check(b.data_ptr(), n, R, K)
    ok = bad == 0 and verify.digest(b.data_ptr(), n, R) == dig_in
    st = rs.last_stats()
    med = statistics.median(ms)
    moved = 2 * R * (st["records_scattered"] + st["records_local"] + st["records_tiny"]) + R * st["records_hist"]
    print(json.dumps({"R": R, "K": K, "n": n, "dist": dist, "ms_median": round(med, 3), "ms_min": round(min(ms), 3),
                      "Grec_s": round(n / med / 1e6, 2), "input_GB": round(n * R / 1e9, 2),
                      "algorithmic_GBs": round(moved / med / 1e6, 1), "levels": st["levels"],
                      "scatter_passes": st["scatter_passes"], "first_digit": st["first_digit"], "verified": ok}),
          flush=True)
    del a, b, t
    torch.cuda.empty_cache()
    return ok


def main():
    mode = sys.argv[1]
    rs.init(0)
    ok = True
    if mode == "size":
        nbytes = int(float(sys.argv[2])) if len(sys.argv) > 2 else 16_000_000_000
        steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
        for R, K in LAYOUTS[1:] + LAYOUTS[:1]:  # (8,8) last: at 16 GB it is the paper's 2 G records, the largest n
            ok &= run_case(R, K, min(nbytes // R, 2_000_000_000), "uniform", steps)
    elif mode == "dist":
        n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 500_000_000
        steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
        for R, K in [(8, 8), (16, 8)]:
            for d in DISTS:
                ok &= run_case(R, K, n, d, steps)
    else:
        R, K, n, dist = int(sys.argv[2]), int(sys.argv[3]), int(float(sys.argv[4])), sys.argv[5]
        ok = run_case(R, K, n, dist, int(sys.argv[6]) if len(sys.argv) > 6 else 3)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
