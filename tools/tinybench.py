"""Tiny-sorter grid (GPU analog of PAPER.md Fig. 1, §4.1): ns per record of each
device tiny sorter for n = 2..128 and three layouts -> stdout (profiles/r01_tinybench.txt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00687_b200 as rs  # noqa: E402

rs.init(0)
NS = [2, 4, 8, 12, 16, 24, 32, 48, 64, 96, 128]
for R, K in [(8, 8), (16, 8), (32, 16)]:
    print(f"# layout R={R} K={K}: ns per record (2^20 records per run, best of 3)")
    print("n     " + "".join(f"{rs.TINY_ALGOS[a][:22]:>26s}" for a in range(4)))
    for n in NS:
        row = []
        for a in range(4):
            if a == 0 and n > 32:
                row.append(f"{'-':>26s}")
                continue
            row.append(f"{rs.tinybench(R, K, n, a, bins=max(1, (1 << 20) // n)):26.4f}")
        print(f"{n:<6d}" + "".join(row))
    print()
