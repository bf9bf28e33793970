#!/bin/bash
# Round-2 closing sweeps (repo root on the GPU box): the record-size sweep (all built layouts
# at 16 GB of uniform-key input, §4.2), the key-distribution sweep on (8,8) and
# (16,8) at 500 M records, and the paper's 2 G-record size for 8-byte records.
set -u
O=${OUT-gpurun_out/r02e}; mkdir -p $O
timeout 1200 python tools/sweep_bench.py size 16e9 3 > $O/sweep_size.jsonl 2> $O/sweep_size.err; echo "size rc=$?"
timeout 1200 python tools/sweep_bench.py dist 5e8 3 > $O/sweep_dist.jsonl 2> $O/sweep_dist.err; echo "dist rc=$?"
timeout 600 python tools/sweep_bench.py case 16 8 2e9 uniform 3 > $O/sweep_2g.jsonl 2> $O/sweep_2g.err; echo "2g rc=$?"
cat $O/sweep_size.jsonl $O/sweep_dist.jsonl $O/sweep_2g.jsonl | cut -c1-220
