#!/bin/bash
# ncu --set full (source-level) of k_local_pipe on c5 and c4
set -u
O=gpurun_out/r02c; mkdir -p $O
for c in ${CFGS-c5 c4}; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_local_pipe" -c 1 -o $O/${c}_local_pipe \
    python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_${c}.log 2>&1; echo "ncu $c rc=$?"
done
