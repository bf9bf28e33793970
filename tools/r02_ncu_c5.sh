#!/bin/bash
set -u
O=gpurun_out/r02; mkdir -p $O
for k in ${KS-k_scatter k_local}; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^$k" -c 1 -o $O/c5_$k python bench.py --config c5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_c5_$k.log 2>&1; echo "ncu $k rc=$?"
done
