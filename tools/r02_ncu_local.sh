#!/bin/bash
set -u
O=gpurun_out/r02; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_local$" -c 1 -o $O/c5_local python bench.py --config c5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_l.log 2>&1; echo "l rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_local_cluster" -c 1 -o $O/c4_cluster python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_cl.log 2>&1; echo "cl rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_scatter" -c 2 -o $O/c5_scatter python bench.py --config c5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_sc.log 2>&1; echo "sc rc=$?"
ls -la $O/*.ncu-rep
