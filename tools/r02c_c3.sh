#!/bin/bash
# c3 diagnostics: local size classes on/off, and ncu of the level-1 scatter (summarised on the box)
set -u
O=gpurun_out/r02c; mkdir -p $O
SETS="RADSORT_LOCAL_SPLIT=1|RADSORT_LOCAL_SPLIT=0" CFGS="c3 kmc" bash tools/r02c_envab.sh
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_scatter" --launch-skip 1 -c 1 -o $O/c3_scatter_l1 \
  python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_c3_scatter_l1.log 2>&1; echo "ncu rc=$?"
python tools/ncu_report.py full $O/c3_scatter_l1.ncu-rep --lines 30 > $O/ncu_c3_scatter_l1.txt 2>&1; rm -f $O/c3_scatter_l1.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_local<8, 8, 32, 256>" -c 1 -o $O/c3_local256 \
  python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_c3_local256.log 2>&1; echo "ncu rc=$?"
python tools/ncu_report.py full $O/c3_local256.ncu-rep --lines 30 > $O/ncu_c3_local256.txt 2>&1; rm -f $O/c3_local256.ncu-rep
