#!/bin/bash
set -u
O=gpurun_out/r02; mkdir -p $O
for dw in 0 1; do
  RADSORT_LIB_PATH=$PWD/scratch/libradsort_prof.so RADSORT_CLUSTER_DW=$dw RADSORT_LOG=1 timeout 600 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/clp_dw$dw.json 2> $O/clp_dw$dw.err
  echo "dw=$dw"; grep "prof\]" $O/clp_dw$dw.err | tail -16
done
