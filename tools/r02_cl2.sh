#!/bin/bash
set -u
O=gpurun_out/r02
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "cluster" > $O/pytest_cl.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_cl.log
for dw in 0 1; do
  RADSORT_CLUSTER_DW=$dw RADSORT_LOG=1 timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/cl_dw$dw.json 2> $O/cl_dw$dw.err
  echo "dw=$dw rc=$? $(grep 'level 1 ms' $O/cl_dw$dw.err | tail -1)"
  RADSORT_LIB_PATH=$PWD/scratch/libradsort_prof.so RADSORT_CLUSTER_DW=$dw RADSORT_LOG=1 timeout 600 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/clp_dw$dw.json 2> $O/clp_dw$dw.err
  grep "prof\] local" $O/clp_dw$dw.err | tail -8
done
