#!/bin/bash
# A/B of the cluster local sort variants on c4 + the tests that cover it.
set -u
O=gpurun_out/r02
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "cluster or multi or fuzz or c4 or level0 or outlier" > $O/pytest_cl.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_cl.log
for dw in 0 1; do
  RADSORT_CLUSTER_DW=$dw RADSORT_LOG=1 timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/cl_dw$dw.json 2> $O/cl_dw$dw.err
  echo "dw=$dw rc=$? $(grep 'level 1 ms' $O/cl_dw$dw.err | tail -1)"
  python -c "import json;d=json.load(open('$O/cl_dw$dw.json'));print(d['ms_per_step'], d['kernel_ms_per_step'])"
done
