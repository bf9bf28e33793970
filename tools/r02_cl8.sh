#!/bin/bash
# A/B of the cluster shapes on c4 (8x256 two per SM vs 4x512) + the tests that cover them
set -u
O=gpurun_out/r02; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "cluster or c4 or fuzz or multi" > $O/pytest_cl8.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_cl8.log | cut -c1-300
for cfg in 8 4; do
  RADSORT_CLUSTER_CFG=$cfg RADSORT_LOG=1 timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/cl8_$cfg.json 2> $O/cl8_$cfg.err
  echo "cfg=$cfg rc=$? $(grep 'clusters resident' $O/cl8_$cfg.err | head -2)"
  python -c "import json;d=json.load(open('$O/cl8_$cfg.json'));print(d['ms_per_step'], {k:round(v,2) for k,v in d['kernel_ms_per_step'].items() if v>0.05})"
done
