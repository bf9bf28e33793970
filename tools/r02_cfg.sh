#!/bin/bash
# scatter tile configurations (RADSORT_SCATTER_CFG) on c4 / c5 / c2
set -u
O=gpurun_out/r02; mkdir -p $O
for c in ${CFGS-c4 c5 c2}; do
  for cfg in 1 0 2 4 3; do
    RADSORT_SCATTER_CFG=$cfg timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/cfg_${c}_$cfg.json 2> /dev/null
    echo "$c cfg=$cfg $(python -c "import json;d=json.load(open('$O/cfg_${c}_$cfg.json'));print(d['ms_per_step'], {k:round(v,3) for k,v in d['kernel_ms_per_step'].items() if v > 0.05})" 2>&1 | tail -1)"
  done
done
