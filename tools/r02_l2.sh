#!/bin/bash
set -u
O=gpurun_out/r02; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q ${PYK-} > $O/pytest_l2.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest_l2.log | cut -c1-300
for c in ${CFGS-c5 c4 c3 c2}; do
  for l2 in ${L2S-1 0}; do
    RADSORT_LOCAL2=$l2 RADSORT_LOG=1 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/l2_${c}_$l2.json 2> $O/l2_${c}_$l2.err
    echo "$c local2=$l2 rc=$? $(python -c "import json;d=json.load(open('$O/l2_${c}_$l2.json'));print(d['ms_per_step'], {k:round(v,2) for k,v in d['kernel_ms_per_step'].items()})" 2>&1 | tail -1)"
  done
done
