#!/bin/bash
# A/B: VAR=name VALS="1 0" CFGS="c5 c3" [PYK="tests..."] bash tools/r02_ab.sh
set -u
O=gpurun_out/r02; mkdir -p $O
if [ -n "${PYK-}" ]; then
  timeout 900 python -m pytest -x -q -m gpu $PYK > $O/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_ab.log | cut -c1-300
fi
for c in ${CFGS-c5 c3}; do
  for v in ${VALS-1 0}; do
    env $VAR=$v RADSORT_LOG=1 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ab_${c}_$v.json 2> $O/ab_${c}_$v.err
    echo "$c $VAR=$v rc=$? $(python -c "import json;d=json.load(open('$O/ab_${c}_$v.json'));print(d['ms_per_step'], {k:round(v,2) for k,v in d['kernel_ms_per_step'].items() if v > 0.05})" 2>&1 | tail -1)"
  done
done
