#!/bin/bash
set -u
O=gpurun_out/r02; mkdir -p $O
RADSORT_LOCAL_PIPE=2 timeout 900 python -m pytest tests/test_gpu_sort.py -x -q -k "local or fuzz or size or dist" > $O/pytest_p2.log 2>&1; echo "pytest pipe2 rc=$?"; tail -2 $O/pytest_p2.log | cut -c1-300
for c in c5 c3 c4; do
  for p in 1 2; do
    RADSORT_LOCAL_PIPE=$p timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/p2_${c}_$p.json 2> $O/p2_${c}_$p.err
    echo "$c pipe=$p rc=$? $(python -c "import json;d=json.load(open('$O/p2_${c}_$p.json'));print(d['ms_per_step'], {k:round(v,3) for k,v in d['kernel_ms_per_step'].items() if v > 0.05})" 2>&1 | tail -1)"
  done
done
