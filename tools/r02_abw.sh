#!/bin/bash
# local-sort A/B: new lib vs base, plus the W delta of k_local_pipe
set -u
O=gpurun_out/r02; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_fuzz.py -x -q > $O/pytest_w.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_w.log | cut -c1-300
CFGS="c5 c3" bash tools/r02_abv.sh
for wd in -1 1; do
  for c in c5 c3; do
    RADSORT_LOCAL_WDELTA=$wd timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/w_${c}_$wd.json 2> /dev/null
    echo "$c wdelta=$wd $(python -c "import json;d=json.load(open('$O/w_${c}_$wd.json'));print(d['ms_per_step'], {k:round(v,3) for k,v in d['kernel_ms_per_step'].items() if v > 0.05})")"
  done
done
