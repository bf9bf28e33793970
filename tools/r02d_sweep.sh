#!/bin/bash
# env sweep of the local sort's composite-digit width (RADSORT_LOCAL_WDELTA) on c5 / c4 / c2 (repo root on the GPU box)
O=gpurun_out/r02d_sweep; mkdir -p $O
for c in c5 c4 c2; do for w in 0 -1 1; do
  RADSORT_LOCAL_WDELTA=$w timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${c}_w$w.json 2> $O/bench_${c}_w$w.err
  echo "$c wdelta=$w rc=$? $(python -c "import json;d=json.load(open('$O/bench_${c}_w$w.json'));print(d.get('ms_per_step'), {k:round(v,2) for k,v in d.get('kernel_ms_per_step',{}).items() if v>0.05})" 2>&1 | tail -1)"
done; done
