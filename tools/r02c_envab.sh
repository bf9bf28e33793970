#!/bin/bash
# A/B over env settings: SETS="A=1 B=2|A=0" CFGS="c4 c5" bash tools/r02c_envab.sh  (per-level ms with RADSORT_LOG=1)
set -u
O=gpurun_out/r02c; mkdir -p $O
IFS='|' read -ra SL <<< "${SETS}"
for c in ${CFGS-c4}; do
  for set in "${SL[@]}"; do
    tag=$(echo "$set" | tr ' =' '_-')
    env $set RADSORT_LOG=1 timeout 600 python bench.py --config $c --steps ${STEPS-3} --warmup 3 --no-cpu-baseline --no-e2e > $O/ab_${c}_$tag.json 2> $O/ab_${c}_$tag.err
    echo "$c [$set] rc=$? $(python -c "import json;d=json.load(open('$O/ab_${c}_$tag.json'));print(d['ms_per_step'], {k:round(v,2) for k,v in d['kernel_ms_per_step'].items() if v > 0.05})" 2>&1 | tail -1)"
    grep "level . ms" $O/ab_${c}_$tag.err | tail -4 | sed 's/^/    /'
  done
done
