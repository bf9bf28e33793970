#!/bin/bash
# per-phase cycle counters (-DRADSORT_PHASE_PROF build, tools/build_prof.sh) on the given configs
set -u
O=gpurun_out/r02; mkdir -p $O
for c in ${CFGS-c4 c5}; do
  RADSORT_LIB_PATH=$PWD/scratch/libradsort_prof.so RADSORT_LOG=1 ${ENVS-} timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/prof_$c.json 2> $O/prof_$c.err
  echo "$c rc=$?"; grep "radsort prof\|level . ms" $O/prof_$c.err | tail -22
done
