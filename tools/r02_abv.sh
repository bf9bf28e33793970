#!/bin/bash
# A/B of the in-tree library against scratch/libradsort_<VARIANT>.so (tools/build_variant.sh), alternating runs
set -u
O=gpurun_out/r02; mkdir -p $O
V=${VARIANT-base}
for c in ${CFGS-c5 c3 c4 c2}; do
  for rep in 1 2; do
    for lib in new $V; do
      if [ $lib = new ]; then LP=""; else LP=$PWD/scratch/libradsort_$V.so; fi
      RADSORT_LIB_PATH=$LP timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/abv_${c}_$lib.json 2> $O/abv_${c}_$lib.err
      echo "$c $lib rc=$? $(python -c "import json;d=json.load(open('$O/abv_${c}_$lib.json'));print(d['ms_per_step'], {k:round(v,3) for k,v in d['kernel_ms_per_step'].items() if v > 0.05})" 2>&1 | tail -1)"
    done
  done
done
