#!/bin/bash
# Round-2 (second half) c4 profile artefacts, from the repo root on a GPU box:
#   launch list with DRAM bytes of one c4 sort, ncu --set full of the level-0
#   scatter, the wide (10-bit) scatter, the wide histogram and the local sort.
set -u
O=gpurun_out/r02b; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/c4_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
for spec in "k_scatter 0 scatter8" "k_scatter 1 scatter10" "k_hist_pre 1 hist10" "k_local_pipe 0 local"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^$1" --launch-skip $2 -c 1 -o $O/c4_$3 \
    python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_$3.log 2>&1; echo "ncu $3 rc=$?"
done
