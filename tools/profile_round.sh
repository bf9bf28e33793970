#!/bin/bash
# Round measurement artefacts (run on the GPU box from the repo root):
#   gpurun_out/prof/bench_all.jsonl      bench.py line per config (c2 with cpu_baseline + e2e)
#   gpurun_out/prof/bench_reference.json bench.py --impl reference (the oracle arm)
#   gpurun_out/prof/c2_launches.csv      ncu launch list of the default bench (gpu__time_duration.sum)
#   gpurun_out/prof/<cfg>_full.ncu-rep   ncu --set full of one sort's hist/scatter/local launches
set -u
mkdir -p gpurun_out/prof
O=gpurun_out/prof
: > $O/bench_all.jsonl
timeout 600 python bench.py --steps 5 --warmup 3 >> $O/bench_all.jsonl 2> $O/bench_c2.err
for c in c1 c3 c4 c5 kmc; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $O/bench_all.jsonl 2> $O/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/c2_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
for c in ${FULL-c2 c5}; do  # FULL="" skips (the return limit is 64 MiB)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_local|k_hist_pre" -c 5 \
    -o $O/${c}_full python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_$c.log 2>&1
done
# the cluster local sort (c4's dominant phase): one full capture
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_local_cluster" -c 1 \
  -o $O/c4_cluster_full python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_c4cl.log 2>&1
# DRAM bytes per launch only (small reports; the gpurun return limit is 64 MiB)
for c in c3 c4 kmc; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_scatter|k_local|k_hist_pre|k_children" -c 12 \
    -o $O/${c}_dram python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_$c.log 2>&1
done
ls -la $O
