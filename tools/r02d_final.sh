#!/bin/bash
# Round-2 closing measurement session (repo root on the GPU box).  STAGES selects:
#   tests  pytest -m gpu
#   bench  the default bench line (c4) + c5 c3 c2 c1 kmc + the reference arm
#   launches  ncu launch lists with DRAM bytes (c4, c5, c2, c3) -> traffic per kernel class
#   ncu    ncu --set full of the top kernels of c4 and c5
set -u
O=${OUT-gpurun_out/r02d_final}; mkdir -p $O
STAGES=${STAGES-"tests bench launches ncu"}
NCU_SPECS=${NCU_SPECS-"c4 k_local_pipe 0 local|c4 k_scatter 0 scatter8|c4 k_scatter 1 scatter10|c4 k_hist_pre 1 hist10|c5 k_local_pipe 0 local|c5 k_scatter 0 scatter8"}
for st in $STAGES; do
  case $st in
  tests) timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log | cut -c1-300 ;;
  bench)
    timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
    for c in c5 c3 c2 c1 kmc; do
      RADSORT_LOG=1 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
      echo "bench $c rc=$?"
    done
    timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_ref.err; echo "ref rc=$?" ;;
  launches)
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
      --log-file $O/c4_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
    for c in c5 c3 c2; do
      timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
        --log-file $O/${c}_launches.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch_$c.log 2>&1; echo "launches $c rc=$?"
    done ;;
  ncu)
    IFS='|' read -ra SPECS <<< "$NCU_SPECS"
    for spec in "${SPECS[@]}"; do
      set -- $spec
      timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^$2" --launch-skip $3 -c 1 -o $O/${1}_$4 \
        python bench.py --config $1 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_${1}_$4.log 2>&1; echo "ncu $1 $4 rc=$?"
      # summarised here (the reports are too big to bring back): counters, stalls, hot lines, DRAM traffic
      { echo "=== $1 $4 (ncu --set full --clock-control none, 1 launch; tools/r02d_final.sh)"; python tools/ncu_report.py full $O/${1}_$4.ncu-rep --lines 25; } > $O/ncu_${1}_$4.txt 2>&1
      rm -f $O/${1}_$4.ncu-rep
    done ;;
  esac
done
for f in $O/bench_*.json; do echo "$f: $(python -c "import json;d=json.load(open('$f'));print(d.get('ms_per_step'), d.get('value'), {k:round(v,2) for k,v in d.get('kernel_ms_per_step',{}).items() if v>0.05})" 2>&1 | tail -1)"; done
