#!/bin/bash
# Round-2 GPU session: gpu tests, the default bench line (c4), the other configs,
# the c4 launch list and one ncu --set full capture per top kernel.
#   STAGES="tests bench others launches ncu" (default all)
set -u
O=gpurun_out/r02
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
STAGES=${STAGES-"tests bench others launches ncu"}
for st in $STAGES; do
  case $st in
  tests)
    timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log | cut -c1-300 ;;
  bench)
    timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?" ;;
  others)
    for c in ${CFGS-c5 c3 c2 c1 kmc}; do
      RADSORT_LOG=1 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
      echo "bench $c rc=$?"
    done ;;
  launches)
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
      --log-file $O/c4_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo "launches rc=$?" ;;
  ncu)
    for k in ${KS-k_local_cluster k_scatter k_hist_pre}; do
      timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" -c 1 -o $O/c4_$k python bench.py --config ${NCFG-c4} --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
    done ;;
  esac
done
for f in $O/bench_*.json; do echo "$f: $(head -c 300 $f)"; done
