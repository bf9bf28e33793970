#!/bin/bash
# Round-2 GPU session: tests, bench lines, per-level timings (run from the repo root on the GPU box).
#   STAGES="tests bench levels" (default all)
set -u
O=gpurun_out/r02
mkdir -p $O
STAGES=${STAGES-"tests bench levels"}
for st in $STAGES; do
  case $st in
  tests)
    timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" ;;
  bench)
    timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
    for c in ${CFGS-c5 c3 c2}; do
      timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
      echo "bench $c rc=$?"
    done ;;
  levels)
    for c in ${LCFGS-c4 c5 c3}; do
      RADSORT_LOG=1 timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/log_$c.json 2> $O/log_$c.err
    done ;;
  esac
done
tail -n 3 $O/pytest_gpu.log 2>/dev/null
for f in $O/bench_*.json; do echo "$f: $(head -c 400 $f)"; done
