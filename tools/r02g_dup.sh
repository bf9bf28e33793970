#!/bin/bash
# The duplicate-gated wide-level rule for R < 24 (k_dupest): tests, then the sizes it changes
# and the configs it must not change.
set -u
O=${OUT-gpurun_out/r02g}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sort.py -m gpu -x -q -k "wide" > $O/pytest_wide.log 2>&1; echo "pytest wide rc=$?"; tail -2 $O/pytest_wide.log | cut -c1-300
for cs in "16 8 1e9 uniform" "16 16 1e9 uniform" "8 8 2e9 uniform" "16 8 2e9 uniform" "16 8 1e9 zipf" "8 8 2e9 zipf" "16 16 413e6 kmer" "8 8 2e9 uniform40" "16 8 1e9 sorted"; do
  RADSORT_LOG=1 timeout 600 python tools/sweep_bench.py case $cs 3 2>> $O/err.log >> $O/dup_rule.jsonl
done
grep "duplicate estimate" $O/err.log | sort | uniq -c
for c in c4 c3 c5 c2 c1 kmc; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2>> $O/err2.log; echo "bench $c rc=$?"
done
cut -c1-200 $O/dup_rule.jsonl
for f in $O/bench_*.json; do echo "$f: $(python -c "import json;d=json.load(open('$f'));print(d.get('ms_per_step'), d.get('gpu_launches'))")"; done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log | cut -c1-300
