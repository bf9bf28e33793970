#!/bin/bash
# key + index sort (NEXT-1): tests + timings against the direct sort per layout
set -u
O=gpurun_out/r02; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sort.py -x -q -k "key_index" > $O/pytest_ki.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_ki.log | cut -c1-300
: > $O/ki_bench.jsonl
for spec in "32 8 1e9" "40 16 5e8" "32 16 1e9" "24 8 9e8"; do
  for ki in 0 1; do
    RADSORT_KEY_INDEX=$ki timeout 600 python tools/layout_bench.py $spec uniform 3 | sed "s/^{/{\"key_index\": $ki, /" >> $O/ki_bench.jsonl
  done
done
cat $O/ki_bench.jsonl
