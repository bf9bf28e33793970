#!/bin/bash
# Level 0 in the wide rule's window for R < 24 (mid-size sorts): old rule (RADSORT_WIDE_MIN_R=24:
# no estimate, two 8-bit passes) vs the default (estimate + sync before level 0, one 10-bit pass).
set -u
O=${OUT-gpurun_out/r02h_mid}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sort.py -m gpu -x -q -k "wide" > $O/pytest_wide.log 2>&1; echo "pytest wide rc=$?"; tail -2 $O/pytest_wide.log | cut -c1-300
for cs in "16 8 3e6 uniform" "16 8 5e6 uniform" "16 8 7.5e6 uniform" "16 16 5e6 uniform" "8 8 6e6 uniform" "8 8 10e6 uniform" "8 8 15e6 uniform" "16 8 5e6 zipf" "8 8 10e6 zipf" "8 8 1e6 uniform" "16 8 2e6 uniform"; do
  for mr in 24 default; do
    if [ $mr = default ]; then unset RADSORT_WIDE_MIN_R; else export RADSORT_WIDE_MIN_R=$mr; fi
    timeout 300 python tools/sweep_bench.py case $cs 20 2>> $O/err.log | sed "s/^{/{\"rule\": \"$mr\", /" >> $O/mid_rule.jsonl
  done
done
unset RADSORT_WIDE_MIN_R
python -c "
import json
for l in open('$O/mid_rule.jsonl'):
    d=json.loads(l); print(d['rule'], (d['R'],d['K']), d['n'], d['dist'], d['ms_median'], d['ms_min'], 'sc', d['scatter_passes'], d['verified'])"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log | cut -c1-300
