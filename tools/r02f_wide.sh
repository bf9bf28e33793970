#!/bin/bash
# The default wide-level rule on R = 8 / 16 (RADSORT_WIDE_MIN_R=8) against R >= 24 only, on the
# sizes where it fires (8-bit children above the CTA-local capacity C, 10-bit ones below).
set -u
O=${OUT-gpurun_out/r02f_wide}; mkdir -p $O
for mr in 24 8; do
  for cs in "16 8 1e9 uniform" "16 16 1e9 uniform" "8 8 2e9 uniform" "16 8 2e9 uniform" "16 8 1e9 zipf" "8 8 2e9 zipf" "16 16 1e9 bytes" "16 16 413e6 kmer"; do
    RADSORT_WIDE_MIN_R=$mr timeout 600 python tools/sweep_bench.py case $cs 3 2>> $O/err.log | sed "s/^{/{\"wide_min_r\": $mr, /" >> $O/wide_rule.jsonl
  done
  for c in c3 c5 c2 kmc; do
    RADSORT_WIDE_MIN_R=$mr timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>> $O/err.log | sed "s/^{/{\"wide_min_r\": $mr, /" >> $O/wide_rule_cfg.jsonl
  done
done
cut -c1-200 $O/wide_rule.jsonl; python -c "
import json
for l in open('$O/wide_rule_cfg.jsonl'):
    d=json.loads(l); print(d['wide_min_r'], d['config']['workload'][:3], d['ms_per_step'])"
