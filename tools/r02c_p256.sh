#!/bin/bash
set -u
SETS="RADSORT_LOCAL_PIPE256=1|RADSORT_LOCAL_PIPE256=0" CFGS="c2 c3 kmc" STEPS=5 bash tools/r02c_envab.sh 2>&1 | grep -v "level [0-9]"
RADSORT_LOCAL_PIPE256=1 timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_sort.py -k "distributions or opt_in or small or capacity or size_classes or write_out" 2>&1 | tail -2
