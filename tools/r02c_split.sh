#!/bin/bash
set -u
VARIANT=base CFGS="c3 kmc c5" bash tools/r02_abv.sh
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_sort.py -k "dominant or distributions or write_out or other_tile" 2>&1 | tail -2
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_multi.py tests/test_gpu_fuzz.py 2>&1 | tail -2
