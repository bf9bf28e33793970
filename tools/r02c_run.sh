#!/bin/bash
# round-2 (third part) GPU session: local-sort tests, then the phase profile of c4 / c5
set -u
O=gpurun_out/r02c; mkdir -p $O
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_sort.py ${PYK-} > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
CFGS="c4 c5" bash tools/r02_prof.sh
