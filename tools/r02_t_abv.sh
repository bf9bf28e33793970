#!/bin/bash
# gpu tests (subset or all) then the A/B against scratch/libradsort_$VARIANT.so
set -u
O=gpurun_out/r02; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q ${PYK-} > $O/pytest_t.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_t.log | cut -c1-400
bash tools/r02_abv.sh
