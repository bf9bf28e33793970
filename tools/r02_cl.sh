#!/bin/bash
# the cluster local sort: tests that cover it + c4 timing (+ optional prof build run)
set -u
O=gpurun_out/r02; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "cluster or c4 or fuzz or multi or level0 or outlier" > $O/pytest_cl.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_cl.log | cut -c1-300
RADSORT_LOG=1 timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/cl_c4.json 2> $O/cl_c4.err
echo "c4 rc=$?"; python -c "import json;d=json.load(open('$O/cl_c4.json'));print(d['ms_per_step'], {k:round(v,2) for k,v in d['kernel_ms_per_step'].items() if v>0.05})"
