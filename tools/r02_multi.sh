#!/bin/bash
# multi-GPU path tests (loopback fused / send-recv, NCCL 1 rank) + a timing of the fused exchange on one GPU
set -u
O=gpurun_out/r02; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > $O/pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -5 $O/pytest_multi.log | cut -c1-400
if [ -n "${MORE-}" ]; then timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu2.log 2>&1; echo "pytest all rc=$?"; tail -3 $O/pytest_gpu2.log | cut -c1-300; fi
