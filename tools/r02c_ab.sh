set -u
O=gpurun_out/s3; mkdir -p $O
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_sort.py -k "write_out or key_index or wide" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for lay in "24 8 9e8" "24 16 9e8" "40 16 5e8" "8 8 1e9"; do
  for v in 2 0; do
    echo "$lay tma=$v $(RADSORT_SCATTER_TMA=$v timeout 300 python tools/layout_bench.py $lay uniform 3 2>&1 | tail -1)"
  done
done
CFGS=c5 bash tools/r02_prof.sh
