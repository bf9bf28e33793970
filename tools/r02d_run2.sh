#!/bin/bash
# candidate-histogram warp aggregation: full GPU suite, c3/c5/c4 bench, c4 + c3 launch lists (repo root on the GPU box)
O=gpurun_out/r02d_run2; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log | cut -c1-300
for c in c3 c5 c4; do RADSORT_LOG=1 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"; done
for c in c4 c3; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file $O/${c}_launches.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch_$c.log 2>&1; echo "launches $c rc=$?"
done
for f in $O/bench_*.json; do echo "$f: $(python -c "import json;d=json.load(open('$f'));print(d.get('ms_per_step'), d.get('value'), {k:round(v,2) for k,v in d.get('kernel_ms_per_step',{}).items() if v>0.05})" 2>&1 | tail -1)"; done
grep "level . ms" $O/bench_c3.err | tail -6
