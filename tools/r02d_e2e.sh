#!/bin/bash
# new streaming e2e + c1 after the sync removal (repo root on the GPU box)
O=gpurun_out/r02d_e2e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sort.py -x -q -k "host_stream or sort_host or smoke or layouts" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
for c in c1 c2; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"; done
for f in $O/bench_*.json; do echo "$f: $(python -c "import json;d=json.load(open('$f'));print(d.get('ms_per_step'), d.get('value'), d.get('e2e'))" 2>&1 | tail -1)"; done
