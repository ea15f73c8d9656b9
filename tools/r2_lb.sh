#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 200 python bench.py --config largebasis --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2_bench_largebasis.json 2>&1; echo "lb rc=$?"
timeout 200 python bench.py --tc --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2_bench_tc.json 2>&1; echo "tc rc=$?"
timeout 200 python bench.py --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r2_bench_dualpol_q.json 2>&1; echo "dp rc=$?"
for f in largebasis tc dualpol_q; do python -c "import json,sys; d=json.loads(open('gpurun_out/r2_bench_$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'])" 2>&1 | tail -1; done
