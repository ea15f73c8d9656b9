#!/bin/bash
# parity (whole GPU parity file) + default dual-pol bench + launch list
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_memory_guards_gpu.py -q -x 2>&1 | tail -2
timeout 200 python bench.py --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r2_bench_dualpol_q.json 2>&1; echo "dp rc=$?"
python -c "import json,sys; d=json.loads(open('gpurun_out/r2_bench_dualpol_q.json').read().strip().splitlines()[-1]); print('dualpol', round(d['value']), d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'])" 2>&1 | tail -1
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/r2_launches_q.csv \
  python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
grep -E "holo" gpurun_out/r2_launches_q.csv | awk -F'","' '{print substr($5,1,40), $NF}' | tail -4
