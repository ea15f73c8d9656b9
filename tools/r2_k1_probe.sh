#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tc2 or two_kernel" > gpurun_out/r2_k1_tests.txt 2>&1; echo rc=$? >> gpurun_out/r2_k1_tests.txt
tail -3 gpurun_out/r2_k1_tests.txt
timeout 120 python tools/tc2_trace.py dualpol > gpurun_out/r2_k1_trace.txt 2>&1; tail -12 gpurun_out/r2_k1_trace.txt
for t in 1 0; do
  HOLO_TAIL=$t timeout 120 python bench.py --tc2 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2_k1_bench_tail$t.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/r2_k1_bench_tail$t.json').read().strip().splitlines()[-1]); print('tail$t', d['value'], d['ms_per_step'])" 2>&1 | tail -1
done
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 6 --csv --log-file gpurun_out/r2_k1_launches.csv \
  python bench.py --tc2 --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
grep -E "tail42|field128|fourier128" gpurun_out/r2_k1_launches.csv | awk -F'","' '{print $5, $NF}' | cut -c1-40,200- | head -6
