#!/bin/bash
# TC2 path with the register-resident tail (default), the warp-pair tail (HOLO_TAIL=2) and the CTA-wide tail (0)
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tc2 or two_kernel" 2>&1 | tail -3
timeout 200 python -m pytest tests/test_memory_guards_gpu.py -q -x 2>&1 | tail -2
for t in ${TAILS:-1 2 0}; do
  HOLO_TAIL=$t timeout 120 python bench.py --tc2 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2_tc2_bench_tail$t.json 2>&1; echo "tc2 tail$t rc=$?"
  python -c "import json,sys; d=json.loads(open('gpurun_out/r2_tc2_bench_tail$t.json').read().strip().splitlines()[-1]); print('tail$t', round(d['value']), d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1
done
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2_launches_tc2.csv \
  python bench.py --tc2 --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
grep -E "holo" gpurun_out/r2_launches_tc2.csv | awk -F'","' '{print substr($5,1,40), $NF}' | tail -6
timeout 120 python tools/tc2_trace.py dualpol > gpurun_out/r2_k1_trace.txt 2>&1; tail -9 gpurun_out/r2_k1_trace.txt
