#!/bin/bash
# round-2 probe: TC2 path with the warp-per-window tail vs the round-1 tail, and the launch split
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_parity.py -q -k "tc2 or two_kernel" > gpurun_out/r2_tc2_tests.txt 2>&1; echo rc=$? >> gpurun_out/r2_tc2_tests.txt
python -m pytest tests/test_autoalign_gpu.py -q -s -k end_to_end 2>&1 | grep -E "deviation|cycles|passed|failed" >> gpurun_out/r2_tc2_tests.txt
for t in 1 0; do
  HOLO_TAIL=$t python bench.py --tc2 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2_tc2_bench_tail$t.json 2>&1
done
python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2_fast_bench.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 6 --csv --log-file gpurun_out/r2_tc2_launches.csv \
  python bench.py --tc2 --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
tail -3 gpurun_out/r2_tc2_tests.txt
for f in gpurun_out/r2_tc2_bench_tail1.json gpurun_out/r2_tc2_bench_tail0.json gpurun_out/r2_fast_bench.json; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1
done
grep -E "tail42|field128|fourier128" gpurun_out/r2_tc2_launches.csv | awk -F'","' '{print $5, $NF}' | head -12
