#!/bin/bash
# round-2 re-entry baseline: GPU tests, default bench, TC2 bench, launch lists
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gpu_tests.txt
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_dualpol.json 2> gpurun_out/r2_bench_dualpol.err; echo "dualpol rc=$?"
for t in 1 0; do
  HOLO_TAIL=$t timeout 120 python bench.py --tc2 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2_tc2_bench_tail$t.json 2>&1; echo "tc2 tail$t rc=$?"
done
timeout 200 python bench.py --config largeframe --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2_bench_largeframe.json 2>&1; echo "lf rc=$?"
timeout 200 python bench.py --config pr1 --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2_bench_pr1.json 2>&1; echo "pr1 rc=$?"
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_launches_dualpol.csv \
  python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_launches_tc2.csv \
  python bench.py --tc2 --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
for f in gpurun_out/r2_bench_dualpol.json gpurun_out/r2_tc2_bench_tail1.json gpurun_out/r2_tc2_bench_tail0.json gpurun_out/r2_bench_largeframe.json gpurun_out/r2_bench_pr1.json; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['ms_per_step'], d['roofline']['frac'], d.get('e2e'))" 2>&1 | tail -1
done
grep -E "kernel" gpurun_out/r2_launches_tc2.csv | awk -F'","' '{print $5, $NF}' | cut -c1-50,180- | tail -8
