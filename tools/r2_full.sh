#!/bin/bash
# full GPU test suite + default bench + SIMT comparison + launch list
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2_gpu_tests.txt
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_dualpol.json 2> gpurun_out/r2_bench_dualpol.err; echo "dualpol rc=$?"
timeout 200 python bench.py --simt --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r2_bench_dualpol_simt.json 2>&1; echo "simt rc=$?"
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_launches_dualpol.csv \
  python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
for f in gpurun_out/r2_bench_dualpol.json gpurun_out/r2_bench_dualpol_simt.json; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'], d.get('gpu_launches'), (d.get('e2e') or {}).get('value'))" 2>&1 | tail -1
done
grep -E "holo" gpurun_out/r2_launches_dualpol.csv | awk -F'","' '{print substr($5,1,40), $NF}' | tail -4
