#!/bin/bash
cd "$(dirname "$0")/.."
for c in pr1 autoalign; do
  timeout 200 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r2_pr1_$c.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/r2_pr1_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value']), round(d['ms_per_step']*1e3,2), 'us')" 2>&1 | tail -1
  timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 40 --csv --log-file gpurun_out/r2_pr1_launch_$c.csv \
    python bench.py --config $c --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > /dev/null 2>&1
  grep -E "holo" gpurun_out/r2_pr1_launch_$c.csv | awk -F'","' '{print substr($5,1,50), $NF}' | tail -3
done
