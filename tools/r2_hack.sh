#!/bin/bash
cd "$(dirname "$0")/.."
for hack in 0 1; do
  if [ $hack = 1 ]; then export HOLO_TAILR_HACK=1; fi
  timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/r2_hack$hack.csv \
    python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
  echo "hack=$hack"; grep -E "tail42r" gpurun_out/r2_hack$hack.csv | awk -F'","' '{print substr($5,1,40), $NF}' | tail -3
done
