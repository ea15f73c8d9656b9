#!/bin/bash
cd "$(dirname "$0")/.."
for pr in 0 2 3; do
  HOLO_TMA_PROMO=$pr timeout 200 python bench.py --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r2_promo$pr.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/r2_promo$pr.json').read().strip().splitlines()[-1]); print('promo $pr', round(d['value']), d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1
done
