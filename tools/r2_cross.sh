#!/bin/bash
# crossover of the two-kernel path against the fused SIMT kernel by batch size (dual-pol frames = 2 windows each)
cd "$(dirname "$0")/.."
for b in 150 222 300 444 600; do
  for mode in "--tc2" "--simt"; do
    timeout 120 python bench.py $mode --batch $b --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r2_cross.json 2>&1
    python -c "import json,sys; d=json.loads(open('gpurun_out/r2_cross.json').read().strip().splitlines()[-1]); print('batch $b $mode', round(d['value']), round(d['ms_per_step']*1e3,1), 'us')" 2>&1 | tail -1
  done
done
