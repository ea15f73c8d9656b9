#!/bin/bash
# quick multi-window K1 check with short timeouts (a hang is killed within 30 s)
cd "$(dirname "$0")/.."
for b in 300 1000; do
  timeout 45 python bench.py --tc2 --batch $b --no-e2e --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/r2_k1q_$b.json 2>&1
  echo "batch $b rc=$?"; tail -c 300 gpurun_out/r2_k1q_$b.json | head -c 300; echo
done
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "two_kernel or tc2" 2>&1 | tail -2
timeout 60 python tools/tc2_trace.py dualpol > gpurun_out/r2_k1_trace.txt 2>&1; tail -9 gpurun_out/r2_k1_trace.txt
