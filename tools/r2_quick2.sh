#!/bin/bash
# like r2_quick.sh with short timeouts (a hang must not eat the GPU budget)
cd "$(dirname "$0")/.."
timeout 60 python -m pytest tests/test_gpu_parity.py -q -x -k "two_kernel_tensor" 2>&1 | tail -1
timeout 60 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2_bench_dualpol_q.json 2>&1; echo "dp rc=$?"
python -c "import json,sys; d=json.loads(open('gpurun_out/r2_bench_dualpol_q.json').read().strip().splitlines()[-1]); print('dualpol', round(d['value']), d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1
timeout 90 python -m pytest tests/test_gpu_parity.py tests/test_full_size_gpu.py -q -x -k "two_kernel or dualpol" 2>&1 | tail -1
timeout 60 python tools/tc2_trace.py dualpol > gpurun_out/r2_k1_trace.txt 2>&1; tail -8 gpurun_out/r2_k1_trace.txt | head -4
