#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gpu_tests.txt
timeout 120 python tools/tc2_trace.py dualpol > gpurun_out/r2_k1_trace.txt 2>&1; tail -12 gpurun_out/r2_k1_trace.txt
