#!/bin/bash
# ncu --set full of one kernel (regex $1) of the TC2 bench; report in gpurun_out/$2.ncu-rep + text summary
cd "$(dirname "$0")/.."
K=$1; OUT=$2; shift 2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 -f -o gpurun_out/$OUT \
  python bench.py "$@" --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/$OUT.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/$OUT.ncu-rep --page details > gpurun_out/$OUT.txt 2>&1
grep -E "Duration|Executed Ipc|Issue Slots Busy|Registers Per|Achieved Occupancy|Theoretical Occ|DRAM Throughput|L2 Cache Throughput|Warp Cycles Per Issued|One or More Eligible|No Eligible" gpurun_out/$OUT.txt | head -20
