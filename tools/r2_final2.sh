#!/bin/bash
# final state: GPU tests, dual-pol bench (+ SIMT comparison), launch list, ncu --set full of both kernels, K1 trace
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/r2f_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -3 $O/r2f_gpu_tests.txt
timeout 400 python bench.py --steps 20 --warmup 5 > $O/r2f_bench_dualpol.json 2> $O/r2f_bench_dualpol.err; echo "dualpol rc=$?"
timeout 200 python bench.py --simt --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > $O/r2f_bench_dualpol_simt.json 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/r2f_bench_reference.json 2> $O/r2f_bench_reference.err; echo "ref rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/r2f_launches_dualpol.csv \
  python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 40 --csv --log-file $O/r2f_traffic_dualpol.csv \
  python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 2 > /dev/null 2>&1
bash tools/r2_ncu_kernel.sh tail42p r2f_tailp_ncu
bash tools/r2_ncu_kernel.sh fourier128_tc2 r2f_k1_ncu
timeout 120 python tools/tc2_trace.py dualpol > $O/r2f_k1_trace.txt 2>&1
python - <<'PY'
import json
for f in ("dualpol", "dualpol_simt", "reference"):
    d = json.loads(open(f"gpurun_out/r2f_bench_{f}.json").read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    print(f, round(d["value"]), d.get("ms_per_step"), round(r.get("frac", 0), 4), r.get("kernel"), "e2e", (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("kind"), d.get("gpu_launches"))
PY
grep -E "holo" $O/r2f_launches_dualpol.csv | awk -F'","' '{print substr($5,1,40), $NF}' | tail -4
