#!/bin/bash
# round-2 final measurements: GPU tests, every bench line, launch lists, traffic captures
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/r2f_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -3 $O/r2f_gpu_tests.txt
timeout 400 python bench.py --steps 20 --warmup 5 > $O/r2f_bench_dualpol.json 2> $O/r2f_bench_dualpol.err; echo "dualpol rc=$?"
timeout 200 python bench.py --simt --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > $O/r2f_bench_dualpol_simt.json 2>&1
timeout 300 python bench.py --config largeframe --no-cpu-baseline --steps 10 --warmup 3 > $O/r2f_bench_largeframe.json 2>&1; echo "lf rc=$?"
timeout 300 python bench.py --config pr1 --no-cpu-baseline --steps 20 --warmup 5 > $O/r2f_bench_pr1.json 2>&1; echo "pr1 rc=$?"
timeout 300 python bench.py --config autoalign --no-cpu-baseline --steps 10 --warmup 3 > $O/r2f_bench_autoalign.json 2>&1; echo "aa rc=$?"
timeout 600 python bench.py --config largebasis --batch 65536 --tile 1024 --steps 5 --warmup 3 --no-cpu-baseline > $O/r2f_bench_lb65536.json 2> $O/r2f_bench_lb65536.err; echo "lb rc=$?"
timeout 600 python bench.py --config largebasis --batch 65536 --tile 1024 --split --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/r2f_bench_lb_split.json 2> $O/r2f_bench_lb_split.err; echo "split rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/r2f_bench_reference.json 2> $O/r2f_bench_reference.err; echo "ref rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/r2f_launches_dualpol.csv \
  python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 120 --csv --log-file $O/r2f_traffic_largeframe.csv \
  python bench.py --config largeframe --no-e2e --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 40 --csv --log-file $O/r2f_traffic_dualpol.csv \
  python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 2 > /dev/null 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 40 --csv --log-file $O/r2f_traffic_lb65536.csv \
  python bench.py --config largebasis --batch 65536 --tile 1024 --no-e2e --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2>&1
for f in dualpol dualpol_simt largeframe pr1 autoalign lb65536 lb_split reference; do
  python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r2f_bench_{f}.json").read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    print(f, round(d["value"]), d.get("ms_per_step"), round(r.get("frac", 0), 4), r.get("kernel"), "e2e", (d.get("e2e") or {}).get("value"), d.get("cpu_baseline", {}).get("kind"))
except Exception as e:
    print(f, "ERR", e)
PY
done
