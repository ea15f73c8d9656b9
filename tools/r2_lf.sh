#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_full_size_gpu.py tests/test_gpu_parity.py -q -x -k "largeframe or large_window or lw or launch_count or 256" 2>&1 | tail -3
timeout 300 python bench.py --config largeframe --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2_lf.json 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/r2_lf.json').read().strip().splitlines()[-1]); print('largeframe', round(d['value']), round(d['ms_per_step']*1e3,1), 'us', d['roofline']['frac'])" 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 120 --csv --log-file gpurun_out/r2_traffic_lf.csv \
  python bench.py --config largeframe --no-e2e --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(l for l in open('gpurun_out/r2_traffic_lf.csv') if l.startswith('"'))]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
agg={}
for r in rows[1:]:
    if 'lw_' in r[ki]:
        k=r[ki].split('(')[0][:40]
        agg.setdefault(k,{}).setdefault(r[mi],[]).append(float(r[vi].replace(',','')))
for k,v in agg.items(): print('  ',k,{m:(len(x), round(sum(x)/len(x),1)) for m,x in v.items()})
PY
