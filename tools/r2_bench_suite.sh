#!/bin/bash
# round-2 bench suite (1 GPU): default dual-pol with e2e variants, config 5 at 65,536 frames (tiled), split mode
cd "$(dirname "$0")/.."
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_suite_dualpol.json 2> gpurun_out/r2_suite_dualpol.err; echo "dualpol rc=$?"
timeout 600 python bench.py --config largebasis --batch 65536 --tile 1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_suite_lb65536.json 2> gpurun_out/r2_suite_lb65536.err; echo "lb65536 rc=$?"
timeout 600 python bench.py --config largebasis --batch 65536 --tile 1024 --split --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_suite_lb_split.json 2> gpurun_out/r2_suite_lb_split.err; echo "split rc=$?"
timeout 300 python -m pytest tests/test_autoalign_gpu.py tests/test_sharded_metrics_gpu.py tests/test_api_benchmark.py tests/test_gpu_parity.py -q -s -k "not fields_and_coefs" 2>&1 | grep -E "deviation|passed|failed" > gpurun_out/r2_suite_tests.txt
cat gpurun_out/r2_suite_tests.txt
for f in dualpol lb65536 lb_split; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r2_suite_{f}.json").read().strip().splitlines()[-1])
    ev = d.get("e2e_variants") or {}
    print(f, round(d["value"]), d["ms_per_step"], round(d["roofline"]["frac"], 4), d.get("scaling"),
          "e2e", None if d.get("e2e") is None else round(d["e2e"]["value"]),
          {k: (round(v["value"]) if isinstance(v, dict) else v) for k, v in ev.items()})
except Exception as e:
    print(f, "ERR", e, open(f"gpurun_out/r2_suite_{f}.err").read()[-600:])
PY
done
