for n in 1 2 4 8; do echo "chunks=$n"; HOLO_PIPE_CHUNKS=$n timeout 200 python tools/e2e_probe.py 2>&1 | head -1; done
python - <<'PY'
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import bench
from paper_2204_02348_b200 import api
from paper_2204_02348_b200.synth import FrameSpec, make_frames
fspec, cfg = bench.config_for("dualpol")
frames = torch.from_numpy(make_frames(FrameSpec(**fspec))).pin_memory()
h = api.create_handle(); eng = api.engine(h)
for k, v in cfg.items(): setattr(eng.config, k, v)
api.set_batch(h, cfg["batchCount"], frames)
eng._PIPE_CHUNKS = 10**9   # disable pipelining
for _ in range(3): api.process_batch(h)
ts = []
for _ in range(20):
    t0 = time.perf_counter(); api.process_batch(h); ts.append(time.perf_counter() - t0)
print("unpipelined median ms", np.median(ts) * 1e3)
PY
