"""A/B of pipelined vs unpipelined api.process_batch in one process (same pinned buffer)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_02348_b200 import api  # noqa: E402
from paper_2204_02348_b200.synth import FrameSpec, make_frames  # noqa: E402

fspec, cfg = bench.config_for("dualpol")
frames = torch.from_numpy(make_frames(FrameSpec(**fspec))).pin_memory()
h = api.create_handle()
eng = api.engine(h)
for k, v in cfg.items():
    setattr(eng.config, k, v)
api.set_batch(h, cfg["batchCount"], frames)
res = {}
for rnd in range(10):
    for n in (10 ** 9, 2, 4):
        eng._PIPE_CHUNKS = n
        for _ in range(2):
            api.process_batch(h)
        ts = []
        for _ in range(15):
            t0 = time.perf_counter()
            api.process_batch(h)
            ts.append(time.perf_counter() - t0)
        res.setdefault(n, []).append(np.median(ts) * 1e3)
for n, v in res.items():
    print("chunks", "off" if n > 100 else n, "median %.3f" % np.median(v), " ".join(f"{x:.2f}" for x in v))
# raw H2D of the same bytes for reference
d = torch.empty(1000 * 128 * 256, dtype=torch.float32, device="cuda")
hsrc = torch.empty(1000 * 128 * 256, dtype=torch.float32).pin_memory()
for _ in range(3):
    d.copy_(hsrc, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    d.copy_(hsrc, non_blocking=True)
torch.cuda.synchronize()
print("contiguous 131 MB H2D ms", (time.perf_counter() - t0) / 10 * 1e3)
