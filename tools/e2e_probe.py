"""Where the time of api.process_batch goes (host overhead vs copies vs kernel)."""
import cProfile
import pstats
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
for _ in range(3):
    api.process_batch(h)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    api.process_batch(h)
    ts.append(time.perf_counter() - t0)
print("process_batch wall ms: median %.3f min %.3f" % (np.median(ts) * 1e3, np.min(ts) * 1e3))
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    api.process_batch(h)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
