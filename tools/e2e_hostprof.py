"""cProfile of api.process_batch on pinned dual-pol frames (host-side cost between the GPU copies)."""
import cProfile
import pstats
import sys

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
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    api.process_batch(h)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(28)
