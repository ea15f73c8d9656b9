"""CUDA activity timeline of one api.process_batch (torch.profiler): copies, kernels, gaps."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

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
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        api.process_batch(h)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{e.time_range.start - t0:9.1f} us  dur {e.time_range.elapsed_us():8.1f}  {e.name[:70]}")
cpu = [e for e in prof.events() if e.name.endswith("process_batch") or "cudaMemcpy" in e.name]
