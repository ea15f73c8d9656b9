"""H2D bandwidth probe: contiguous pinned copies vs the window-only 3-D copies of hpg_upload_windows."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2204_02348_b200 import api, native  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


dev = torch.device("cuda", 0)
for mb in (16, 131, 512):
    n = mb * 1024 * 1024 // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device=dev)
    t = timed(lambda: d.copy_(h, non_blocking=True))
    print(f"contiguous pinned H2D {mb} MB: {n * 4 / t / 1e9:.1f} GB/s")
    t = timed(lambda: h.copy_(d, non_blocking=True))
    print(f"contiguous pinned D2H {mb} MB: {n * 4 / t / 1e9:.1f} GB/s")

# window-only upload as api.process_batch does it (dual-pol, 1000 frames 640x256)
F, W, H = 1000, 640, 256
host = torch.empty((F, H, W), dtype=torch.float32).pin_memory()
host.numpy()[:] = np.random.default_rng(0).random((F, H, W), dtype=np.float32)
h = api.create_handle()
eng = api.engine(h)
cfg = eng.config
cfg.frameWidth, cfg.frameHeight, cfg.polCount, cfg.batchCount = W, H, 2, F
cfg.beamCentre = [[-160 * 20e-6, 160 * 20e-6], [0.0, 0.0]]
api.set_batch(h, F, host)
eng.run_pipeline(0)
plan0 = eng._native_plan(eng._plan_key(0, (1.0, 1.0)))
packed = torch.empty((F, 128, 256), dtype=torch.float32, device=dev)
lib = native.lib()
t = timed(lambda: lib.hpg_upload_windows(plan0.handle, ctypes.c_void_p(host.data_ptr()), 0, F,
                                         ctypes.c_void_p(packed.data_ptr()), native.stream_handle()))
print(f"window-only 3-D upload: {packed.numel() * 4 / t / 1e9:.1f} GB/s ({t * 1e3:.2f} ms)")
# two pols on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def two_streams():
    ev = torch.cuda.Event()
    ev.record()
    for k, s in enumerate((s1, s2)):
        s.wait_event(ev)
        lib.hpg_upload_windows(plan0.handle, ctypes.c_void_p(host.data_ptr() + k * (F // 2) * W * H * 4), 0, F // 2,
                               ctypes.c_void_p(packed.data_ptr() + k * (F // 2) * 128 * 256 * 4), ctypes.c_void_p(s.cuda_stream))
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t = timed(two_streams)
print(f"window-only 3-D upload, 2 streams: {packed.numel() * 4 / t / 1e9:.1f} GB/s ({t * 1e3:.2f} ms)")
t = timed(lambda: api.process_batch(h))
print(f"api.process_batch e2e: {F / t:.0f} frames/s ({t * 1e3:.2f} ms)")
