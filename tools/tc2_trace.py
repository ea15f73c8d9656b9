"""Per-phase timeline of CTA 0 of the TC2 Fourier kernel (clock64 marks, HOLO trace)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2204_02348_b200 import api, native  # noqa: E402
from paper_2204_02348_b200.synth import FrameSpec, make_frames  # noqa: E402
import bench  # noqa: E402

fspec, cfg = bench.config_for(sys.argv[1] if len(sys.argv) > 1 else "dualpol")
frames = make_frames(FrameSpec(**fspec))
h = api.create_handle()
eng = api.engine(h)
eng.use_tc2 = True
for k, v in cfg.items():
    setattr(eng.config, k, v)
dev = torch.device("cuda", 0)
api.set_batch(h, cfg["batchCount"], torch.from_numpy(frames).to(dev))
eng.run_pipeline(0)
L = eng.prepare_launch()
for _ in range(3):
    L.launch()
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (2 * 64 * 8))()
lib = native.lib()
lib.hpg_debug_trace.argtypes = [ctypes.c_void_p]
assert lib.hpg_debug_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(2, 64, 8).astype(np.float64)
t0 = t[0, 0, 0]
P = t[0] - t0
C = t[1] - t0
names_p = ["start", "-", "converted", "fac ready", "mma1 issued", "mma2 issued"]
names_c = ["start", "mma1a done", "drained1", "mma2 done", "drained2", "W stored"]
for k in range(min(14, 64)):
    print(f"k={k:2d} P: " + " ".join(f"{n}={P[k, i]:8.0f}" for i, n in enumerate(names_p) if n != "-"))
    print(f"      C: " + " ".join(f"{n}={C[k, i]:8.0f}" for i, n in enumerate(names_c)))
n = 12
print("per-window period (consumer W stored):", np.diff(C[2:n, 5]).mean(), " producer:", np.diff(P[2:n, 0]).mean())
print("producer convert", (P[2:n, 2] - P[2:n, 0]).mean(), " fac", (P[2:n, 3] - P[2:n, 2]).mean())
print("  stfree0 wait", (P[2:n, 1] - P[2:n, 0]).mean(), " lfull0 wait", (P[2:n, 6] - P[2:n, 1]).mean(),
      " chunk0-1 convert + lfull2 wait", (P[2:n, 7] - P[2:n, 6]).mean(), " chunks 2-3", (P[2:n, 2] - P[2:n, 7]).mean())
print("mma1b issued - mma2 issued(prev)", (P[2:n, 4] - P[1:n - 1, 5]).mean(), " mma2 issued - mma1b issued",
      (P[2:n, 5] - P[2:n, 4]).mean())
print("consumer wait mma1a:", (C[2:n, 1] - C[2:n, 0]).mean(), " drain1 (both halves):", (C[2:n, 2] - C[2:n, 1]).mean(),
      " wait mma2:", (C[2:n, 3] - C[2:n, 2]).mean(), " drain2:", (C[2:n, 4] - C[2:n, 3]).mean(),
      " W:", (C[2:n, 5] - C[2:n, 4]).mean())
