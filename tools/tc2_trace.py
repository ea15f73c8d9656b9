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
buf = (ctypes.c_longlong * (3 * 64 * 8))()
lib = native.lib()
lib.hpg_debug_trace.argtypes = [ctypes.c_void_p]
assert lib.hpg_debug_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(3, 64, 8).astype(np.float64)
t0 = t[0, 0, 0]
P = t[0] - t0
C = t[1] - t0
M = t[2] - t0
# P (producers) per half h: 4h+0 start, 4h+1 stfree passed, 4h+2 landed, 4h+3 converted (after barrier)
# M (MMA): 0/1 S1h0 ready/issued, 2/3 S1h1, 4/5 S2h0, 6/7 S2h1
# C (consumers): 0/1 D1h0 ready/drained, 2/3 D1h1 ready/drained, 4 fac ready, 5 D2 ready, 6 W stored
n = 14
np.set_printoptions(linewidth=200)
for k in range(n):
    print(f"k={k:2d} P " + " ".join(f"{v:7.0f}" for v in P[k]))
    print(f"     M " + " ".join(f"{v:7.0f}" for v in M[k]))
    print(f"     C " + " ".join(f"{v:7.0f}" for v in C[k]))
a, b = 3, n - 1
d = lambda X, i, j: (X[a:b, j] - X[a:b, i]).mean()
print("period", np.diff(M[a:b, 3]).mean())
print("P h0: stfree wait", d(P, 0, 1), "land wait", d(P, 1, 2), "convert", d(P, 2, 3), "| h1: gap", d(P, 3, 4),
      "stfree wait", d(P, 4, 5), "land wait", d(P, 5, 6), "convert", d(P, 6, 7))
print("M: S1h0 issue", d(M, 0, 1), "S1h1 issue", d(M, 2, 3), "S2h0 issue", d(M, 4, 5), "S2h1 issue", d(M, 6, 7))
print("C: D1h0 drain", d(C, 0, 1), "D1h1 drain", d(C, 2, 3), "D2 drain", d(C, 5, 6))
