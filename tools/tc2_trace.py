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
buf = (ctypes.c_longlong * (4 * 64 * 8))()
lib = native.lib()
lib.hpg_debug_trace.argtypes = [ctypes.c_void_p]
assert lib.hpg_debug_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(4, 64, 8).astype(np.float64)
t0 = t[0, 0, 0]
P = t[0] - t0
C = t[1] - t0
M = t[2] - t0
D = t[3] - t0
# P (producers) per half h: 4h+0 start, 4h+1 stfree passed, 4h+2 landed, 4h+3 converted (after barrier)
# M: 0 S1 ready, 1 S1 issued, 2 fac/meta arrived (producer), 4/5 S2h0 ready/issued, 6/7 S2h1 ready/issued
# C: 0 D1 ready (meta + d1full), 1 D1 converted (sub), 5 D2 ready, 6 planes stored
n = 14
for k in range(n):
    print(f"k={k:2d} P " + " ".join(f"{v:7.0f}" for v in P[k]))
    print(f"     M " + " ".join(f"{v:7.0f}" for v in M[k]))
    print(f"     C " + " ".join(f"{v:7.0f}" for v in C[k]))
a, b = 3, n - 1
d = lambda X, i, j: (X[a:b, j] - X[a:b, i]).mean()
print("period (S1 issue)", np.diff(M[a:b, 1]).mean())
print("P h0: stfree wait", d(P, 0, 1), "land wait", d(P, 1, 2), "convert", d(P, 2, 3), "| h1: stfree", d(P, 4, 5),
      "land", d(P, 5, 6), "convert", d(P, 6, 7))
print("M: S1 issue", d(M, 0, 1), "S2h0 issue", d(M, 4, 5), "S2h1 issue", d(M, 6, 7))
print("C: D1 convert", d(C, 0, 1), "D2 drain", d(C, 5, 6))
sp = (ctypes.c_longlong * (160 * 4))()
lib.hpg_debug_span.argtypes = [ctypes.c_void_p]
assert lib.hpg_debug_span(sp) == 0
sp = np.frombuffer(sp, dtype=np.int64).reshape(160, 4).astype(np.float64)
g = sp[:148]
t0 = g[:, 0].min()
print("CTA start (us) min/med/max", (g[:, 0] - t0).min() / 1e3, np.median(g[:, 0] - t0) / 1e3, (g[:, 0] - t0).max() / 1e3)
print("CTA end   (us) min/med/max", (g[:, 1] - t0).min() / 1e3, np.median(g[:, 1] - t0) / 1e3, (g[:, 1] - t0).max() / 1e3)
cyc = g[:, 3] - g[:, 2]
ns = g[:, 1] - g[:, 0]
print("CTA duration cycles min/med/max", cyc.min(), np.median(cyc), cyc.max(), " -> GHz", np.median(cyc / ns))
c0 = sp[0, 2]
last = max(C[k, 6] for k in range(64) if C[k, 6] > 0) + t0_cycles if False else None
raw = np.frombuffer(buf, dtype=np.int64).reshape(4, 64, 8).astype(np.float64)
print("CTA0: setup (entry -> first producer mark) cycles", raw[0, 0, 0] - c0,
      " last W -> exit", sp[0, 3] - raw[1, :, 6].max())
