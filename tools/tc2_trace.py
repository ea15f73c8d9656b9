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
# P (producers): 0 window start, 1 half 0 landed, 2 half 1 landed, 3 stfree[K0] passed, 4 K half 0 staged,
#   5 stfree[K1] passed, 6 K half 1 staged, 7 fac / meta published
# M: 0 K half 0 staged seen, 1 row GEMM issued, 4/5 S2h0 ready/issued, 6/7 S2h1 ready/issued
# C: 0 D1 ready (meta + d1full), 1 D1 converted (sub), 5 D2 ready, 6 W stored
n = 14
for k in range(n):
    print(f"k={k:2d} P " + " ".join(f"{v:7.0f}" for v in P[k]))
    print(f"     M " + " ".join(f"{v:7.0f}" if v > -1e9 else "      -" for v in M[k]))
    print(f"     C " + " ".join(f"{v:7.0f}" if v > -1e9 else "      -" for v in C[k]))
a, b = 3, n - 1
d = lambda X, i, j: (X[a:b, j] - X[a:b, i]).mean()
print("period (row GEMM issued)", np.diff(M[a:b, 1]).mean())
print("P: land wait h0", d(P, 0, 1), "read+max h0 / land h1", d(P, 1, 2), "read+max h1 / stfree K0", d(P, 2, 3),
      "write K0", d(P, 3, 4), "stfree K1 wait", d(P, 4, 5), "write K1", d(P, 5, 6), "fac", d(P, 6, 7))
print("M: row GEMM (staged K0 -> issued)", d(M, 0, 1), "S2h0 issue", d(M, 4, 5), "S2h1 issue", d(M, 6, 7))
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
