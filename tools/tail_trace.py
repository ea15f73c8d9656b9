"""Phase timeline of two CTAs of the register-resident tail (build with -DHOLO_TAIL_TRACE)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2204_02348_b200 import api, native  # noqa: E402
from paper_2204_02348_b200.synth import FrameSpec, make_frames  # noqa: E402
import bench  # noqa: E402

fspec, cfg = bench.config_for("dualpol")
frames = make_frames(FrameSpec(**fspec))
h = api.create_handle()
eng = api.engine(h)
for k, v in cfg.items():
    setattr(eng.config, k, v)
api.set_batch(h, cfg["batchCount"], torch.from_numpy(frames).to("cuda:0"))
eng.run_pipeline(0)
L = eng.prepare_launch()
for _ in range(3):
    L.launch()
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 32)()
lib = native.lib()
lib.hpg_debug_tail_trace.argtypes = [ctypes.c_void_p]
assert lib.hpg_debug_tail_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(2, 16).astype(np.float64)
names = ["entry", "set-up done", "windows landed", "columns in registers", "IDFT y done", "-", "rows in registers",
         "IDFT x done", "removal + peak done", "peak barrier passed", "quantised + folded", "overlap x done",
         "U barrier passed", "overlap y done (thread 0)"]
for c in range(2):
    print("CTA", "0" if c == 0 else "grid/2")
    prev = t[c, 0]
    for i, n in enumerate(names):
        if n == "-" or t[c, i] == 0:
            continue
        print(f"  {n:32s} {t[c, i] - t[c, 0]:9.0f}  (+{t[c, i] - prev:7.0f})")
        prev = t[c, i]
