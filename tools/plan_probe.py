"""Time native.Plan creation from Python vs inside hpg_plan_create."""
import copy, os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_02348_b200 import native
from paper_2204_02348_b200.engine import Engine
from tests.golden.autoalign_case import FRAMES, start_config
from paper_2204_02348_b200.synth import FrameSpec, make_frames
eng = Engine()
for k, v in start_config().items():
    setattr(eng.config, k, copy.deepcopy(v))
eng.source.set_float32(make_frames(FrameSpec(**FRAMES)))
eng.run_pipeline(0)
torch.cuda.synchronize()
key = eng._plan_key()
ts = []
for i in range(20):
    k2 = list(key)
    k2[-1] = (key[-1][0] * (1 + 1e-3 * (i + 1)), key[-1][1])
    t0 = time.perf_counter()
    eng._native_plan(tuple(k2))
    ts.append(time.perf_counter() - t0)
print("native plan (idle GPU) us:", np.round(np.array(ts) * 1e6).astype(int))
ts = []
for i in range(20):
    eng.run_pipeline(0)      # queue GPU work, then create a plan
    k2 = list(key)
    k2[-1] = (key[-1][0] * (1 + 1e-3 * (i + 30)), key[-1][1])
    t0 = time.perf_counter()
    eng._native_plan(tuple(k2))
    ts.append(time.perf_counter() - t0)
print("native plan (after queued work) us:", np.round(np.array(ts) * 1e6).astype(int))
