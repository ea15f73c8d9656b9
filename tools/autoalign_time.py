"""Time-to-converge of AutoAlign (BASELINE config 4 starting point) on the GPU engine, per-evaluation cost."""
import copy
import os
import sys
import time
import cProfile
import pstats

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_02348_b200 import align  # noqa: E402
from paper_2204_02348_b200.engine import Engine  # noqa: E402
from paper_2204_02348_b200.synth import FrameSpec, make_frames  # noqa: E402
from tests.golden.autoalign_case import FRAMES, start_config  # noqa: E402

frames = make_frames(FrameSpec(**FRAMES))


def run(tol):
    eng = Engine()
    for k, v in start_config().items():
        setattr(eng.config, k, copy.deepcopy(v))
    eng.config.autoAlignTol = tol
    eng.source.set_float32(frames)
    eng.eval_log = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    goal = align.auto_align(eng)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, goal, len(eng.eval_log)


run(1e-4)   # warm-up (plans, JIT of nothing, allocator)
for tol in (0.0, 1e-4):
    ts = [run(tol) for _ in range(3)]
    t, goal, n = min(ts)
    print(f"tol {tol:g}: time-to-converge {t * 1e3:.1f} ms, {n} evaluations, {t / n * 1e6:.0f} us/eval, goal {goal:.4f} dB")
pr = cProfile.Profile()
pr.enable()
run(1e-4)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
