"""Per-evaluation host/GPU breakdown of AutoAlign (run_pipeline vs calc_metrics)."""
import copy, os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_02348_b200 import align
from paper_2204_02348_b200.engine import Engine
from paper_2204_02348_b200.synth import FrameSpec, make_frames
from tests.golden.autoalign_case import FRAMES, start_config
frames = make_frames(FrameSpec(**FRAMES))
acc = {"run": [], "metrics": [], "sync_run": []}
orig = align._evaluate
def timed_eval(eng, from_stage):
    t0 = time.perf_counter()
    eng.run_pipeline(from_stage)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    eng.calc_metrics()
    t3 = time.perf_counter()
    acc["run"].append(t1 - t0); acc["sync_run"].append(t2 - t1); acc["metrics"].append(t3 - t2)
    g = eng.config.autoAlignGoalIdx
    return eng.metric(g) * align._direction(g)
align._evaluate = timed_eval
def run():
    eng = Engine()
    for k, v in start_config().items():
        setattr(eng.config, k, copy.deepcopy(v))
    eng.config.autoAlignTol = 1e-4
    eng.source.set_float32(frames)
    t0 = time.perf_counter()
    align.auto_align(eng)
    return time.perf_counter() - t0
run()
for k in acc: acc[k].clear()
T = run()
n = len(acc["run"])
print(f"total {T*1e3:.1f} ms, {n} evals")
for k, v in acc.items():
    print(f"  {k:10s} mean {np.mean(v)*1e6:7.0f} us  sum {np.sum(v)*1e3:7.1f} ms")
