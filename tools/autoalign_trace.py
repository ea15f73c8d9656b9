"""Diagnostic: run AutoAlign on the GPU engine and compare its evaluation
trajectory with the reference's recorded one (tests/golden/autoalign_*.npz)."""
import copy
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_02348_b200 import align  # noqa: E402
from paper_2204_02348_b200.engine import Engine  # noqa: E402
from paper_2204_02348_b200.synth import FrameSpec, make_frames  # noqa: E402
from tests.golden.autoalign_case import FRAMES, start_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "autoalign_tol1e-4"
g = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
eng = Engine()
for k, v in start_config().items():
    setattr(eng.config, k, copy.deepcopy(v))
eng.config.autoAlignTol = 1e-4 if "1e-4" in name else 0.0
eng.source.set_float32(make_frames(FrameSpec(**FRAMES)))
eng.eval_log = []
goal = align.auto_align(eng)
print("goal gpu", goal, "ref", float(g["goal"]), "evals", len(eng.eval_log), len(g["stages"]))
ref_p, ref_v, ref_s = g["params"], g["values"], g["stages"]
for i, (st, v, prm) in enumerate(eng.eval_log):
    if i >= len(ref_p):
        break
    dp = np.abs(np.array(prm) - ref_p[i]) / np.maximum(np.abs(ref_p[i]), 1e-12)
    if st != ref_s[i] or dp.max() > 1e-6 or abs(v - ref_v[i]) > 1e-4:
        print(f"first divergence at eval {i}: stage {st} vs {ref_s[i]}")
        for j in range(max(0, i - 3), min(i + 3, len(ref_p))):
            print(j, eng.eval_log[j][0], eng.eval_log[j][1], ref_s[j], ref_v[j])
            print("   gpu", np.array(eng.eval_log[j][2]))
            print("   ref", ref_p[j])
        break
else:
    print("trajectories agree")
