"""Viewport renders (holopipe/viewport.py:61-115) of the 'pr1' golden case, every display mode, by the
REFERENCE itself.  Run in the build container: python tests/golden/make_viewport_golden.py"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from holopipe import api as R  # noqa: E402

from paper_2204_02348_b200.synth import FrameSpec, make_frames  # noqa: E402
from tests.golden.cases import CASES  # noqa: E402

case = CASES["pr1"]
frames = make_frames(FrameSpec(**case["frames"]))
h = R.create_handle()
eng = R.engine(h)
for k, v in case["config"].items():
    setattr(eng.config, k, v)
eng.config.threadCount = 1
R.set_batch(h, case["config"]["batchCount"], frames)
R.process_batch(h)
out = {}
for mode in range(1, 9):
    rgb, w, hh, title = R.get_viewport(h, mode, 0)
    out[f"mode{mode}"] = rgb
np.savez_compressed(os.path.join(HERE, "viewport_pr1.npz"), **out)
print({k: v.shape for k, v in out.items()})
