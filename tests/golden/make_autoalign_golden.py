"""AutoAlign fixtures from the REFERENCE itself (holopipe), config-4-like.

Runs holopipe.align.auto_align on seeded frames with a seeded perturbed
starting configuration and records every pipeline evaluation (parameters,
from_stage, the nine metrics) so the GPU engine can be checked in lockstep
(SURVEY.md section 0.10 / 8(d)).  Two runs: tol 0 (lockstep sequence) and
tol 1e-4 dB (end-to-end convergence).  Run in the build container:

    python tests/golden/make_autoalign_golden.py
"""

import copy
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from paper_2204_02348_b200.synth import FrameSpec, frames_digest, make_frames  # noqa: E402
from tests.golden.autoalign_case import FRAMES, start_config  # noqa: E402


def run(tol):
    from holopipe import align
    from holopipe.engine import Engine
    frames = make_frames(FrameSpec(**FRAMES))
    eng = Engine()
    for k, v in start_config().items():
        setattr(eng.config, k, copy.deepcopy(v))
    eng.config.autoAlignTol = tol
    eng.config.threadCount = 1
    eng.source.set_float32(frames)
    log = []
    orig = align._evaluate

    def rec(e, from_stage):
        c = e.config
        params = [c.tilt[0][0], c.tilt[1][0], c.beamCentre[0][0], c.beamCentre[1][0],
                  c.defocus[0], c.basisWaist[0]]
        v = orig(e, from_stage)
        m = np.stack([e.metrics_array(i) for i in range(9)])
        log.append((params, from_stage, m, v))
        return v

    align._evaluate = rec
    snap = {}
    orig_snap = align.snap_estimate

    def snap_rec(e):
        orig_snap(e)
        c = e.config
        snap["params"] = [c.tilt[0][0], c.tilt[1][0], c.beamCentre[0][0], c.beamCentre[1][0],
                          c.defocus[0], c.basisWaist[0]]

    align.snap_estimate = snap_rec
    try:
        goal = align.auto_align(eng)
    finally:
        align._evaluate = orig
        align.snap_estimate = orig_snap
    c = eng.config
    final = [c.tilt[0][0], c.tilt[1][0], c.beamCentre[0][0], c.beamCentre[1][0], c.defocus[0], c.basisWaist[0]]
    eng.calc_metrics()
    return {
        "frames_sha256": np.array(frames_digest(frames)),
        "params": np.array([p for p, _, _, _ in log]),
        "stages": np.array([s for _, s, _, _ in log]),
        "metrics": np.stack([m for _, _, m, _ in log]),
        "values": np.array([v for _, _, _, v in log]),
        "snap": np.array(snap.get("params", [np.nan] * 6)),
        "final": np.array(final), "goal": np.array(goal), "cycles": np.array(eng.tweak_cycles),
        "final_metrics": np.stack([eng.metrics_array(i) for i in range(9)]),
    }


if __name__ == "__main__":
    for tol, name in ((0.0, "autoalign_tol0"), (1e-4, "autoalign_tol1e-4")):
        out = run(tol)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, len(out["stages"]), "evaluations, cycles", int(out["cycles"]), "goal", float(out["goal"]))
