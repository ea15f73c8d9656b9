"""AutoAlign parity against the reference's own run.

lockstep : replay the reference's evaluation sequence (parameters, from_stage)
           on the GPU engine; every evaluation's metrics within 1e-3 dB.
snap     : the coarse estimate from the same starting point.
end2end  : tol 1e-4 dB, converged goal within 1e-3 dB.
"""

import copy
import os

import numpy as np
import pytest

from paper_2204_02348_b200.synth import FrameSpec, frames_digest, make_frames
from tests.golden.autoalign_case import FRAMES, start_config

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_frames = {}


def _fx():
    if "f" not in _frames:
        _frames["f"] = make_frames(FrameSpec(**FRAMES))
    return _frames["f"]


def _engine(tol=0.0):
    from paper_2204_02348_b200.engine import Engine
    eng = Engine()
    for k, v in start_config().items():
        setattr(eng.config, k, copy.deepcopy(v))
    eng.config.autoAlignTol = tol
    eng.source.set_float32(_fx())
    return eng


def _set(eng, prm):
    c = eng.config
    c.tilt[0][0] = c.tilt[0][1] = prm[0]
    c.tilt[1][0] = c.tilt[1][1] = prm[1]
    c.beamCentre[0][0], c.beamCentre[1][0] = prm[2], prm[3]
    c.defocus[0] = c.defocus[1] = prm[4]
    c.basisWaist[0] = c.basisWaist[1] = prm[5]


def test_lockstep_metrics_match_reference():
    g = np.load(os.path.join(GOLDEN, "autoalign_tol0.npz"))
    assert frames_digest(_fx()) == str(g["frames_sha256"])
    eng = _engine()
    worst = 0.0
    for prm, st, ref in zip(g["params"], g["stages"], g["metrics"]):
        _set(eng, prm)
        eng.run_pipeline(int(st))
        eng.calc_metrics()
        got = np.stack([eng.metrics_array(i) for i in range(9)])
        ok = ref > -1e30
        assert np.array_equal(ok, got > -1e30)
        worst = max(worst, float(np.abs(got[ok] - ref[ok]).max()))
    assert worst <= 1e-3, worst


def test_snap_estimate_matches_reference():
    from paper_2204_02348_b200 import align
    g = np.load(os.path.join(GOLDEN, "autoalign_tol0.npz"))
    eng = _engine()
    align.snap_estimate(eng)
    c = eng.config
    got = np.array([c.tilt[0][0], c.tilt[1][0], c.beamCentre[0][0], c.beamCentre[1][0], c.defocus[0],
                    c.basisWaist[0]])
    ref = g["snap"]
    assert np.allclose(got[:2], ref[:2], atol=1e-6)            # degrees
    assert np.allclose(got[2:4], ref[2:4], atol=1e-9)          # metres
    assert abs(got[4] - ref[4]) <= 1e-3 * max(1.0, abs(ref[4]))
    assert abs(got[5] / ref[5] - 1) <= 1e-5


def test_end_to_end_converges_like_reference():
    """The tweak stage is a trajectory: a 2e-6 dB difference in one parabola
    point moves a vertex by a sub-nanometre amount and later decisions diverge
    (tools/autoalign_trace.py finds the first divergent evaluation).  The bar
    is therefore on the converged goal: not worse than the reference's by more
    than 1e-3 dB, and the converged parameters in the same basin."""
    from paper_2204_02348_b200 import align
    g = np.load(os.path.join(GOLDEN, "autoalign_tol1e-4.npz"))
    eng = _engine(tol=1e-4)
    goal = align.auto_align(eng)
    ref = float(g["goal"])
    assert goal >= ref - 1e-3, (goal, ref)
    assert goal <= ref + 0.05, (goal, ref)
    c = eng.config
    got = np.array([c.tilt[0][0], c.tilt[1][0], c.beamCentre[0][0], c.beamCentre[1][0], c.defocus[0],
                    c.basisWaist[0]])
    fin = g["final"]
    assert np.all(np.abs(got[:2] - fin[:2]) <= 0.01)          # degrees
    assert np.all(np.abs(got[2:4] - fin[2:4]) <= 2e-6)        # metres (0.1 px)
    assert abs(got[5] / fin[5] - 1) <= 0.02
