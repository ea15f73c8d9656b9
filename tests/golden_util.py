"""Helpers to load the golden fixtures and regenerate their seeded frames."""

import os

import numpy as np

from paper_2204_02348_b200.synth import FrameSpec, frames_digest, make_frames
from tests.golden.cases import CASES

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_cache = {}


def load(name):
    """(case dict, golden npz dict, frames) with the frame digest verified."""
    if name not in _cache:
        case = CASES[name]
        g = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
        frames = make_frames(FrameSpec(**case["frames"]))
        assert frames_digest(frames) == str(g["frames_sha256"]), \
            f"{name}: regenerated frames differ from the ones the reference saw"
        _cache[name] = (case, g, frames)
    return _cache[name]


def rel_l2_rows(a, b):
    a = np.asarray(a, np.complex128).reshape(a.shape[0], -1)
    b = np.asarray(b, np.complex128).reshape(b.shape[0], -1)
    den = np.linalg.norm(b, axis=1)
    den = np.where(den > 0, den, 1.0)
    return float(np.max(np.linalg.norm(a - b, axis=1) / den))


def dequant(fr, fi, scale):
    return (fr.astype(np.float32) + 1j * fi.astype(np.float32)) / scale[..., None, None]
