"""Viewport renders (holopipe/viewport.py): colour rules on CPU, every display mode against the reference's
own renders of the pr1 golden case on the GPU engine (tests/golden/make_viewport_golden.py)."""
import os
import struct

import numpy as np
import pytest

from paper_2204_02348_b200 import api, viewport
from tests.golden.cases import CASES
from tests.golden_util import load

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "viewport_pr1.npz")


def test_colour_rules():
    z = np.array([[1.0, 1j, -1.0, -1j, 0.0]])
    rgb = viewport.complex_to_rgb(z)
    assert rgb.shape == (1, 5, 3) and rgb.dtype == np.uint8
    assert tuple(rgb[0, 4]) == (0, 0, 0)                       # zero magnitude -> black
    assert tuple(rgb[0, 2]) == (255, 0, 0)                     # phase pi -> hue 1 -> red
    assert tuple(rgb[0, 0]) == (0, 255, 255)                   # phase 0 -> hue 1/2 -> cyan
    assert tuple(rgb[0, 1]) == (128, 0, 255) and tuple(rgb[0, 3]) == (128, 255, 0)
    g = viewport.magnitude_to_rgb(np.array([[1.0, 0.5, 1e-4]]), db=True)
    # 0 dB -> 255; -6.02 dB -> 255 (1 - 6.02 / 60) = 229; -80 dB is below the -60 dB floor -> 0
    assert g[0, 0, 0] == 255 and g[0, 1, 0] == 229 and g[0, 2, 0] == 0 and np.all(g[..., 0] == g[..., 2])
    assert viewport.magnitude_to_rgb(np.zeros((2, 2))).max() == 0


def test_bmp_layout(tmp_path):
    rgb = np.arange(2 * 3 * 3, dtype=np.uint8).reshape(2, 3, 3)
    p = tmp_path / "x.bmp"
    viewport.write_bmp(str(p), rgb)
    raw = p.read_bytes()
    assert raw[:2] == b"BM" and struct.unpack("<I", raw[2:6])[0] == len(raw) == 54 + 2 * 12
    w, h = struct.unpack("<ii", raw[18:26])
    assert (w, h) == (3, 2)
    assert raw[54:57] == bytes(rgb[1, 0, ::-1])               # bottom row first, BGR


def test_invalid_handle_and_mode():
    assert api.get_viewport(123456, 1) is None
    assert api.get_viewport_to_file(123456, 1, 0, "x.bmp") == 2
    h = api.create_handle()
    assert api.get_viewport(h, 99) is None
    api.destroy_handle(h)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", range(1, 9))
def test_render_matches_reference(mode, tmp_path):
    case, g, frames = load("pr1")
    ref = np.load(G)[f"mode{mode}"]
    h = api.create_handle()
    eng = api.engine(h)
    for k, v in case["config"].items():
        setattr(eng.config, k, v)
    api.set_batch(h, case["config"]["batchCount"], frames)
    api.process_batch(h)
    rgb, w, hh, title = api.get_viewport(h, mode, 0)
    assert rgb.shape == ref.shape and (w, hh) == (ref.shape[1], ref.shape[0])
    diff = np.abs(rgb.astype(int) - ref.astype(int))
    # fields / planes agree to ~1e-5 relative: colour levels within a few counts, hue wraps aside
    assert np.mean(diff <= 3) >= 0.99, (mode, diff.max(), np.mean(diff <= 3))
    assert api.get_viewport_to_file(h, mode, 0, str(tmp_path / "v.bmp")) == 0
    api.destroy_handle(h)
