"""The B200 package exposes every public function of the reference api (drop-in surface)."""
import json
import os

import pytest

from paper_2204_02348_b200 import api

HERE = os.path.dirname(os.path.abspath(__file__))


def test_every_reference_api_function_exists():
    names = json.load(open(os.path.join(HERE, "golden", "reference_api_names.json")))["names"]
    missing = [n for n in names if not callable(getattr(api, n, None))]
    assert not missing, missing


def test_handle_errors_follow_the_reference_codes():
    assert api.get_viewport_to_file(123456, 0, 0, "x") == 2          # INVALIDHANDLE
    assert api.process_batch(123456) == (None, 0, 0, 0)               # api.py:854-861
    h = api.create_handle()
    assert api.config_set_frame_dimensions(h, 320, 256) == 0
    assert api.destroy_handle(h) == 0


def test_pipeline_chunk_count_policy():
    """process_batch chunks: one per ~48 MB of window upload, 4..16, and >= 8 rows per chunk."""
    from paper_2204_02348_b200.engine import Engine
    if Engine._PIPE_CHUNKS_ENV:
        pytest.skip("HOLO_PIPE_CHUNKS set")
    e = Engine.__new__(Engine)
    mb = 1 << 20
    assert e._pipe_chunks(1000, 131 * mb) == 4        # dual-pol: 1000 frames x 2 x 128^2 f32
    assert e._pipe_chunks(8192, 537 * mb) == 12       # large basis: 8192 frames x 128^2 f32
    assert e._pipe_chunks(65536, 4300 * mb) == 16     # capped
    assert e._pipe_chunks(40, 4300 * mb) == 5         # >= 8 rows per chunk
    assert e._pipe_chunks(32, 1 * mb) == 4            # floor


def test_parameter_lists_match_the_reference():
    """Keyword callers of holopipe.api (e.g. config_set_batch_count(h, batch_count=8)) keep working:
    every function has the reference's parameter names, order and defaults."""
    import inspect
    ref = json.load(open(os.path.join(HERE, "golden", "reference_api_names.json")))["params"]
    bad = []
    for name, plist in ref.items():
        sig = inspect.signature(getattr(api, name))
        ours = [[p.name] if p.default is inspect.Parameter.empty else [p.name, p.default]
                for p in sig.parameters.values()]
        if ours != plist:
            bad.append((name, plist, ours))
    assert not bad, bad


def test_keyword_setters():
    h = api.create_handle()
    assert api.config_set_batch_count(h, batch_count=8) == 0
    assert api.config_get_batch_count(h) == 8
    assert api.config_set_tilt(h, axis=0, pol=0, tilt=1.25) == 0
    assert api.config_get_tilt(h, 0, 0) == 1.25
    assert api.config_set_fft_window_size_x(h, width=100) == 96
    assert api.config_set_auto_align_mode(h, align_mode=7) == 8      # INVALIDARGUMENT
    assert api.config_set_pol_lock_tilt(h, pol_lock=1) == 0
    assert api.config_set_basis_group_count(123456, group_count=3) == 2
    api.destroy_handle(h)
