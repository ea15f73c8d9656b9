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
