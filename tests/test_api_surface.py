"""The B200 package exposes every public function of the reference api (drop-in surface)."""
import json
import os

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
