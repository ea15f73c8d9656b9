"""Output writers (holopipe/settings.py:186-293): file formats pinned against files the REFERENCE wrote for
the pr1 golden case (tests/golden/make_writer_golden.py)."""
import os

import numpy as np
import pytest

from paper_2204_02348_b200 import api, writers
from tests.golden.cases import CASES
from tests.golden_util import dequant, load, rel_l2_rows

W = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "writers")


def _handle():
    case = CASES["pr1"]
    h = api.create_handle()
    eng = api.engine(h)
    for k, v in case["config"].items():
        setattr(eng.config, k, v)
    eng.config.threadCount = 1
    return h, case


def test_readers_parse_reference_files():
    case, g, _ = load("pr1")
    f = writers.read_fields(os.path.join(W, "pr1_fields.bin"))
    assert f.shape == g["fr"].shape
    assert np.array_equal(f, dequant(g["fr"], g["fi"], g["scale"]).astype(np.complex64))
    c = writers.read_coefs(os.path.join(W, "pr1_coefs.bin"))
    assert np.array_equal(c, g["coefs"])


def test_settings_dump_matches_reference_summary():
    """The settings block of write_summary is byte-identical to the reference's for the same config."""
    h, case = _handle()
    ref = open(os.path.join(W, "pr1_summary.txt")).read()
    ours = writers.serialise_settings(h)
    assert ref.startswith(ours), (ours, ref[:len(ours)])
    api.destroy_handle(h)


def test_writer_errors():
    h, _ = _handle()
    from paper_2204_02348_b200.errors import HoloError
    with pytest.raises(HoloError):
        writers.write_coefs(h, "/nonexistent-dir/x.bin")
    api.destroy_handle(h)


@pytest.mark.gpu
def test_writers_round_trip_on_the_gpu_engine(tmp_path):
    case, g, frames = load("pr1")
    h, _ = _handle()
    api.set_batch(h, case["config"]["batchCount"], frames)
    api.process_batch(h)
    api.auto_align_calc_metrics(h)
    assert writers.write_fields(h, str(tmp_path / "f.bin")) == 0
    assert writers.write_coefs(h, str(tmp_path / "c.bin")) == 0
    assert writers.write_summary(h, str(tmp_path / "s.txt")) == 0
    f = writers.read_fields(str(tmp_path / "f.bin"))
    assert np.array_equal(f, api.get_fields(h)[0])
    assert rel_l2_rows(f, writers.read_fields(os.path.join(W, "pr1_fields.bin"))) <= 1e-4
    c = writers.read_coefs(str(tmp_path / "c.bin"))
    assert np.array_equal(c, api.basis_get_coefs(h)[0])
    assert rel_l2_rows(c, writers.read_coefs(os.path.join(W, "pr1_coefs.bin"))) <= 1e-4
    ours, ref = writers.read_summary(str(tmp_path / "s.txt")), writers.read_summary(os.path.join(W, "pr1_summary.txt"))
    assert ours.keys() == ref.keys()
    for k in ref:
        if k.startswith("Metric."):
            assert np.allclose(np.float64(ours[k]), np.float64(ref[k]), atol=1e-3), k
        else:
            assert ours[k] == ref[k], k
    api.destroy_handle(h)
