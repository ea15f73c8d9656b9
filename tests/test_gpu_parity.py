"""GPU parity: the CUDA path (through the C ABI, via the engine) against the
reference's own outputs (golden fixtures) and the oracle on the same frames."""

import numpy as np
import pytest

from tests.golden.cases import CASES, make_custom, make_ref_cal
from tests.golden_util import dequant, load, rel_l2_rows

pytestmark = pytest.mark.gpu

FIELD_TOL = 1e-4      # BASELINE.json north_star: max relative L2 on fields and coefs
COEF_TOL = 1e-4
METRIC_TOL_DB = 1e-3


def _engine(case, frames):
    from paper_2204_02348_b200.engine import Engine
    eng = Engine()
    for k, v in case["config"].items():
        setattr(eng.config, k, v)
    eng.source.set_float32(frames)
    if case.get("batch_cal") is not None:
        cal = np.asarray(case["batch_cal"], np.complex64)
        eng.set_batch_calibration(cal.reshape(-1), cal.shape[0], cal.shape[1])
    if case.get("ref_cal") is not None:
        kind, raw = make_ref_cal(case)
        Lc, Hc, Wc = raw.shape
        (eng.ref_cal.set_intensity if kind == 1 else eng.ref_cal.set_field)(raw, Lc, Wc, Hc)
    if case.get("custom") is not None:
        eng.custom_transform = make_custom(case)
    return eng


def _run(eng, case):
    """run_pipeline(0), or the case's sweep entry point (holopipe/engine.py:419-442)."""
    sw = case.get("sweep")
    if sw is None:
        eng.run_pipeline(0)
    elif sw["kind"] == "linear":
        eng.process_batch_frequency_sweep_linear(sw["start"], sw["stop"], sw["count"])
    else:
        eng.process_batch_wavelength_sweep_arbitrary(np.asarray(sw["wavelengths"]), sw["count"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_fields_and_coefs_match_reference(name):
    case, g, frames = load(name)
    eng = _engine(case, frames)
    _run(eng, case)
    fr, fi, sc = (t.cpu().numpy() for t in eng.fields16_device())
    assert fr.shape == g["fr"].shape
    ef = rel_l2_rows(dequant(fr, fi, sc), dequant(g["fr"], g["fi"], g["scale"]))
    assert ef <= FIELD_TOL, f"{name}: field rel L2 {ef:.3e}"
    lsb = max(np.abs(fr.astype(int) - g["fr"]).max(), np.abs(fi.astype(int) - g["fi"]).max())
    assert lsb <= 2, f"{name}: {lsb} LSB"
    assert np.allclose(sc, g["scale"], rtol=1e-5)
    assert np.array_equal(eng._field_axes[0], g["x_axis"]) and np.array_equal(eng._field_axes[1], g["y_axis"])
    assert np.array_equal(eng._window_meta["k0"], g["k0"])
    if "coefs" in g:
        coefs, b, m, p = eng.coef_view()
        ec = rel_l2_rows(coefs, g["coefs"])
        assert ec <= COEF_TOL, f"{name}: coef rel L2 {ec:.3e}"
        eng.calc_metrics()
        got = np.stack([eng.metrics_array(i) for i in range(9)])
        assert np.allclose(got, g["metrics"], atol=METRIC_TOL_DB, rtol=0), np.abs(got - g["metrics"]).max()


@pytest.mark.parametrize("name", ["pr1", "dualpol", "offcentre", "mode0", "average"])
def test_field_summary_matches_reference(name):
    from paper_2204_02348_b200 import constants as C
    case, g, frames = load(name)
    eng = _engine(case, frames)
    eng.run_pipeline(0)
    s = eng.batch_summary(C.PLANE_FIELD)
    ref = g["field_params"]
    assert s.parameters.shape == ref.shape
    for k in (0, 1, 2, 3, 5, 6):
        scale = np.abs(ref[k]).max() + 1e-30
        assert np.allclose(s.parameters[k], ref[k], rtol=2e-4, atol=2e-4 * scale), k
    # MAXABSIDX (analysis.py:61-64): the same flat pixel, except where the two pixels' magnitudes are a
    # proven tie -- equal within fp32 rounding in the oracle's unquantised field (aggregate slot: in
    # sqrt(sum_b |F|^2), analysis.py:88-91)
    same = s.parameters[4].view(np.int32) == ref[4].view(np.int32)
    if not same.all():
        from oracle import holo_oracle as O
        F = O.run_chain(O.Cfg(**case["config"]), frames, batch_cal=case.get("batch_cal"))["fields"]
        B = F.shape[0]
        for q, slot in zip(*np.nonzero(~same)):
            ig = int(s.parameters[4, q, slot].view(np.int32))
            ir = int(ref[4, q, slot].view(np.int32))
            img = (np.abs(F[slot, q]) if slot < B else
                   np.sqrt((np.abs(F[:, q].astype(np.complex128)) ** 2).sum(0))).ravel()
            assert abs(float(img[ig]) - float(img[ir])) <= 2e-6 * float(img[ir]), (name, q, slot, ig, ir)
    assert np.allclose(s.total_intensity, g["field_inten"], rtol=2e-4, atol=1e-4 * g["field_inten"].max())


def test_fourier_plane_and_window_match_reference():
    from paper_2204_02348_b200 import constants as C
    case, g, frames = load("pr1")
    eng = _engine(case, frames)
    eng.run_pipeline(0)
    win = eng.get_fourier_plane_window()[0]
    assert rel_l2_rows(win.reshape(len(win), -1), g["window"].reshape(len(win), -1)) <= 1e-5
    s = eng.batch_summary(C.PLANE_FOURIER)
    for k in (0, 1, 2, 3, 5, 6):
        assert np.allclose(s.parameters[k], g["fourier_params"][k], rtol=1e-4, atol=1e-6), k
    assert np.allclose(s.total_intensity, g["fourier_inten"], rtol=1e-4, atol=1e-5 * g["fourier_inten"].max())


def test_full_fourier_plane_matches_oracle():
    from oracle import holo_oracle as O
    case, g, frames = load("offcentre")
    eng = _engine(case, frames)
    eng.process_fft()
    plane = eng.get_fourier_plane_full()[0]
    ref = O.run_chain(O.Cfg(**case["config"]), frames, stop_after="fft")["plane"]
    assert plane.shape == ref.shape
    assert rel_l2_rows(plane.reshape(len(plane), -1), ref.reshape(len(ref), -1)) <= 1e-5


def test_determinism_bit_equal_repeat():
    case, g, frames = load("dualpol")
    eng = _engine(case, frames)
    a = eng.process_batch()[0]
    b = eng.process_batch()[0]
    assert np.array_equal(a, b)


def test_staged_equals_fused():
    case, g, frames = load("offcentre")
    eng = _engine(case, frames)
    eng.process_fft(); eng.process_ifft(); eng.process_remove_tilt(); eng.extract_coefs()
    staged = eng.coef_view()[0]
    fused = eng.process_batch()[0]
    assert rel_l2_rows(staged, fused) <= 1e-6


def test_uint16_source_matches_float32():
    case, g, frames = load("dualpol")  # Poisson 12-bit frames are integer valued
    eng = _engine(case, frames)
    a = eng.process_batch()[0]
    eng.source.set_uint16(frames.astype(np.uint16))
    b = eng.process_batch()[0]
    assert np.array_equal(a, b)
    eng.source.set_uint16(np.ascontiguousarray(np.transpose(frames.astype(np.uint16), (0, 2, 1))), 1)
    c = eng.process_batch()[0]       # transposed frames take the generic kernel
    assert rel_l2_rows(c, a) <= 1e-5


@pytest.mark.parametrize("name", ["pr1", "dualpol", "largebasis", "multiwl", "dualpol_cal"])
def test_specialised_kernel_matches_generic(name):
    case, g, frames = load(name)
    eng = _engine(case, frames)
    eng.run_pipeline(0)
    fast = [t.cpu().numpy().copy() for t in eng.fields16_device()] + [eng.coefs_device().cpu().numpy().copy()]
    eng.force_generic = True
    eng.run_pipeline(0)
    gen = [t.cpu().numpy() for t in eng.fields16_device()] + [eng.coefs_device().cpu().numpy()]
    assert np.abs(fast[0].astype(int) - gen[0]).max() <= 1 and np.abs(fast[1].astype(int) - gen[1]).max() <= 1
    assert np.allclose(fast[2], gen[2], rtol=1e-5)
    assert rel_l2_rows(fast[3], gen[3]) <= 2e-5


def test_window_upload_from_host_matches_device_source():
    import torch
    case, g, frames = load("dualpol")
    eng = _engine(case, frames)                 # numpy source: window-only upload
    a = eng.process_batch()[0]
    assert eng.last_h2d_bytes == frames.shape[0] * 2 * 128 * 128 * 4
    eng.source.set_float32(torch.from_numpy(frames).cuda())   # device source: no copy
    b = eng.process_batch()[0]
    assert np.array_equal(a, b)
    eng.source.set_float32(frames)
    eng.process_fft()
    plane_host = eng.get_fourier_plane_full()[0]
    eng.source.set_float32(torch.from_numpy(frames).cuda())
    eng.process_fft()
    assert np.array_equal(plane_host, eng.get_fourier_plane_full()[0])


@pytest.mark.parametrize("name", ["pr1", "dualpol", "largebasis", "dualpol_cal"])
def test_tensor_core_row_dft_matches_simt_fft(name):
    """tcgen05 row DFT (fp16 split operands) vs the register FFT path: same fields/coefs."""
    case, g, frames = load(name)
    eng = _engine(case, frames)
    eng.use_tc = True
    eng.run_pipeline(0)
    tc = [t.cpu().numpy().copy() for t in eng.fields16_device()] + [eng.coefs_device().cpu().numpy().copy()]
    eng.use_tc = False
    eng.run_pipeline(0)
    simt = [t.cpu().numpy() for t in eng.fields16_device()] + [eng.coefs_device().cpu().numpy()]
    assert np.abs(tc[0].astype(int) - simt[0]).max() <= 2 and np.abs(tc[1].astype(int) - simt[1]).max() <= 2
    assert np.allclose(tc[2], simt[2], rtol=1e-5)
    assert rel_l2_rows(tc[3], simt[3]) <= 2e-5
    ef = rel_l2_rows(dequant(tc[0], tc[1], tc[2]), dequant(g["fr"], g["fi"], g["scale"]))
    assert ef <= FIELD_TOL


@pytest.mark.parametrize("name", ["refcal_int", "refcal_field"])
def test_reference_calibration_table_matches_reference(name):
    """Processed reference-wave calibration (engine.py:276-335) vs the reference's own table."""
    case, g, frames = load(name)
    eng = _engine(case, frames)
    eng.run_pipeline(0)
    got = eng.get_ref_calibration_fields()
    assert got is not None
    applied, lc, pols, xa, ya, nx, ny = got
    assert applied.shape == g["ref_applied"].shape and lc == applied.shape[0] and pols == applied.shape[1]
    ref = g["ref_applied"].reshape(-1, applied.shape[-2] * applied.shape[-1])
    assert rel_l2_rows(applied.reshape(ref.shape), ref) <= 1e-4
    # disabling the calibration drops it from the next tilt-removal stage (engine.py:250-251)
    eng.ref_cal.enabled = 0
    eng.run_pipeline(2)
    fr, fi, sc = (t.cpu().numpy() for t in eng.fields16_device())
    assert rel_l2_rows(dequant(fr, fi, sc), dequant(g["fr"], g["fi"], g["scale"])) > 1e-2


@pytest.mark.parametrize("name", ["pr1", "dualpol", "largebasis", "dualpol_cal"])
def test_two_kernel_tensor_core_path_matches_reference(name):
    """HPG_FLAG_TC2: row + column DFT on tcgen05 (fp16 split operands), SIMT field kernel."""
    case, g, frames = load(name)
    eng = _engine(case, frames)
    eng.use_tc2 = True
    eng.run_pipeline(0)
    fr, fi, sc = (t.cpu().numpy() for t in eng.fields16_device())
    ef = rel_l2_rows(dequant(fr, fi, sc), dequant(g["fr"], g["fi"], g["scale"]))
    assert ef <= FIELD_TOL, f"{name}: field rel L2 {ef:.3e}"
    lsb = max(np.abs(fr.astype(int) - g["fr"]).max(), np.abs(fi.astype(int) - g["fi"]).max())
    assert lsb <= 2, f"{name}: {lsb} LSB"
    assert np.allclose(sc, g["scale"], rtol=1e-5)
    coefs, _, _, _ = eng.coef_view()
    assert rel_l2_rows(coefs, g["coefs"]) <= COEF_TOL


@pytest.mark.parametrize("name", sorted(CASES))
def test_two_kernel_flag_on_every_case(name):
    """HPG_FLAG_TC2 on every golden case: where the two-kernel path applies (128 window, 42 x 42 field, one
    wavelength, no reference calibration / fill factor / averaging) it must match the reference, and where it
    does not hpg_run must fall back to the kernel that does."""
    from paper_2204_02348_b200 import native
    case, g, frames = load(name)
    eng = _engine(case, frames)
    eng.use_tc2 = True
    _run(eng, case)
    # the cases the two-kernel path must take (two launches): bases of 4 to 45 orders, LG / custom transforms,
    # batch calibration, reference calibration of one wavelength
    if name in {"custom", "dualpol", "dualpol_cal", "dualpol_g24", "largebasis", "lg", "pr1", "refcal_int"}:
        assert native.lib().hpg_last_launch_count() == 2, name
    fr, fi, sc = (t.cpu().numpy() for t in eng.fields16_device())
    ef = rel_l2_rows(dequant(fr, fi, sc), dequant(g["fr"], g["fi"], g["scale"]))
    assert ef <= FIELD_TOL, f"{name}: field rel L2 {ef:.3e}"
    assert max(np.abs(fr.astype(int) - g["fr"]).max(), np.abs(fi.astype(int) - g["fi"]).max()) <= 2
    if "coefs" in g:
        coefs, _, _, _ = eng.coef_view()
        assert rel_l2_rows(coefs, g["coefs"]) <= COEF_TOL


def test_two_kernel_tail_variants_agree(monkeypatch):
    """The half-table tail (five CTAs per SM) and the full shared-memory-basis tail (the variant of large or
    non-symmetric bases) on the same windows: same int16 fields, coefficients to 2e-6."""
    case, g, frames = load("dualpol")
    a = _engine(case, frames)
    a.use_tc2 = True
    a.run_pipeline(0)
    fa = _outputs(a)
    monkeypatch.setenv("HOLO_TAILR_SMEM_BASIS", "1")
    b = _engine(case, frames)
    b.use_tc2 = True
    b.run_pipeline(0)
    fb = _outputs(b)
    for x, y in zip(fa[:3], fb[:3]):
        assert np.array_equal(x, y)
    assert rel_l2_rows(fa[3], fb[3]) <= 2e-6
    assert rel_l2_rows(fb[3], g["coefs"]) <= COEF_TOL


def test_frames_from_a_file_match_the_uint16_buffer(tmp_path):
    """set_frame_buffer_from_file (holopipe/frames.py:61-75: raw little-endian uint16): same outputs as the same
    integers handed over as a uint16 buffer, through the handle API."""
    from paper_2204_02348_b200 import api
    from paper_2204_02348_b200.errors import ErrorCode
    case, g, frames = load("dualpol")
    u16 = np.rint(frames).astype("<u2")
    path = tmp_path / "frames.bin"
    u16.tofile(path)

    def run(setter):
        h = api.create_handle()
        eng = api.engine(h)
        for k, v in case["config"].items():
            setattr(eng.config, k, v)
        assert setter(h) == ErrorCode.SUCCESS
        coefs, b, m, p = api.process_batch(h)
        fields = api.get_fields16(h)[:3]
        api.destroy_handle(h)
        return coefs, fields

    ca, fa = run(lambda h: api.set_frame_buffer_from_file(h, str(path)))
    cb, fb = run(lambda h: api.set_frame_buffer_uint16(h, u16))
    assert np.array_equal(ca, cb)
    for x, y in zip(fa, fb):
        assert np.array_equal(x, y)
    assert rel_l2_rows(ca, g["coefs"]) <= COEF_TOL
    h = api.create_handle()
    assert api.set_frame_buffer_from_file(h, str(tmp_path / "missing.bin")) == ErrorCode.FILENOTFOUND
    api.destroy_handle(h)


def _outputs(eng):
    out = [t.cpu().numpy().copy() for t in eng.fields16_device()]
    co = eng.coefs_device()
    return out + [None if co is None or co.numel() == 0 else co.cpu().numpy().copy()]


def test_two_kernel_path_uint16_frames_equal_float32():
    """The Fourier kernel's uint16 instantiation (camera format, holopipe/frames.py:49-59): bit-equal to the
    float32 run of the same integers."""
    case, g, frames = load("dualpol")
    frames = np.rint(frames)
    a = _engine(case, frames.astype(np.float32))
    a.use_tc2 = True
    a.run_pipeline(0)
    b = _engine(case, frames.astype(np.float32))
    b.source.set_uint16(frames.astype(np.uint16))
    b.use_tc2 = True
    b.run_pipeline(0)
    for x, y in zip(_outputs(a), _outputs(b)):
        assert np.array_equal(x, y)


def test_two_kernel_path_fields_only():
    """No basis (basisGroupCount 0): the tail stops after the int16 fields; same fields as the fused kernel."""
    case, g, frames = load("dualpol")
    case = dict(case, config=dict(case["config"], basisGroupCount=0))
    a = _engine(case, frames)
    a.use_tc2 = True
    a.run_pipeline(0)
    b = _engine(case, frames)
    b.run_pipeline(0)
    fa, fb = _outputs(a), _outputs(b)
    assert fa[3] is None and fb[3] is None
    assert np.abs(fa[0].astype(int) - fb[0]).max() <= 2 and np.abs(fa[1].astype(int) - fb[1]).max() <= 2
    assert np.allclose(fa[2], fb[2], rtol=1e-5)
    ef = rel_l2_rows(dequant(fa[0], fa[1], fa[2]), dequant(g["fr"], g["fi"], g["scale"]))
    assert ef <= FIELD_TOL


def test_two_kernel_path_chosen_for_large_batches_and_chunked():
    """hpg_run picks the two-kernel path by itself for >= 6 windows per SM; 1,100 dual-pol rows = 2,200 windows
    cross its 2,048-window chunk boundary.  Every repetition of the tiled golden frames must reproduce the
    first bit for bit, and the rows must match the reference fixture."""
    import torch
    from paper_2204_02348_b200 import native
    case, g, frames = load("dualpol")
    n = frames.shape[0]
    rows = 1100
    reps = -(-rows // n)
    big = np.ascontiguousarray(np.concatenate([frames] * reps)[:rows])
    case = dict(case, config=dict(case["config"], batchCount=rows))
    eng = _engine(case, torch.from_numpy(big).cuda())
    eng.run_pipeline(0)
    assert native.lib().hpg_last_launch_count() == 4   # two chunks x (Fourier kernel + tail)
    fr, fi, sc, co = _outputs(eng)
    for r in range(1, rows // n):
        for x in (fr, fi, sc, co):
            assert np.array_equal(x[r * n:(r + 1) * n], x[:n])
    ef = rel_l2_rows(dequant(fr[:n], fi[:n], sc[:n]), dequant(g["fr"], g["fi"], g["scale"]))
    assert ef <= FIELD_TOL
    assert rel_l2_rows(co[:n], g["coefs"]) <= COEF_TOL


@pytest.mark.parametrize("name", ["dualpol", "pr1", "multiwl"])
def test_pipelined_process_batch_matches_staged(name):
    """api.process_batch on host frames (chunked upload / kernel / readback) == run_pipeline + coef_view."""
    from paper_2204_02348_b200.engine import Engine
    case, g, frames = load(name)
    rows = 48 if name != "multiwl" else 40
    reps = -(-rows // frames.shape[0])
    big = np.ascontiguousarray(np.concatenate([frames] * reps)[:rows * max(1, case["config"].get("avgCount", 1))])
    def make():
        eng = Engine()
        for k, v in case["config"].items():
            setattr(eng.config, k, v)
        eng.config.batchCount = rows
        eng.source.set_float32(big)
        return eng
    a = make()
    assert a._pipeline_ok()
    ca, ba, ma, pa = a.process_batch()
    b = make()
    b.run_pipeline(0)
    cb, bb, mb, pb = b.coef_view()
    assert (ba, ma, pa) == (bb, mb, pb)
    assert np.array_equal(ca, cb)
    fa = [t.cpu().numpy() for t in a.fields16_device()]
    fb = [t.cpu().numpy() for t in b.fields16_device()]
    for x, y in zip(fa, fb):
        assert np.array_equal(x, y)
    # staged getters still work after the pipelined call
    assert a.get_fields16() is not None
    # second call reuses the buffers
    cc, _, _, _ = a.process_batch()
    assert np.array_equal(cc, ca)


@pytest.mark.parametrize("name", ["dualpol", "pr1"])
def test_pipelined_fields_only_matches_staged(name):
    """No basis: the pipelined process_batch reads the int16 fields back chunk by chunk; get_fields16 then
    returns them (once), bit-equal to run_pipeline + get_fields16, and the next call reads the device again."""
    from paper_2204_02348_b200.engine import Engine
    case, g, frames = load(name)
    rows = 48
    big = np.ascontiguousarray(np.concatenate([frames] * -(-rows // frames.shape[0]))[:rows])
    def make():
        eng = Engine()
        for k, v in case["config"].items():
            setattr(eng.config, k, v)
        eng.config.batchCount = rows
        eng.config.basisGroupCount = 0
        eng.source.set_float32(big)
        return eng
    a = make()
    assert a._pipeline_ok()
    assert a.process_batch()[0] is None
    fa = a.get_fields16()
    b = make()
    b.run_pipeline(0)
    fb = b.get_fields16()
    for x, y in zip(fa[:3], fb[:3]):
        assert np.array_equal(x, y)
    fa2 = a.get_fields16()   # second read comes from the device
    for x, y in zip(fa2[:3], fb[:3]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("name", ["largebasis", "dualpol_g24"])
def test_tensor_core_overlap_matches_simt_overlap(name):
    """HG overlap on tcgen05 (exact int16 splits) vs the SIMT overlap: same fields, coefs within 2e-6."""
    case, g, frames = load(name)
    eng = _engine(case, frames)
    eng.run_pipeline(0)
    a = [t.cpu().numpy().copy() for t in eng.fields16_device()] + [eng.coefs_device().cpu().numpy().copy()]
    eng.simt_overlap = True
    eng.run_pipeline(0)
    b = [t.cpu().numpy() for t in eng.fields16_device()] + [eng.coefs_device().cpu().numpy()]
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)
    assert rel_l2_rows(a[3], b[3]) <= 2e-6
    assert rel_l2_rows(a[3], g["coefs"]) <= COEF_TOL


@pytest.mark.parametrize("name", ["largeframe", "n256"])
def test_large_window_path_matches_generic(name):
    """Chunked large-window kernels (rows / columns / field / pack) == the generic fused kernel."""
    case, g, frames = load(name)
    eng = _engine(case, frames)
    eng.run_pipeline(0)
    a = [t.cpu().numpy().copy() for t in eng.fields16_device()]
    eng.force_generic = True
    eng.run_pipeline(0)
    b = [t.cpu().numpy() for t in eng.fields16_device()]
    assert np.abs(a[0].astype(int) - b[0]).max() <= 2 and np.abs(a[1].astype(int) - b[1]).max() <= 2
    assert np.allclose(a[2], b[2], rtol=1e-5)


def test_large_window_path_features_match_generic():
    """Large-window kernels with dual-pol, two wavelengths, batch calibration and uint16 frames
    against the generic fused kernel on the same inputs (rows independent, per-row wavelength)."""
    from paper_2204_02348_b200.engine import Engine
    from paper_2204_02348_b200.synth import FrameSpec, make_frames
    PIX = 20e-6
    frames = make_frames(FrameSpec(width=640, height=256, pol_count=2, batch=4, group_count=6, waist=300e-6,
                                   tilt=(1.0, 1.1), noise="poisson", seed=31))
    def make(u16):
        eng = Engine()
        c = eng.config
        c.frameWidth, c.frameHeight, c.polCount, c.batchCount = 640, 256, 2, 4
        c.fftWindowSizeX = c.fftWindowSizeY = 256
        c.framePixelSize, c.wavelengthCentre = PIX, 1565e-9
        c.fourierWindowRadius = 0.32 * np.degrees(1565e-9 / (2 * PIX))
        c.wavelengths = [1550e-9, 1580e-9]
        c.tilt = [[1.0, 1.0], [1.1, 1.1]]
        c.beamCentre = [[-160 * PIX, 160 * PIX], [0.0, 0.0]]
        c.basisGroupCount, c.basisWaist = 6, [300e-6, 300e-6]
        cal = np.array([[1.0 + 0.5j, 0.8 - 0.1j], [0.3j + 1, 1.2]], np.complex64)
        eng.set_batch_calibration(cal.reshape(-1), 2, 2)
        if u16:
            eng.source.set_uint16(np.rint(frames).astype(np.uint16))
        else:
            eng.source.set_float32(np.rint(frames).astype(np.float32))
        return eng
    out = []
    for u16, generic in ((False, False), (True, False), (False, True)):
        eng = make(u16)
        eng.force_generic = generic
        eng.run_pipeline(0)
        out.append([t.cpu().numpy().copy() for t in eng.fields16_device()] + [eng.coefs_device().cpu().numpy()])
    lw, lw16, gen = out
    for x, y in zip(lw[:2], lw16[:2]):
        assert np.array_equal(x, y)                       # uint16 == float32 of the same integers
    assert np.abs(lw[0].astype(int) - gen[0]).max() <= 2 and np.abs(lw[1].astype(int) - gen[1]).max() <= 2
    assert np.allclose(lw[2], gen[2], rtol=1e-5)
    assert rel_l2_rows(lw[3], gen[3]) <= 2e-5


@pytest.mark.parametrize("path", ["default", "tc", "tc2", "generic"])
def test_zero_frames_give_zero_fields_and_unit_scale(path):
    """peak = 0 -> scale 1, all-zero int16 fields and coefficients (pipeline.py:194-198), every kernel."""
    case, g, frames = load("dualpol")
    eng = _engine(case, np.zeros_like(frames))
    eng.use_tc = path == "tc"
    eng.use_tc2 = path == "tc2"
    eng.force_generic = path == "generic"
    eng.run_pipeline(0)
    fr, fi, sc = (t.cpu().numpy() for t in eng.fields16_device())
    assert not fr.any() and not fi.any()
    assert np.all(sc == 1.0)
    assert not np.abs(eng.coefs_device().cpu().numpy()).any()


def test_single_frame_batch():
    """B = 1 through the default kernel equals row 0 of the 3-frame batch."""
    case, g, frames = load("dualpol")
    a = _engine(case, frames)
    a.run_pipeline(0)
    one = dict(case, config=dict(case["config"], batchCount=1))
    b = _engine(one, frames[:1])
    b.run_pipeline(0)
    for x, y in zip(a.fields16_device(), b.fields16_device()):
        assert np.array_equal(x.cpu().numpy()[:1], y.cpu().numpy())
    assert np.array_equal(a.coefs_device().cpu().numpy()[:1], b.coefs_device().cpu().numpy())


@pytest.mark.parametrize("name", ["pr1", "dualpol"])
def test_fill_factor_in_the_fast_kernel_matches_generic(name):
    """Fill-factor envelope folded into the separable recentring tables == the generic window table."""
    case, g, frames = load(name)
    case = dict(case, config=dict(case["config"], fillFactorCorrectionEnabled=1))
    eng = _engine(case, frames)
    eng.run_pipeline(0)
    a = [t.cpu().numpy().copy() for t in eng.fields16_device()] + [eng.coefs_device().cpu().numpy().copy()]
    eng.force_generic = True
    eng.run_pipeline(0)
    b = [t.cpu().numpy() for t in eng.fields16_device()] + [eng.coefs_device().cpu().numpy()]
    assert np.abs(a[0].astype(int) - b[0]).max() <= 2 and np.abs(a[1].astype(int) - b[1]).max() <= 2
    assert np.allclose(a[2], b[2], rtol=1e-5)
    assert rel_l2_rows(a[3], b[3]) <= 2e-5
    # ... and folded into the DFT matrices of the two-kernel tensor-core path
    from paper_2204_02348_b200 import native
    eng.force_generic = False
    eng.use_tc2 = True
    eng.run_pipeline(0)
    assert native.lib().hpg_last_launch_count() == 2
    c = [t.cpu().numpy() for t in eng.fields16_device()] + [eng.coefs_device().cpu().numpy()]
    assert np.abs(c[0].astype(int) - b[0]).max() <= 2 and np.abs(c[1].astype(int) - b[1]).max() <= 2
    assert np.allclose(c[2], b[2], rtol=1e-5)
    assert rel_l2_rows(c[3], b[3]) <= 2e-5
    # the correction is not a no-op on these frames: without it the fields differ
    off = _engine(dict(case, config=dict(case["config"], fillFactorCorrectionEnabled=0)), frames)
    off.run_pipeline(0)
    d = [t.cpu().numpy() for t in off.fields16_device()]
    assert rel_l2_rows(dequant(d[0], d[1], d[2]), dequant(b[0], b[1], b[2])) > 1e-3
