"""Output writers: fields / coefficients / run summary in the reference's file formats
(holopipe/settings.py:186-293), on top of the handle getters.

Formats (little-endian float32, interleaved (re, im)):
  fields   [batch][pol][height][width][2] + sidecar '<path>.txt' (batchCount, polCount, width, height,
           xSpacing, ySpacing, format)
  coefs    [batch][pol * modeCount][2] (pol blocks HH..VV) + sidecar (batchCount, modeCount, polCount, format)
  summary  settings dump (one 'Key<TAB>values' line per setting, the reference's key order) followed by
           ResultBatchCount / ResultModeCount / ResultPolCount and one 'Metric.<NAME>' line per metric.
The readers re-ingest files written by either implementation.
"""

from __future__ import annotations

import numpy as np

from . import api
from .errors import ErrorCode, HoloError


def _pols(h):
    return range(api.config_get_pol_count(h))


# setting key -> getter (values), in the order of holopipe/settings.py:_SERIALISE_ORDER
_SETTINGS = [
    ("FrameDimensions", lambda h: list(api.config_get_frame_dimensions(h))),
    ("FramePixelSize", lambda h: [api.config_get_frame_pixel_size(h)]),
    ("PolCount", lambda h: [api.config_get_pol_count(h)]),
    ("fftWindowSize", lambda h: list(api.config_get_fft_window_size(h))),
    ("FourierWindowRadius", lambda h: [api.config_get_fourier_window_radius(h)]),
    ("IFFTResolutionMode", lambda h: [api.config_get_ifft_resolution_mode(h)]),
    ("FillFactorCorrectionEnabled", lambda h: [api.config_get_fill_factor_correction_enabled(h)]),
    ("WavelengthCentre", lambda h: [api.config_get_wavelength_centre(h)]),
    ("Wavelengths", lambda h: list(api.config_get_wavelengths(h)[0])),
    ("WavelengthOrderingIn", lambda h: [api.config_get_wavelength_ordering(h, 0)]),
    ("WavelengthOrderingOut", lambda h: [api.config_get_wavelength_ordering(h, 1)]),
    ("BeamCentreX", lambda h: [api.config_get_beam_centre(h, 0, p) for p in _pols(h)]),
    ("BeamCentreY", lambda h: [api.config_get_beam_centre(h, 1, p) for p in _pols(h)]),
    ("TiltX", lambda h: [api.config_get_tilt(h, 0, p) for p in _pols(h)]),
    ("TiltY", lambda h: [api.config_get_tilt(h, 1, p) for p in _pols(h)]),
    ("Defocus", lambda h: [api.config_get_defocus(h, p) for p in _pols(h)]),
    ("BasisWaist", lambda h: [api.config_get_basis_waist(h, p) for p in _pols(h)]),
    ("PolLockTilt", lambda h: [api.config_get_pol_lock_tilt(h)]),
    ("PolLockDefocus", lambda h: [api.config_get_pol_lock_defocus(h)]),
    ("PolLockBasisWaist", lambda h: [api.config_get_pol_lock_basis_waist(h)]),
    ("BasisGroupCount", lambda h: [api.config_get_basis_group_count(h)]),
    ("BasisType", lambda h: [api.config_get_basis_type(h)]),
    ("BatchCount", lambda h: [api.config_get_batch_count(h)]),
    ("AvgCount", lambda h: [api.config_get_batch_avg_count(h)]),
    ("AvgMode", lambda h: [api.config_get_batch_avg_mode(h)]),
    ("ThreadCount", lambda h: [api.config_get_thread_count(h)]),
    ("Verbosity", lambda h: [api.config_get_verbosity(h)]),
    ("FFTPlanMode", lambda h: [api.config_get_plan_mode(h)]),
    ("AutoAlignTilt", lambda h: [api.config_get_auto_align_tilt(h)]),
    ("AutoAlignBeamCentre", lambda h: [api.config_get_auto_align_beam_centre(h)]),
    ("AutoAlignDefocus", lambda h: [api.config_get_auto_align_defocus(h)]),
    ("AutoAlignBasisWaist", lambda h: [api.config_get_auto_align_basis_waist(h)]),
    ("AutoAlignFourierWindowRadius", lambda h: [api.config_get_auto_align_fourier_window_radius(h)]),
    ("AutoAlignTol", lambda h: [api.config_get_auto_align_tol(h)]),
    ("AutoAlignMode", lambda h: [api.config_get_auto_align_mode(h)]),
    ("AutoAlignGoalIdx", lambda h: [api.config_get_auto_align_goal_idx(h)]),
    ("AutoAlignPolIndependence", lambda h: [api.config_get_auto_align_pol_independence(h)]),
    ("AutoAlignBasisMulConjTrans", lambda h: [api.config_get_auto_align_basis_mul_conj_trans(h)]),
]

METRIC_NAMES = ["IL", "MDL", "DIAG", "SNRAVG", "DIAGBEST", "DIAGWORST", "SNRBEST", "SNRWORST", "SNRMG"]


def _fmt(value):
    if isinstance(value, (int, np.integer)):
        return str(int(value))
    return repr(float(value))   # round-trip exact


def serialise_settings(handle):
    """The handle's configuration as settings text (one tab-separated line per key)."""
    return "".join("\t".join([key] + [_fmt(v) for v in get(handle)]) + "\n" for key, get in _SETTINGS)


def _interleave(z):
    out = np.empty(z.shape + (2,), dtype="<f4")
    out[..., 0] = z.real
    out[..., 1] = z.imag
    return out


def _sidecar(path, rows):
    with open(str(path) + ".txt", "w") as fh:
        for k, v in rows:
            fh.write(f"{k}\t{v}\n")


def _read_sidecar(path):
    meta = {}
    with open(str(path) + ".txt") as fh:
        for line in fh:
            parts = line.rstrip("\n").split("\t")
            if len(parts) == 2:
                meta[parts[0]] = parts[1]
    return meta


def write_fields(handle, path):
    """Dequantised fields, float32 interleaved, batch-major then pol-major, plus the sidecar."""
    got = api.get_fields(handle)
    if got is None:
        raise HoloError(ErrorCode.NULLPOINTER, "no fields to write")
    fields, batch, pol, x_axis, y_axis, _, _ = got
    dx = float(x_axis[1] - x_axis[0]) if x_axis.size > 1 else 0.0
    dy = float(y_axis[1] - y_axis[0]) if y_axis.size > 1 else 0.0
    try:
        _interleave(fields).tofile(path)
        _sidecar(path, [("batchCount", batch), ("polCount", pol), ("width", x_axis.size), ("height", y_axis.size),
                        ("xSpacing", repr(dx)), ("ySpacing", repr(dy)),
                        ("format", "float32 interleaved (re, im), batch-major, pol-major, row-major")])
    except OSError:
        raise HoloError(ErrorCode.FILENOTCREATED, str(path))
    return ErrorCode.SUCCESS


def read_fields(path):
    meta = _read_sidecar(path)
    shape = (int(meta["batchCount"]), int(meta["polCount"]), int(meta["height"]), int(meta["width"]), 2)
    raw = np.fromfile(path, dtype="<f4").reshape(shape)
    return (raw[..., 0] + 1j * raw[..., 1]).astype(np.complex64)


def write_coefs(handle, path):
    """Coefficients (output ordering, pol blocks HH..VV), float32 interleaved, plus the sidecar."""
    coefs, batch, mode_count, pol = api.basis_get_coefs(handle)
    if coefs is None:
        raise HoloError(ErrorCode.NULLPOINTER, "no coefficients to write")
    try:
        _interleave(coefs).tofile(path)
        _sidecar(path, [("batchCount", batch), ("modeCount", mode_count), ("polCount", pol),
                        ("format", "float32 interleaved (re, im), batch-major, pol-block-major (HH..VV)")])
    except OSError:
        raise HoloError(ErrorCode.FILENOTCREATED, str(path))
    return ErrorCode.SUCCESS


def read_coefs(path):
    meta = _read_sidecar(path)
    batch, modes, pol = int(meta["batchCount"]), int(meta["modeCount"]), int(meta["polCount"])
    raw = np.fromfile(path, dtype="<f4").reshape(batch, pol * modes, 2)
    return (raw[..., 0] + 1j * raw[..., 1]).astype(np.complex64)


def write_summary(handle, path):
    """Settings dump, result dimensions and one line per metric (all wavelength slots + average)."""
    coefs, batch, mode_count, pol = api.basis_get_coefs(handle)
    try:
        with open(path, "w") as fh:
            fh.write(serialise_settings(handle))
            fh.write(f"ResultBatchCount\t{batch}\n")
            fh.write(f"ResultModeCount\t{mode_count}\n")
            fh.write(f"ResultPolCount\t{pol}\n")
            for idx, name in enumerate(METRIC_NAMES):
                vals = api.auto_align_get_metrics(handle, idx)
                if vals is not None:
                    fh.write("\t".join([f"Metric.{name}"] + [repr(float(v)) for v in vals]) + "\n")
    except OSError:
        raise HoloError(ErrorCode.FILENOTCREATED, str(path))
    return ErrorCode.SUCCESS


def read_summary(path):
    """{key: [values as str]} of a summary (or settings) file."""
    out = {}
    with open(path) as fh:
        for line in fh:
            parts = line.rstrip("\n").split("\t")
            if parts and parts[0]:
                out[parts[0]] = parts[1:]
    return out
