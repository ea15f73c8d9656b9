"""ctypes binding of the C ABI in include/holo_b200.h (libholo_b200.so).

The library is built in-tree by ``paper_2204_02348_b200._build`` (nvcc,
sm_100a) and is the only compute path of the package: if it is missing or a
CUDA device is absent, every processing call raises -- there is no CPU
fallback.  Device buffers are torch tensors; only their raw pointers and the
current CUDA stream handle cross the boundary.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ErrorCode, HoloError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libholo_b200.so")

c_int32, c_int64, c_double, c_void_p, c_size_t = (ctypes.c_int32, ctypes.c_int64, ctypes.c_double,
                                                    ctypes.c_void_p, ctypes.c_size_t)

HPG_FLAG_SUMMARY = 1
HPG_FLAG_GENERIC = 2
HPG_FLAG_SIMT = 4
HPG_FLAG_TC = 8
HPG_FLAG_TC2 = 16
HPG_FLAG_SIMT_OVERLAP = 32

# Every symbol include/holo_b200.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "hpg_version", "hpg_plan_create", "hpg_plan_destroy", "hpg_plan_get_info", "hpg_plan_get_axes",
    "hpg_plan_get_basis", "hpg_workspace_size", "hpg_run", "hpg_finalize_summary",
    "hpg_fourier_full", "hpg_extract_coefs", "hpg_ref_calibration_finish", "hpg_metric_partials", "hpg_plane_summary",
    "hpg_plane_summary_workspace", "hpg_field_intensity", "hpg_upload_windows", "hpg_last_error",
    "hpg_last_launch_count", "hpg_coef_transform", "hpg_host_register", "hpg_host_unregister",
]


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("frame_width", c_int32), ("frame_height", c_int32), ("pol_count", c_int32),
        ("fft_nx", c_int32), ("fft_ny", c_int32), ("resolution_mode", c_int32),
        ("fill_factor", c_int32), ("group_count", c_int32), ("wavelength_count", c_int32),
        ("reserved", c_int32),
        ("pixel_size", c_double), ("wavelength_centre", c_double), ("window_radius_deg", c_double),
        ("wavelengths", ctypes.POINTER(c_double)),
        ("beam_centre", (c_double * 2) * 2), ("tilt_deg", (c_double * 2) * 2),
        ("removal_tilt_deg", (c_double * 2) * 2), ("removal_beam_centre", (c_double * 2) * 2),
        ("defocus", c_double * 2), ("waist", c_double * 2),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("wh", c_int32), ("ww", c_int32), ("gh", c_int32), ("gw", c_int32),
        ("col0", c_int32 * 2), ("row0", c_int32 * 2), ("mode_count", c_int32),
        ("k0", ((c_int32 * 2) * 16) * 2),
    ]


class Batch(ctypes.Structure):
    _fields_ = [
        ("frames", c_void_p), ("frame_format", c_int32), ("transpose", c_int32),
        ("frame_count", c_int64), ("batch_count", c_int32), ("avg_count", c_int32),
        ("members", c_void_p), ("wl_of_row", c_void_p),
        ("batch_cal", c_void_p), ("cal_pols", c_int32), ("cal_batch", c_int32),
        ("ref_cal", c_void_p), ("ref_cal_count", c_int32), ("row_offset", c_int32),
        ("layout_width", c_int32), ("layout_height", c_int32),
        ("layout_col0", c_int32 * 2), ("layout_row0", c_int32 * 2),
    ]


class Outputs(ctypes.Structure):
    _fields_ = [
        ("field_r", c_void_p), ("field_i", c_void_p), ("field_scale", c_void_p),
        ("coefs", c_void_p), ("raw_fields", c_void_p), ("windows", c_void_p),
        ("field_params", c_void_p), ("param_slots", c_int32), ("reserved", c_int32),
        ("workspace", c_void_p), ("workspace_bytes", c_size_t),
    ]


class MetricArgs(ctypes.Structure):
    _fields_ = [
        ("coefs", c_void_p), ("rows", c_int32), ("cols", c_int32),
        ("row_ids", c_void_p), ("col_offset", c_void_p), ("col_count", c_void_p),
        ("labels", c_void_p), ("ndiag", c_int32), ("diag_offset", c_int32),
        ("gram_rows", c_int32), ("ld", c_int32),
        ("row_power", c_void_p), ("diag_power", c_void_p), ("group_power", c_void_p),
        ("gram", c_void_p),
    ]


_lib = None


def lib():
    """The loaded library (raises HoloError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise HoloError(ErrorCode.ERROR,
                        f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    L.hpg_version.restype = c_int32
    L.hpg_last_launch_count.restype = c_int32
    L.hpg_last_error.restype = ctypes.c_char_p
    L.hpg_plan_create.argtypes = [P(PlanDesc), P(c_void_p)]
    L.hpg_plan_destroy.argtypes = [c_void_p]
    L.hpg_plan_get_info.argtypes = [c_void_p, P(PlanInfo)]
    L.hpg_plan_get_axes.argtypes = [c_void_p, c_void_p, c_void_p]
    L.hpg_plan_get_basis.argtypes = [c_void_p, c_void_p, c_void_p]
    L.hpg_workspace_size.argtypes = [c_void_p, c_int32, ctypes.c_uint32, P(c_size_t)]
    L.hpg_run.argtypes = [c_void_p, P(Batch), P(Outputs), ctypes.c_uint32, c_void_p]
    L.hpg_finalize_summary.argtypes = [c_void_p, P(Batch), P(Outputs), c_void_p, c_void_p]
    L.hpg_fourier_full.argtypes = [c_void_p, P(Batch), c_void_p, c_void_p, c_size_t, c_void_p]
    L.hpg_extract_coefs.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_void_p,
                                    c_void_p]
    L.hpg_metric_partials.argtypes = [P(MetricArgs), c_void_p]
    L.hpg_coef_transform.argtypes = [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_int32, c_int32, c_int32,
                                     c_int32, c_void_p, c_void_p]
    L.hpg_plane_summary.argtypes = [c_void_p, c_int64, c_int32, c_int32, c_int32, c_void_p, c_void_p,
                                    c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]
    L.hpg_field_intensity.argtypes = [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_int32, c_int32,
                                      c_void_p, c_void_p]
    L.hpg_plane_summary_workspace.argtypes = [c_int64, c_int32, c_int32, c_int32]
    L.hpg_ref_calibration_finish.argtypes = [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]
    L.hpg_upload_windows.argtypes = [c_void_p, c_void_p, c_int32, c_int64, c_void_p, c_void_p]
    L.hpg_host_register.argtypes = [c_void_p, c_size_t]
    L.hpg_host_unregister.argtypes = [c_void_p]
    for name in EXPORTS:
        getattr(L, name).restype = c_int32
    L.hpg_last_error.restype = ctypes.c_char_p
    L.hpg_plane_summary_workspace.restype = c_size_t
    _lib = L
    return L


def check(code, what=""):
    if code != 0:
        msg = lib().hpg_last_error()
        msg = msg.decode() if msg else ""
        raise HoloError(code, f"{what}: {msg}" if what else msg)


def ptr(t):
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_handle(device=None):
    """The current CUDA stream of ``device`` (default: the current device) as a void*.

    Uses torch's C binding directly: torch.cuda.current_stream() re-validates the
    device through NVML on every call, which costs ~0.1 ms per process_batch."""
    import torch
    if device is None:
        idx = torch.cuda.current_device()
    else:
        idx = device.index if getattr(device, "index", None) is not None else torch.cuda.current_device()
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(idx))


class Plan:
    """Owns one hpg_plan (constant device tables of one configuration)."""

    def __init__(self, desc: PlanDesc):
        self._lib = lib()
        h = c_void_p()
        check(self._lib.hpg_plan_create(ctypes.byref(desc), ctypes.byref(h)), "hpg_plan_create")
        self.handle = h
        info = PlanInfo()
        check(self._lib.hpg_plan_get_info(h, ctypes.byref(info)), "hpg_plan_get_info")
        self.info = info
        self.wh, self.ww, self.gh, self.gw = info.wh, info.ww, info.gh, info.gw
        self.mode_count = info.mode_count

    def axes(self):
        import numpy as np
        if getattr(self, "_axes", None) is None:   # constant per plan: read once, hand out copies
            x = np.empty(self.gw, np.float32)
            y = np.empty(self.gh, np.float32)
            check(self._lib.hpg_plan_get_axes(self.handle, x.ctypes.data_as(c_void_p),
                                              y.ctypes.data_as(c_void_p)))
            self._axes = (x, y)
        return self._axes[0].copy(), self._axes[1].copy()

    def basis(self, pol_count, group_count):
        import numpy as np
        hx = np.zeros((pol_count, max(group_count, 1), self.gw), np.float32)
        hy = np.zeros((pol_count, max(group_count, 1), self.gh), np.float32)
        check(self._lib.hpg_plan_get_basis(self.handle, hx.ctypes.data_as(c_void_p),
                                           hy.ctypes.data_as(c_void_p)))
        return hx[:, :group_count], hy[:, :group_count]

    def k0(self, pol, wl):
        return int(self.info.k0[pol][wl][0]), int(self.info.k0[pol][wl][1])

    def workspace_size(self, batch, flags):
        n = c_size_t()
        check(self._lib.hpg_workspace_size(self.handle, batch, flags, ctypes.byref(n)))
        return n.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.hpg_plan_destroy(h)
            except Exception:
                pass
            self.handle = None
