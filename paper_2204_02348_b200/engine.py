"""Engine: the GPU-resident counterpart of holopipe.engine.Engine.

Same staged methods and getters as the reference (holopipe/engine.py:45-541),
backed by the CUDA library (include/holo_b200.h):

  * ``run_pipeline(0)`` / ``process_batch`` is ONE fused kernel launch
    (hpg_run): frames -> int16 fields + scales + HG coefficients.
  * The staged entry points keep the reference's semantics: each stage
    snapshots the configuration it depends on (window origins at process_fft,
    carrier bins at process_ifft, removal phase at process_remove_tilt, basis
    at extract_coefs), and later stages re-use those snapshots, so
    ``run_pipeline(from_stage)`` gives the same products as the reference's
    partial re-runs.  Re-running from the frames is cheaper on the GPU than
    storing the reference's full-size intermediates, and the kernels are
    deterministic, so products are bit-identical to a full re-run.
  * Diagnostic products (full Fourier plane, Fourier-window bins, plane
    summaries) are produced on demand by their own kernels.

There is no CPU path: every numeric product comes from libholo_b200.so.
"""

from __future__ import annotations

import collections
import math
import ctypes

import numpy as np

from . import constants as C
from . import native
from .analysis import AnalysisSummary, MetricsReport, average_slot, finish_metrics, metrics_of_matrix
from .config import HoloConfig
from .errors import ErrorCode, HoloError
from .frames import CAL_INTENSITY, FrameSource, RefCalibration

_PLAN_CACHE = 8


def _torch():
    import torch
    return torch


def mode_indices(group_count):
    """Group-major (m, n), m descending within a group (holopipe/hgbasis.py:17-27)."""
    return [(g - n, n) for g in range(group_count) for n in range(g + 1)]


def mode_group_of_index(idx):
    g = 0
    while (g + 1) * (g + 2) // 2 <= idx:
        g += 1
    return g


def wavelength_reorder_indices(total, wavelength_count, ordering_in, ordering_out):
    """Permutation between wavelength-fast and -slow layouts (engine.py:22-34)."""
    if ordering_in == ordering_out or wavelength_count <= 1:
        return np.arange(total)
    if total % wavelength_count:
        raise HoloError(ErrorCode.INVALIDARGUMENT, "element count does not factor into wavelengths")
    idx = np.arange(total)
    rest = total // wavelength_count
    if ordering_in == C.WAVELENGTHORDER_FAST:
        return idx.reshape(rest, wavelength_count).T.reshape(-1)
    return idx.reshape(wavelength_count, rest).T.reshape(-1)


def apply_wavelength_ordering(data, wavelength_count, ordering_in, ordering_out):
    data = np.asarray(data)
    return data[wavelength_reorder_indices(data.shape[0], wavelength_count, ordering_in, ordering_out)]


class _Launch:
    """Prepared hpg_run arguments (kept alive with their tensors)."""

    def launch(self, stream=None):
        native.check(self.lib.hpg_run(self.plan.handle, self.bref, self.oref, self.flags,
                                      stream if stream is not None else native.stream_handle()), "hpg_run")


class Engine:
    def __init__(self, device=None):
        self.config = HoloConfig()
        self.source = FrameSource()
        self.ref_cal = RefCalibration()
        self.batch_cal = None
        self.batch_cal_enabled = 0
        self.custom_transform = None
        self.backup = None
        self.window_title = ""
        self.tweak_cycles = 0
        self._device = device
        self.force_generic = False      # diagnostic: bypass the specialised kernels
        self.force_simt = False         # diagnostic: specialised kernel without tensor cores
        self.use_tc = False             # tcgen05 row-pass kernel (HPG_FLAG_TC)
        self.use_tc2 = False            # two-kernel tensor-core path (HPG_FLAG_TC2)
        self.simt_overlap = False       # diagnostic: HG overlap on SIMT (HPG_FLAG_SIMT_OVERLAP)
        self.last_h2d_bytes = 0
        self._ref_applied = None        # processed reference calibration (engine.py:75)
        self._deferred = None           # host upload postponed by the pipelined process_batch
        self._plans = collections.OrderedDict()
        self._bufs = {}
        self._views = {}
        self._clear_products()

    # ------------------------------------------------------------ plumbing
    @property
    def device(self):
        if self._device is None:
            torch = _torch()
            if not torch.cuda.is_available():
                raise HoloError(ErrorCode.ERROR, "no CUDA device: the B200 path has no CPU fallback")
            self._device = torch.device("cuda", torch.cuda.current_device())
        return self._device

    def _buf(self, name, shape, dtype):
        """Device scratch `name` viewed as `shape` (grown on demand; views cached per shape)."""
        views = self._views.setdefault(name, {})
        v = views.get((shape, dtype))
        if v is not None:
            return v
        torch = _torch()
        t = self._bufs.get(name)
        n = math.prod(shape)
        if t is None or t.numel() < n or t.dtype != dtype:
            t = torch.empty(max(n, 1), dtype=dtype, device=self.device)
            self._bufs[name] = t
            views.clear()   # views of the previous allocation
        v = t[:n].view(*shape) if shape else t[:1]
        views[(shape, dtype)] = v
        return v

    def _clear_products(self):
        self._host_fields16 = None
        self._st0 = None
        self._st1 = None
        self._st2 = None
        self._st3 = None
        self._plan = None
        self._frames_dev = None
        self._fourier_full = None
        self._fourier_axes = None
        self._summary_fourier = None
        self._window = None
        self._window_meta = None
        self._field_axes = None
        self._field_r = None
        self._field_i = None
        self._field_scale = None
        self._summary_field = None
        self._coefs = None
        self._mode_count = 0
        self._metrics = None

    def _effective(self):
        """Tilt/defocus/waist with the polarisation locks applied (engine.py:79-92)."""
        cfg = self.config
        tilt = [list(cfg.tilt[0]), list(cfg.tilt[1])]
        defocus = list(cfg.defocus)
        waist = list(cfg.basisWaist)
        if cfg.polLockTilt:
            tilt[0][1] = tilt[0][0]
            tilt[1][1] = tilt[1][0]
        if cfg.polLockDefocus:
            defocus[1] = defocus[0]
        if cfg.polLockBasisWaist:
            waist[1] = waist[0]
        return tilt, defocus, waist

    def _batch_plan(self):
        """Averaging membership and wavelength per row (engine.py:94-120)."""
        cfg = self.config
        b, a = max(1, cfg.batchCount), max(1, cfg.avgCount)
        mode = cfg.avgMode if cfg.avgMode in (0, 1, 2) else C.AVGMODE_SEQUENTIAL
        lams = cfg.wavelength_list()
        L = len(lams)
        rows = np.arange(b)
        if cfg.wavelengthOrdering[C.WAVELENGTHORDER_INPUT] == C.WAVELENGTHORDER_FAST or L <= 1:
            wl = rows % L
        else:
            wl = np.minimum(rows * L // b, L - 1)
        av = np.arange(a)
        if mode == C.AVGMODE_INTERLACED:
            members = rows[:, None] + av[None, :] * b
        elif mode == C.AVGMODE_SEQUENTIALSWEEP and L > 1:
            members = ((rows // L) * a * L)[:, None] + av[None, :] * L + (rows % L)[:, None]
        else:
            members = rows[:, None] * a + av[None, :]
        return {"batch": b, "avg": a, "mode": mode, "lambdas": lams, "wl_of_batch": wl.astype(np.int64),
                "members": members.astype(np.int64), "frame_count": b * a}

    def output_permutation(self):
        plan = self._plan or self._batch_plan()
        lam = len(plan["lambdas"])
        if lam <= 1 or plan["batch"] % lam:
            return None   # identity
        cfg = self.config
        return wavelength_reorder_indices(plan["batch"], lam,
                                          cfg.wavelengthOrdering[C.WAVELENGTHORDER_INPUT],
                                          cfg.wavelengthOrdering[C.WAVELENGTHORDER_OUTPUT])

    # ------------------------------------------------------ native plans
    def _plan_key(self, group_count=None, waist=None):
        st0, st1, st2 = self._st0, self._st1, self._st2
        if st1 is None:   # stage-0 products only (full Fourier plane): window params are inert
            cfg = self.config
            st1 = {"tilt": [[0.0, 0.0], [0.0, 0.0]], "radius": float(cfg.fourierWindowRadius),
                   "lamc": float(cfg.wavelengthCentre), "fill": 0, "mode": 1}
        st2 = st2 or {"tilt": st1["tilt"], "centre": st0["centre"], "defocus": [0.0, 0.0]}
        if group_count is None:
            group_count = max(self.config.basisGroupCount, 0)
            waist = self._effective()[2]
        return (st0["W"], st0["H"], st0["P"], st0["nx"], st0["ny"], st1["mode"], st1["fill"],
                int(group_count), tuple(st0["lambdas"]), st0["pixel"], st1["lamc"], st1["radius"],
                tuple(map(tuple, st0["centre"])), tuple(map(tuple, st1["tilt"])),
                tuple(map(tuple, st2["tilt"])), tuple(map(tuple, st2["centre"])),
                tuple(st2["defocus"]), tuple(float(w) for w in waist))

    def _native_plan(self, key):
        plan = self._plans.get(key)
        if plan is not None:
            self._plans.move_to_end(key)
            return plan
        (W, H, P, nx, ny, mode, fill, G, lams, pix, lamc, radius, centre, tilt, rtilt, rcentre,
         defocus, waist) = key
        d = native.PlanDesc()
        d.frame_width, d.frame_height, d.pol_count = W, H, P
        d.fft_nx, d.fft_ny = nx, ny
        d.resolution_mode, d.fill_factor, d.group_count = mode, fill, G
        d.wavelength_count = len(lams)
        wl = (ctypes.c_double * len(lams))(*lams)
        d.wavelengths = ctypes.cast(wl, ctypes.POINTER(ctypes.c_double))
        d.pixel_size, d.wavelength_centre, d.window_radius_deg = pix, lamc, radius
        for a in range(2):
            for q in range(2):
                d.beam_centre[a][q] = centre[a][q]
                d.tilt_deg[a][q] = tilt[a][q]
                d.removal_tilt_deg[a][q] = rtilt[a][q]
                d.removal_beam_centre[a][q] = rcentre[a][q]
        for q in range(2):
            d.defocus[q] = defocus[q]
            d.waist[q] = waist[q] if waist[q] > 0 else -1.0
        if len(lams) > 16:
            raise HoloError(ErrorCode.INVALIDARGUMENT, "at most 16 wavelengths per batch")
        with _torch().cuda.device(self.device):
            plan = native.Plan(d)
        self._plans[key] = plan
        if len(self._plans) > _PLAN_CACHE:
            self._plans.popitem(last=False)
        return plan

    # ------------------------------------------------------------ stages
    def process_fft(self, _defer_upload=False):
        """Stage 0: window origins + frame staging (engine.py:135-168).

        The full R2C plane and its summary are produced on demand
        (get_fourier_plane_full / batch_summary(PLANE_FOURIER))."""
        cfg = self.config
        plan = self._batch_plan()
        nx, ny = cfg.fftWindowSizeX, cfg.fftWindowSizeY
        for q in range(cfg.polCount):   # origin validation (pipeline.py:35-37)
            lo, hi = (0, cfg.frameWidth) if cfg.polCount == 1 else \
                ((0, cfg.frameWidth // 2) if q == 0 else (cfg.frameWidth // 2, cfg.frameWidth))
            if nx > hi - lo or ny > cfg.frameHeight:
                raise HoloError(ErrorCode.INVALIDDIMENSION, "fft window does not fit the frame region")
        self._clear_products()
        self._plan = plan
        self._st0 = {"W": cfg.frameWidth, "H": cfg.frameHeight, "P": cfg.polCount, "nx": nx, "ny": ny,
                     "pixel": float(cfg.framePixelSize), "lambdas": [float(v) for v in plan["lambdas"]],
                     "centre": [list(map(float, cfg.beamCentre[0][:2])), list(map(float, cfg.beamCentre[1][:2]))]}
        self._frames_dev = self._stage_frames(plan["frame_count"], defer=_defer_upload)
        self._fourier_axes_key = (nx, ny, float(cfg.framePixelSize), float(cfg.wavelengthCentre))
        self._fourier_axes_f64 = None   # built on first use (Fourier-plane products only)
        return ErrorCode.SUCCESS

    def _fourier_axes_pair(self):
        """Fourier-plane angle axes of stage 0 (engine.py:157-161), fp64 and float32."""
        if self._fourier_axes_f64 is None:
            from .geometry import fourier_angle_axis
            nx, ny, p, lam0 = self._fourier_axes_key
            fx = fourier_angle_axis(np.arange(nx // 2 + 1), nx, p, lam0)
            fy = fourier_angle_axis(np.fft.fftfreq(ny) * ny, ny, p, lam0)
            self._fourier_axes_f64 = (fx, fy)
            self._fourier_axes = (fx.astype(np.float32), fy.astype(np.float32))
        return self._fourier_axes_f64

    def _stage_frames(self, F, defer=False):
        """Device copy of the frames the pipeline reads: (tensor, fmt, transpose, layout).

        Host sources (numpy / CPU tensors) are uploaded window-only
        (hpg_upload_windows: one 3-D copy per pol, packed [F][ny][P*nx]);
        device sources are used in place."""
        cfg = self.config
        src = self.source
        host = src.host_array() if src._pinned is None else None
        if host is not None and not (src.format() == 1 and src.transpose):
            torch = _torch()
            with torch.cuda.device(self.device):
                src.ensure_registered()   # pageable numpy sources: page-locked in place, once per buffer
            st0 = self._st0
            fmt = src.format()
            need = F * st0["W"] * st0["H"]
            n = host.numel() if hasattr(host, "numel") else host.size
            if n < need:
                raise HoloError(ErrorCode.INVALIDDIMENSION, f"frame buffer holds {n} pixels, need {need}")
            plan0 = self._native_plan(self._plan_key(0, (1.0, 1.0)))
            P, nx, ny = st0["P"], st0["nx"], st0["ny"]
            packed = self._buf("packed", (F, ny, P * nx), torch.float32 if fmt == 0 else torch.int16)
            ptr = host.data_ptr() if hasattr(host, "data_ptr") else host.ctypes.data
            self._deferred = (plan0, ptr, fmt, F) if defer else None
            if not defer:
                with torch.cuda.device(self.device):
                    native.check(native.lib().hpg_upload_windows(plan0.handle, ctypes.c_void_p(ptr), fmt, F,
                                                                 native.ptr(packed), native.stream_handle()),
                                 "hpg_upload_windows")
            layout = (P * nx, ny, [q * nx for q in range(P)], [0, 0])
            self.last_h2d_bytes = packed.numel() * packed.element_size()
            return packed, fmt, 0, layout
        frames, fmt, tr = src.staged(F, cfg.frameWidth, cfg.frameHeight, self.device)
        self.last_h2d_bytes = 0 if host is None else frames.numel() * frames.element_size()
        return frames, fmt, tr, None

    def _batch_frames(self, b):
        """Fill the frame fields (and layout override) of an hpg_batch."""
        frames, fmt, tr, layout = self._frames_dev
        b.frames = frames.data_ptr()
        b.frame_format, b.transpose = fmt, tr
        if layout is not None:
            b.layout_width, b.layout_height = layout[0], layout[1]
            for q in range(2):
                b.layout_col0[q] = layout[2][q] if q < len(layout[2]) else 0
                b.layout_row0[q] = layout[3][q]
            b.frame_count = frames.numel() // (layout[0] * layout[1])
        else:
            b.frame_count = frames.numel() // (self._st0["W"] * self._st0["H"])

    def process_ifft(self, _next_plan=False):
        """Stage 1: carrier bins, window, IFFT grid (engine.py:170-220).

        ``_next_plan`` (run_pipeline): take the stage-1 products from the plan the fused launch that
        follows will use (same k0, window and axes), so a restart builds one plan instead of two."""
        if self._st0 is None:
            raise HoloError(ErrorCode.NULLPOINTER, "FFT stage has not run")
        cfg = self.config
        tilt, _, _ = self._effective()
        self._st1 = {"tilt": [list(map(float, tilt[0])), list(map(float, tilt[1]))],
                     "radius": float(cfg.fourierWindowRadius), "lamc": float(cfg.wavelengthCentre),
                     "fill": int(bool(cfg.fillFactorCorrectionEnabled)), "mode": int(cfg.resolutionMode)}
        self._st2 = self._st3 = None
        self._window = None
        self._field_r = self._field_i = self._field_scale = None
        self._host_fields16 = None
        self._summary_field = None
        self._coefs = None
        if _next_plan:
            self._st2 = self._stage2_snapshot()
            G = max(cfg.basisGroupCount, 0)
            key = self._plan_key(G, self._effective()[2]) if G >= 1 else self._plan_key(0, (1.0, 1.0))
            self._st2 = None
        else:
            key = self._plan_key(0, (1.0, 1.0))
        plan = self._native_plan(key)
        self._field_axes = plan.axes()
        k0 = np.zeros((self._plan["batch"], self._st0["P"], 2), np.int64)
        for q in range(self._st0["P"]):
            for w in range(len(self._st0["lambdas"])):
                k0[self._plan["wl_of_batch"] == w, q] = plan.k0(q, w)
        self._window_meta = {"wh": plan.wh, "ww": plan.ww, "k0": k0}
        if self.ref_cal.enabled and self.ref_cal.kind:
            self._process_ref_calibration()
        return ErrorCode.SUCCESS

    def _process_ref_calibration(self):
        """Reference-wave calibration -> applied correction (engine.py:276-335), on the GPU.

        The calibration windows run through the same fused kernel as the frames:
        * intensity: sqrt(normalised intensity) with the carrier at DC (k0 = 0), no
          removal phase -- a plan with zero tilt / defocus reproduces exactly
          forward_fft -> fill_window_r2c(0, 0) -> mask * recentring -> inverse_fft;
        * field: conj(raw) = a + i b with a = Re raw, b = -Im raw; every step after the
          C2C transform is linear, so proc = chain(a) + i chain(b) with the r2c window
          sampling of each real part equal to fill_window_c2c of the complex spectrum
          (no fill-factor envelope on this path, engine.py:314-316), removal phase at
          the configured tilt / defocus / beam centre.
        hpg_ref_calibration_finish then forms conj(proc) / max(|proc|^2, 1e-6)."""
        torch = _torch()
        cal = self.ref_cal
        inten = cal.normalised_intensity()
        if inten is None:
            return
        st0, st1, cfg = self._st0, self._st1, self.config
        if inten.shape[1] != st0["H"] or inten.shape[2] != st0["W"]:
            raise HoloError(ErrorCode.INVALIDARGUMENT, "calibration dimensions do not match the frames")
        tilt, defocus, _ = self._effective()
        Lc, L, P = cal.wavelength_count, len(st0["lambdas"]), st0["P"]
        centre = tuple(map(tuple, st0["centre"]))
        if cal.kind == CAL_INTENSITY:
            frames = np.sqrt(inten).astype(np.float32)
            zero = ((0.0, 0.0), (0.0, 0.0))
            key = (st0["W"], st0["H"], P, st0["nx"], st0["ny"], st1["mode"], st1["fill"], 0, tuple(st0["lambdas"]),
                   st0["pixel"], st1["lamc"], st1["radius"], centre, zero, zero, centre, (0.0, 0.0), (1.0, 1.0))
            wl_rows = None
        else:
            raw = cal.raw
            frames = np.concatenate([raw.real, -raw.imag]).astype(np.float32)
            tl = tuple(tuple(float(v) for v in tilt[a][:2]) for a in range(2))
            rcentre = tuple(tuple(float(v) for v in cfg.beamCentre[a][:2]) for a in range(2))
            key = (st0["W"], st0["H"], P, st0["nx"], st0["ny"], st1["mode"], 0, 0, tuple(st0["lambdas"]),
                   st0["pixel"], st1["lamc"], st1["radius"], centre, tl, tl, rcentre,
                   (float(defocus[0]), float(defocus[1])), (1.0, 1.0))
            wl_rows = [min(ci, L - 1) for ci in range(Lc)] * 2
        plan = self._native_plan(key)
        B = frames.shape[0]
        gh, gw = plan.gh, plan.gw
        dev = self.device
        with torch.cuda.device(dev):
            fr_dev = torch.from_numpy(np.ascontiguousarray(frames)).to(dev)
            raw_out = torch.empty((B, P, gh, gw), dtype=torch.complex64, device=dev)
            fr16 = torch.empty((B, P, gh, gw), dtype=torch.int16, device=dev)
            fi16 = torch.empty_like(fr16)
            sc = torch.empty((B, P), dtype=torch.float32, device=dev)
            ws_bytes = plan.workspace_size(B, 0)
            ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
            b = native.Batch()
            b.frames, b.frame_format, b.transpose = fr_dev.data_ptr(), 0, 0
            b.frame_count, b.batch_count, b.avg_count = B, B, 1
            keep = [fr_dev]
            if wl_rows is not None and L > 1:
                wl = torch.as_tensor(np.asarray(wl_rows, np.int32), device=dev)
                b.wl_of_row = wl.data_ptr()
                keep.append(wl)
            o = native.Outputs()
            o.field_r, o.field_i, o.field_scale = fr16.data_ptr(), fi16.data_ptr(), sc.data_ptr()
            o.raw_fields = raw_out.data_ptr()
            o.workspace, o.workspace_bytes = ws.data_ptr(), ws_bytes
            lib = native.lib()
            native.check(lib.hpg_run(plan.handle, ctypes.byref(b), ctypes.byref(o), 0, native.stream_handle()),
                         "hpg_run (reference calibration)")
            applied = torch.empty((Lc, P, gh, gw), dtype=torch.complex64, device=dev)
            second = raw_out[Lc:].data_ptr() if wl_rows is not None else None
            native.check(lib.hpg_ref_calibration_finish(raw_out[:Lc].data_ptr(), second, Lc * P * gh * gw,
                                                        applied.data_ptr(), native.stream_handle()),
                         "hpg_ref_calibration_finish")
        self._ref_applied = applied

    def process_remove_tilt(self):
        """Stage 2: removal phase, calibrations, int16 packing (engine.py:222-274)."""
        if self._st1 is None:
            raise HoloError(ErrorCode.NULLPOINTER, "IFFT stage has not run")
        self._st2 = self._stage2_snapshot()
        self._st3 = None
        self._coefs = None
        self._run_fused(with_coefs=False)
        return ErrorCode.SUCCESS

    def _stage2_snapshot(self):
        """What process_remove_tilt depends on (engine.py:226-255)."""
        cfg = self.config
        tilt, defocus, _ = self._effective()
        rcal = None
        if self.ref_cal.enabled and self.ref_cal.kind and self._ref_applied is not None:
            rcal = self._ref_applied
        return {"tilt": [list(map(float, tilt[0])), list(map(float, tilt[1]))],
                "centre": [list(map(float, cfg.beamCentre[0][:2])), list(map(float, cfg.beamCentre[1][:2]))],
                "defocus": [float(defocus[0]), float(defocus[1])],
                "bcal": self.batch_cal.copy() if (self.batch_cal_enabled and self.batch_cal is not None) else None,
                "rcal": rcal}

    def extract_coefs(self):
        """Stage 3: separable HG overlap of the int16 fields (engine.py:353-385)."""
        cfg = self.config
        if cfg.basisGroupCount < 1:
            self._coefs = None
            self._mode_count = 0
            return ErrorCode.SUCCESS
        if self._field_r is None:
            raise HoloError(ErrorCode.NULLPOINTER, "tilt-removal stage has not run")
        G = cfg.basisGroupCount
        waist = self._effective()[2]
        plan = self._native_plan(self._plan_key(G, waist))
        B, P = self._plan["batch"], self._st0["P"]
        M = plan.mode_count
        hg = self._buf("coefs", (B, P * M), _torch().complex64)
        with _torch().cuda.device(self.device):
            native.check(native.lib().hpg_extract_coefs(
                plan.handle, native.ptr(self._field_r), native.ptr(self._field_i),
                native.ptr(self._field_scale), B, native.ptr(hg), native.stream_handle()),
                "hpg_extract_coefs")
        self._finish_coefs(hg, M, P)
        return ErrorCode.SUCCESS

    def _finish_coefs(self, hg, M, P):
        """Optional LG / custom transform (engine.py:371-384), on the GPU (hpg_coef_transform, fp64
        accumulation like the reference's complex128 einsum)."""
        cfg = self.config
        torch = _torch()
        B = hg.shape[0]
        transform, block = None, 0
        if cfg.basisType == C.BASISTYPE_LG:
            key = ("lg", cfg.basisGroupCount)
            cached = self._bufs.get("lg_T")
            if cached is None or cached[0] != key:
                from .hgbasis import hg_to_lg_transform
                T = np.ascontiguousarray(np.conj(hg_to_lg_transform(cfg.basisGroupCount)))
                cached = (key, torch.as_tensor(T, dtype=torch.complex128, device=self.device))
                self._bufs["lg_T"] = cached
            transform, block = cached[1], 1
        elif cfg.basisType == C.BASISTYPE_CUSTOM and self.custom_transform is not None:
            transform = torch.as_tensor(np.ascontiguousarray(self.custom_transform), dtype=torch.complex128,
                                        device=self.device)
        if transform is not None:
            m_out, ld = transform.shape
            use = min(M, ld)
            out = self._buf("coefs_t", (B, P * m_out), torch.complex64)
            with torch.cuda.device(self.device):
                native.check(native.lib().hpg_coef_transform(native.ptr(hg), B, P, M, native.ptr(transform), m_out,
                                                             use, ld, block, native.ptr(out),
                                                             native.stream_handle()), "hpg_coef_transform")
            self._mode_count = m_out
            self._coefs = out
        else:
            self._mode_count = M
            self._coefs = hg
        self._metrics = None

    def _prepare_fused(self, with_coefs, summary=False, windows=False):
        """Build the hpg_run arguments for the current stage snapshots (no launch)."""
        torch = _torch()
        st0 = self._st0
        cfg = self.config
        G = max(cfg.basisGroupCount, 0) if with_coefs else 0
        waist = self._effective()[2] if with_coefs else (1.0, 1.0)
        key = self._plan_key(G, waist) if (with_coefs and G > 0) else self._plan_key(0, (1.0, 1.0))
        plan = self._native_plan(key)
        B, A, P = self._plan["batch"], self._plan["avg"], st0["P"]
        gh, gw = plan.gh, plan.gw
        L = _Launch()
        L.plan, L.G, L.waist = plan, G, waist
        L.fr = self._buf("fr", (B, P, gh, gw), torch.int16)
        L.fi = self._buf("fi", (B, P, gh, gw), torch.int16)
        L.sc = self._buf("scale", (B, P), torch.float32)
        L.coefs = self._buf("coefs", (B, P * plan.mode_count), torch.complex64) if (with_coefs and G > 0) else None
        L.flags = ((native.HPG_FLAG_SUMMARY if summary else 0) | (native.HPG_FLAG_GENERIC if self.force_generic else 0)
                   | (native.HPG_FLAG_SIMT if self.force_simt else 0) | (native.HPG_FLAG_TC if self.use_tc else 0)
                   | (native.HPG_FLAG_TC2 if self.use_tc2 else 0)
                   | (native.HPG_FLAG_SIMT_OVERLAP if self.simt_overlap else 0))
        L.params = L.inten = None
        slots = B * A + 1
        if summary:
            L.params = torch.zeros((C.ANALYSIS_COUNT, P, slots), dtype=torch.float32, device=self.device)
            L.inten = torch.zeros((gh, gw), dtype=torch.float32, device=self.device)
        L.win = torch.empty((B, P, plan.wh, plan.ww), dtype=torch.complex64, device=self.device) if windows else None
        ws_bytes = plan.workspace_size(B, L.flags)
        ws = self._buf("ws", (ws_bytes,), torch.uint8)
        b = native.Batch()
        self._batch_frames(b)
        b.batch_count, b.avg_count = B, A
        L.keep = [self._frames_dev[0], ws]
        if A > 1 or self._plan["mode"] != C.AVGMODE_SEQUENTIAL:
            members = torch.as_tensor(self._plan["members"].reshape(-1).astype(np.int32), device=self.device)
            b.members = members.data_ptr()
            L.keep.append(members)
        if len(self._plan["lambdas"]) > 1:
            wl = torch.as_tensor(self._plan["wl_of_batch"].astype(np.int32), device=self.device)
            b.wl_of_row = wl.data_ptr()
            L.keep.append(wl)
        if self._st2 is not None and self._st2.get("bcal") is not None:
            cal = self._st2["bcal"]
            bcal = torch.as_tensor(np.ascontiguousarray(cal, dtype=np.complex64), device=self.device)
            b.batch_cal = bcal.data_ptr()
            b.cal_pols, b.cal_batch = cal.shape
            L.keep.append(bcal)
        if self._st2 is not None and self._st2.get("rcal") is not None:
            rcal = self._st2["rcal"]
            b.ref_cal, b.ref_cal_count = rcal.data_ptr(), rcal.shape[0]
            L.keep.append(rcal)
        o = native.Outputs()
        o.field_r, o.field_i, o.field_scale = L.fr.data_ptr(), L.fi.data_ptr(), L.sc.data_ptr()
        o.coefs = L.coefs.data_ptr() if L.coefs is not None else None
        o.windows = L.win.data_ptr() if L.win is not None else None
        o.field_params = L.params.data_ptr() if L.params is not None else None
        o.param_slots = slots
        o.workspace, o.workspace_bytes = ws.data_ptr(), ws_bytes
        L.batch, L.out, L.device = b, o, self.device
        L.lib = native.lib()
        L.bref, L.oref = ctypes.byref(b), ctypes.byref(o)
        return L

    def prepare_launch(self):
        """The fused launch of the current configuration as a cheap re-launchable object.

        ``launch()`` issues exactly one hpg_run on the current stream (used by
        bench.py to time the kernel without Python engine overhead)."""
        if self._st0 is None or self._st1 is None:
            self.run_pipeline(0)
        return self._prepare_fused(with_coefs=self.config.basisGroupCount >= 1)

    def _run_fused(self, with_coefs, summary=False, windows=False):
        """One hpg_run launch with the current stage snapshots."""
        torch = _torch()
        L = self._prepare_fused(with_coefs, summary, windows)
        with torch.cuda.device(self.device):
            L.launch()
            if summary:
                native.check(L.lib.hpg_finalize_summary(L.plan.handle, L.bref, L.oref, native.ptr(L.inten),
                                                        native.stream_handle()), "hpg_finalize_summary")
        self._field_r, self._field_i, self._field_scale = L.fr, L.fi, L.sc
        self._host_fields16 = None
        self._field_axes = L.plan.axes()
        if summary:
            self._summary_field = (L.params, L.inten)
        if windows:
            self._window = L.win
        if with_coefs and L.G > 0:
            self._st3 = {"G": L.G, "waist": tuple(L.waist)}
            self._finish_coefs(L.coefs, L.plan.mode_count, self._st0["P"])
        return L.plan

    # -------------------------------------------------------- top level
    def run_pipeline(self, from_stage=0):
        """Stages from ``from_stage`` (0 fft, 1 ifft, 2 tilt, 3 coefs), engine.py:389-402."""
        if from_stage <= 0 or self._st0 is None:
            self.process_fft()
        if from_stage <= 1 or self._st1 is None:
            self.process_ifft(_next_plan=True)
        if from_stage <= 2 or self._field_r is None:
            self._st2 = self._stage2_snapshot()
            self._summary_field = None
            self._window = None
            if self.config.basisGroupCount >= 1:
                self._run_fused(with_coefs=True)
                return
            self._run_fused(with_coefs=False)
            self._coefs = None
            self._mode_count = 0
            return
        self.extract_coefs()

    def process_batch(self):
        """run_pipeline(0) + coef_view (engine.py:404-417).

        For host frames the upload, the fused kernel and the coefficient readback
        are pipelined in chunks of rows (copy stream / compute stream), which is
        the same computation on the same rows -- rows are independent."""
        if self._pipeline_ok():
            return self._process_batch_pipelined()
        self.run_pipeline(0)
        return self.coef_view()

    # chunk count: HOLO_PIPE_CHUNKS if set, else one chunk per ~48 MB of window upload, 4..16
    # (B200 sweep, profiles/r1s3_pipe_chunks.txt: dual-pol 131 MB flat over 2..16 chunks, PCIe-bound;
    # large basis 537 MB + 68 MB coefficient readback 464 K frames/s at 4 chunks -> 563 K at 12)
    _PIPE_CHUNKS_ENV = int(__import__("os").environ.get("HOLO_PIPE_CHUNKS", "0"))
    _PIPE_CHUNKS = _PIPE_CHUNKS_ENV or 4       # minimum used by the eligibility check
    _PIPE_CHUNK_BYTES = 48 << 20

    def _pipe_chunks(self, B, upload_bytes):
        if self._PIPE_CHUNKS_ENV:
            return self._PIPE_CHUNKS_ENV
        n = -(-upload_bytes // self._PIPE_CHUNK_BYTES)
        return int(max(self._PIPE_CHUNKS, min(16, n, B // 8)))

    def _pipeline_ok(self):
        cfg, src = self.config, self.source
        host = src.host_array() if src._pinned is None else None
        return (host is not None and not (src.format() == 1 and src.transpose)
                and max(1, cfg.avgCount) == 1 and (cfg.basisGroupCount < 1 or cfg.basisType == C.BASISTYPE_HG)
                and max(1, cfg.batchCount) >= 8 * self._PIPE_CHUNKS
                and not (self.force_generic or self.force_simt))

    def _process_batch_pipelined(self):
        torch = _torch()
        self.process_fft(_defer_upload=True)
        plan0, hptr, fmt, F = self._deferred
        self._deferred = None
        B, P = self._plan["batch"], self._st0["P"]
        W, H, nx, ny = self._st0["W"], self._st0["H"], self._st0["nx"], self._st0["ny"]
        es = 4 if fmt == 0 else 2
        packed = self._frames_dev[0]
        dev = self.device
        lib = native.lib()
        nchunks = self._pipe_chunks(B, B * ny * P * nx * es)
        bounds = np.linspace(0, B, nchunks + 1).astype(int)
        arrived = []   # (r0, r1, event): coefficient rows of a chunk are in host_out
        with torch.cuda.device(dev):
            comp = torch.cuda.current_stream(dev)
            copy, back = self._bufs.get("copy_stream"), self._bufs.get("back_stream")
            if copy is None:
                copy, back = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
                self._bufs["copy_stream"], self._bufs["back_stream"] = copy, back
            copy.wait_stream(comp)   # buffers of the previous call are free
            back.wait_stream(comp)
            cs = ctypes.c_void_p(copy.cuda_stream)
            ups = []
            for c in range(nchunks):   # every upload queued first: host work below overlaps them
                r0, r1 = int(bounds[c]), int(bounds[c + 1])
                if r1 > r0:
                    native.check(lib.hpg_upload_windows(plan0.handle, ctypes.c_void_p(hptr + r0 * W * H * es), fmt,
                                                        r1 - r0,
                                                        ctypes.c_void_p(packed.data_ptr() + r0 * ny * P * nx * es),
                                                        cs), "hpg_upload_windows")
                ev = torch.cuda.Event()
                ev.record(copy)
                ups.append(ev)
        try:
            self.process_ifft()
            self._st2 = self._stage2_snapshot()
            with_coefs = self.config.basisGroupCount >= 1
            L = self._prepare_fused(with_coefs=with_coefs)
            M = L.plan.mode_count if with_coefs else 0
            hw = L.fr.shape[-1] * L.fr.shape[-2]
            # the step's result read back chunk by chunk: coefficients, or the int16 fields + scales (no basis)
            per_row = P * M * 8 if with_coefs else P * (2 * hw * 2 + 4)
            host_out = self._bufs.get("result_host")
            if host_out is None or host_out.numel() < B * per_row:
                host_out = torch.empty(B * per_row, dtype=torch.uint8).pin_memory()
                self._bufs["result_host"] = host_out
            if with_coefs:
                hc = host_out[:B * P * M * 8].view(torch.complex64)
            else:
                hfr = host_out[:B * P * hw * 2].view(torch.int16)
                hfi = host_out[B * P * hw * 2:2 * B * P * hw * 2].view(torch.int16)
                hsc = host_out[2 * B * P * hw * 2:2 * B * P * hw * 2 + B * P * 4].view(torch.float32)
            with torch.cuda.device(dev):
                ks = ctypes.c_void_p(comp.cuda_stream)
                wl = L.batch.wl_of_row
                for c in range(nchunks):
                    r0, r1 = int(bounds[c]), int(bounds[c + 1])
                    n = r1 - r0
                    if n == 0:
                        continue
                    comp.wait_event(ups[c])
                    b = type(L.batch).from_buffer_copy(L.batch)
                    o = type(L.out).from_buffer_copy(L.out)
                    b.frames = packed.data_ptr() + r0 * ny * P * nx * es
                    b.frame_count = b.batch_count = n
                    b.row_offset = L.batch.row_offset + r0   # batch calibration follows the global row
                    if wl:
                        b.wl_of_row = wl + r0 * 4
                    o.field_r = L.fr.data_ptr() + r0 * P * hw * 2
                    o.field_i = L.fi.data_ptr() + r0 * P * hw * 2
                    o.field_scale = L.sc.data_ptr() + r0 * P * 4
                    if with_coefs:
                        o.coefs = L.coefs.data_ptr() + r0 * P * M * 8
                    native.check(lib.hpg_run(L.plan.handle, ctypes.byref(b), ctypes.byref(o), L.flags, ks), "hpg_run")
                    done = torch.cuda.Event()
                    done.record(comp)
                    back.wait_event(done)   # readback on its own stream: uploads keep streaming
                    with torch.cuda.stream(back):
                        if with_coefs:
                            hc[r0 * P * M:r1 * P * M].copy_(L.coefs.view(-1)[r0 * P * M:r1 * P * M], non_blocking=True)
                        else:
                            hfr[r0 * P * hw:r1 * P * hw].copy_(L.fr.view(-1)[r0 * P * hw:r1 * P * hw], non_blocking=True)
                            hfi[r0 * P * hw:r1 * P * hw].copy_(L.fi.view(-1)[r0 * P * hw:r1 * P * hw], non_blocking=True)
                            hsc[r0 * P:r1 * P].copy_(L.sc.view(-1)[r0 * P:r1 * P], non_blocking=True)
                    got = torch.cuda.Event()
                    got.record(back)
                    arrived.append((r0, r1, got))
                fin = torch.cuda.Event()
                fin.record(back)
                comp.wait_stream(copy)
                comp.wait_stream(back)
            self.last_h2d_bytes = packed.numel() * packed.element_size()
            self._field_r, self._field_i, self._field_scale = L.fr, L.fi, L.sc
            self._field_axes = L.plan.axes()
            if not with_coefs:   # fields-only configuration: the int16 fields are the step's result
                gh, gw = L.fr.shape[-2:]
                out_fr = np.empty((B, P, gh, gw), np.int16)
                out_fi = np.empty((B, P, gh, gw), np.int16)
                out_sc = np.empty((B, P), np.float32)
                sfr, sfi = hfr.numpy().reshape(B, P, gh, gw), hfi.numpy().reshape(B, P, gh, gw)
                ssc = hsc.numpy().reshape(B, P)
                for r0, r1, got in arrived:   # copy-out chunk by chunk as each readback lands
                    got.synchronize()
                    out_fr[r0:r1], out_fi[r0:r1], out_sc[r0:r1] = sfr[r0:r1], sfi[r0:r1], ssc[r0:r1]
                fin.synchronize()
                self._coefs = None
                self._mode_count = 0
                self._host_fields16 = (out_fr, out_fi, out_sc)   # handed out by the next get_fields16
                return None, B, 0, P
            self._st3 = {"G": L.G, "waist": tuple(L.waist)}
            self._finish_coefs(L.coefs, M, P)
            # copy-out (engine.py:416) chunk by chunk as each readback lands, while later chunks still stream
            staged = hc.numpy().reshape(B, P * M)
            coefs = np.empty((B, P * M), np.complex64)
            for r0, r1, got in arrived:
                got.synchronize()
                coefs[r0:r1] = staged[r0:r1]
            fin.synchronize()
            perm = self.output_permutation()
            return (coefs if perm is None else coefs[perm]), B, self._mode_count, P
        except BaseException:
            # a failure after the uploads were queued: the compute stream must not run ahead of
            # the in-flight copies into `packed`, and no half-made product may survive
            with torch.cuda.device(dev):
                comp.wait_stream(copy)
                comp.wait_stream(back)
            self._clear_products()
            raise

    def coef_view(self):
        plan = self._plan
        if plan is None or self._coefs is None:
            if self.config.basisGroupCount < 1 and plan is not None:
                return None, plan["batch"], 0, self.config.polCount
            return None, 0, 0, 0
        perm = self.output_permutation()
        coefs = self._coefs.cpu().numpy()   # a fresh host array (copy-out, engine.py:416)
        return (coefs if perm is None else coefs[perm]), plan["batch"], self._mode_count, self._st0["P"]

    def coefs_device(self):
        """Coefficients as a CUDA tensor (input row order), no host copy."""
        return self._coefs

    def process_batch_frequency_sweep_linear(self, lambda_start, lambda_stop, lambda_count):
        if lambda_count < 1 or lambda_start <= 0 or lambda_stop <= 0:
            raise HoloError(ErrorCode.INVALIDDIMENSION, "invalid wavelength sweep")
        if lambda_count == 1:
            lams = [float(lambda_start)]
        else:
            f0, f1 = 1.0 / lambda_start, 1.0 / lambda_stop
            lams = list(1.0 / (f0 + np.arange(lambda_count) * (f1 - f0) / (lambda_count - 1)))
        self.config.wavelengths = lams
        return self.process_batch()

    def process_batch_wavelength_sweep_arbitrary(self, wavelengths, lambda_count):
        if wavelengths is None:
            raise HoloError(ErrorCode.NULLPOINTER, "wavelengths is null")
        lams = [float(v) for v in np.asarray(wavelengths).reshape(-1)[:lambda_count]]
        if lambda_count < 1 or len(lams) < lambda_count:
            raise HoloError(ErrorCode.INVALIDDIMENSION, "invalid wavelength count")
        self.config.wavelengths = lams
        return self.process_batch()

    # ------------------------------------------------------------ getters
    def get_fields16(self):
        if self._field_r is None:
            raise HoloError(ErrorCode.NULLPOINTER, "no processed fields")
        perm = self.output_permutation()
        x_axis, y_axis = self._field_axes
        staged, self._host_fields16 = getattr(self, "_host_fields16", None), None
        if staged is not None:   # fresh host arrays the pipelined process_batch already read back
            fr, fi, sc = staged
        else:
            fr, fi, sc = (t.cpu().numpy() for t in (self._field_r, self._field_i, self._field_scale))
        if perm is not None:
            fr, fi, sc = fr[perm], fi[perm], sc[perm]
        return (fr, fi, sc, x_axis, y_axis, x_axis.size, y_axis.size, self._plan["batch"], self._st0["P"])

    def get_fields(self):
        fr, fi, scale, x_axis, y_axis, width, height, b, pol = self.get_fields16()
        fields = (fr.astype(np.float32) + 1j * fi.astype(np.float32))
        fields /= scale[:, :, None, None]
        return fields.astype(np.complex64), b, pol, x_axis, y_axis, width, height

    def fields16_device(self):
        return self._field_r, self._field_i, self._field_scale

    def _fourier_plane_device(self):
        if self._fourier_full is None:
            torch = _torch()
            st0 = self._st0
            plan = self._native_plan(self._plan_key(0, (1.0, 1.0)))
            F = self._plan["frame_count"]
            P, ny, nh = st0["P"], st0["ny"], st0["nx"] // 2 + 1
            plane = torch.empty((F, P, ny, nh), dtype=torch.complex64, device=self.device)
            ws_bytes = plan.workspace_size(max(F, 1), 0)
            ws = self._buf("ws", (ws_bytes,), torch.uint8)
            with torch.cuda.device(self.device):
                fb = native.Batch()
                self._batch_frames(fb)
                fb.frame_count = F
                native.check(native.lib().hpg_fourier_full(plan.handle, ctypes.byref(fb), native.ptr(plane),
                                                           native.ptr(ws), ws_bytes, native.stream_handle()),
                             "hpg_fourier_full")
            self._fourier_full = plane
        return self._fourier_full

    def get_fourier_plane_full(self):
        if self._st0 is None:
            return None
        plane = self._fourier_plane_device().cpu().numpy()
        return plane, self._plan["frame_count"], self._st0["P"], plane.shape[-1], plane.shape[-2]

    def get_fourier_plane_window(self):
        if self._st1 is None:
            return None
        if self._window is None:
            keep = (self._field_r, self._field_i, self._field_scale, self._field_axes)
            self._run_fused(with_coefs=False, windows=True)
            # the window run recomputes identical fields; keep the stage state as it was
            self._field_r, self._field_i, self._field_scale, self._field_axes = keep
        w = self._window.cpu().numpy()
        return w, self._plan["batch"], self._st0["P"], w.shape[-1], w.shape[-2]

    def _plane_summary(self, data, xa, ya, pol_sums=False):
        torch = _torch()
        count, P, h, w = data.shape
        slots = count + 1
        params = torch.zeros((C.ANALYSIS_COUNT, P, slots), dtype=torch.float32, device=self.device)
        inten = torch.zeros((h, w), dtype=torch.float32, device=self.device)
        xa_d = torch.as_tensor(np.asarray(xa, np.float64), device=self.device)
        ya_d = torch.as_tensor(np.asarray(ya, np.float64), device=self.device)
        L = native.lib()
        wsb = L.hpg_plane_summary_workspace(count, P, h, w)
        ws = self._buf("ws_sum", (wsb,), torch.uint8)
        pol_total = torch.empty((P, h, w), dtype=torch.float64, device=self.device) if pol_sums else None
        with torch.cuda.device(self.device):
            native.check(L.hpg_plane_summary(native.ptr(data), count, P, h, w, native.ptr(xa_d),
                                             native.ptr(ya_d), native.ptr(params), slots, native.ptr(inten),
                                             native.ptr(pol_total), native.ptr(ws), wsb, native.stream_handle()),
                         "hpg_plane_summary")
        if pol_sums:
            return params, inten, pol_total
        return params, inten

    # ------------------------------------------------ AutoAlign reductions
    def fourier_intensity_per_pol(self):
        """sum_b |F|^2 over the full R2C plane per pol, fp64 (holopipe/align.py:53-55)."""
        fx, fy = self._fourier_axes_pair()
        _, _, pt = self._plane_summary(self._fourier_plane_device(), fx, fy, pol_sums=True)
        return pt.cpu().numpy()

    def window_intensity_per_pol(self):
        """sum_b |window|^2 per pol, fp64 (holopipe/align.py:177)."""
        self.get_fourier_plane_window()
        w = self._window
        wh, ww = w.shape[-2:]
        xa = np.arange(ww, dtype=np.float64)
        ya = np.arange(wh, dtype=np.float64)
        _, _, pt = self._plane_summary(w, xa, ya, pol_sums=True)
        return pt.cpu().numpy()

    def field_intensity_per_pol(self):
        """sum_b |dequantised int16 field|^2 per pol, fp64 (holopipe/align.py:163-169)."""
        torch = _torch()
        B, P, h, w = self._field_r.shape
        out = torch.empty((P, h, w), dtype=torch.float64, device=self.device)
        with torch.cuda.device(self.device):
            native.check(native.lib().hpg_field_intensity(
                native.ptr(self._field_r), native.ptr(self._field_i), native.ptr(self._field_scale),
                B, P, h, w, native.ptr(out), native.stream_handle()), "hpg_field_intensity")
        return out.cpu().numpy()

    def batch_summary(self, plane_idx):
        if plane_idx not in (C.PLANE_FOURIER, C.PLANE_FIELD):
            raise HoloError(ErrorCode.INVALIDDIMENSION, "invalid plane index")
        if plane_idx == C.PLANE_FOURIER:
            if self._st0 is None:
                raise HoloError(ErrorCode.NULLPOINTER, "plane has not been processed")
            if self._summary_fourier is None:
                fx, fy = self._fourier_axes_pair()
                params, inten = self._plane_summary(self._fourier_plane_device(), fx, fy)
                self._summary_fourier = AnalysisSummary(params.cpu().numpy(), inten.cpu().numpy(),
                                                        self._fourier_axes[0], self._fourier_axes[1], plane_idx)
            return self._summary_fourier
        if self._field_r is None or self._st2 is None:
            raise HoloError(ErrorCode.NULLPOINTER, "plane has not been processed")
        if self._summary_field is None:
            keep = (self._field_r, self._field_i, self._field_scale, self._coefs, self._mode_count, self._st3)
            self._run_fused(with_coefs=False, summary=True)
            (self._field_r, self._field_i, self._field_scale, self._coefs, self._mode_count, self._st3) = keep
        params, inten = self._summary_field
        if not isinstance(params, np.ndarray):
            x_axis, y_axis = self._field_axes
            self._summary_field = (params.cpu().numpy(), inten.cpu().numpy())
            params, inten = self._summary_field
        x_axis, y_axis = self._field_axes
        return AnalysisSummary(params, inten, x_axis, y_axis, plane_idx)

    def get_ref_calibration_fields(self):
        """(applied, wavelength_count, pol_count, x, y, nx, ny) (engine.py:484-490)."""
        if self._ref_applied is None:
            return None
        x_axis, y_axis = self._field_axes
        return (self._ref_applied.cpu().numpy(), self.ref_cal.wavelength_count, self._st0["P"],
                x_axis, y_axis, x_axis.size, y_axis.size)

    def basis_get_fields(self):
        cfg = self.config
        if cfg.basisGroupCount < 1 or self._field_axes is None:
            return None
        G = cfg.basisGroupCount
        plan = self._native_plan(self._plan_key(G, self._effective()[2]))
        hx, hy = plan.basis(self._st0["P"], G)
        idx = mode_indices(G)
        modes = np.stack([np.stack([np.outer(hy[q, n], hx[q, m]) for (m, n) in idx])
                          for q in range(self._st0["P"])], axis=1).astype(np.complex64)
        x_axis, y_axis = self._field_axes
        return modes, modes.shape[0], self._st0["P"], x_axis, y_axis, x_axis.size, y_axis.size

    # ------------------------------------------------------------ metrics
    def calc_metrics(self):
        """Transfer-matrix metrics (engine.py:503-515, analysis.py:213-248)."""
        if self._coefs is None:
            raise HoloError(ErrorCode.NULLPOINTER, "no coefficients have been computed")
        cfg = self.config
        plan = self._plan
        L = len(plan["lambdas"])
        wl = plan["wl_of_batch"]
        per = np.full((C.METRIC_COUNT, L), C.METRIC_UNSET)
        pending = []
        for w in range(L):
            rows = np.nonzero(wl == w)[0]
            if rows.size == 0:
                continue
            per[:, w] = self._metrics_rows(rows, pending, w)
        self._metrics = average_slot(per)
        self._metrics.defer_mdl(pending)
        return ErrorCode.SUCCESS

    def _metrics_rows(self, rows, pending=None, slot=0):
        torch = _torch()
        cfg = self.config
        P, M = self._st0["P"], self._mode_count
        cols = P * M
        pol_ind = bool(cfg.autoAlignPolIndependence) and P > 1
        if cfg.autoAlignBasisMulConjTrans:
            A = self._coefs[torch.as_tensor(rows, device=self.device)].to(torch.complex128)
            if pol_ind:
                blocks = torch.zeros((P * len(rows), cols), dtype=torch.complex128, device=self.device)
                for q in range(P):
                    blocks[q * len(rows):(q + 1) * len(rows), q * M:(q + 1) * M] = A[:, q * M:(q + 1) * M]
                A = blocks
            G = (A @ A.conj().T).cpu().numpy()
            return metrics_of_matrix(G, None)
        if pol_ind:
            vrows = np.concatenate([rows for _ in range(P)])
            offs = np.repeat(np.arange(P) * M, len(rows))
            cnts = np.full(P * len(rows), M)
        else:
            vrows, offs, cnts = rows, None, None
        R = len(vrows)
        dev = self.device
        # device index tables of this row set / layout, cached across AutoAlign evaluations
        key = (vrows.tobytes(), P, M, pol_ind)
        cache = self._bufs.get("metric_idx")
        if cache is None or cache[0] != key:
            labels = np.array([q * 1000 + mode_group_of_index(i) for q in range(P) for i in range(M)], np.int32)
            t_rows = torch.as_tensor(vrows.astype(np.int32), device=dev)
            t_off = torch.as_tensor(offs.astype(np.int32), device=dev) if offs is not None else None
            t_cnt = torch.as_tensor(cnts.astype(np.int32), device=dev) if cnts is not None else None
            cache = (key, t_rows, t_off, t_cnt, torch.as_tensor(labels, device=dev))
            self._bufs["metric_idx"] = cache
        _, t_rows, t_off, t_cnt, t_lab = cache
        gram_rows = 1 if R <= cols else 0
        n = R if gram_rows else cols
        # one packed fp64 buffer (row | diag | group powers, Gram) -> a single device-to-host copy
        r3 = (3 * R + 1) & ~1
        packed = self._buf("metric_out", (r3 + 2 * n * n,), torch.float64)
        a = native.MetricArgs()
        a.coefs = self._coefs.data_ptr()
        a.rows, a.cols, a.ld = R, cols, cols
        a.row_ids = t_rows.data_ptr()
        a.col_offset = t_off.data_ptr() if t_off is not None else None
        a.col_count = t_cnt.data_ptr() if t_cnt is not None else None
        a.labels = t_lab.data_ptr()
        a.ndiag, a.diag_offset, a.gram_rows = min(R, cols), 0, gram_rows
        base = packed.data_ptr()
        a.row_power, a.diag_power, a.group_power = base, base + 8 * R, base + 16 * R
        big = not gram_rows and R * cols * cols > (1 << 28)   # large batches: Gram by cuBLAS zgemm
        a.gram = None if big else base + 8 * r3
        with torch.cuda.device(dev):
            native.check(native.lib().hpg_metric_partials(ctypes.byref(a), native.stream_handle(dev)),
                         "hpg_metric_partials")
            if big:
                from .distributed import gram_of_rows
                gview = packed[r3:].view(torch.complex128).view(n, n)
                gview.zero_()
                gram_of_rows(self._coefs, t_rows.long(), gview)
        host = packed.cpu().numpy()
        gram = host[r3:].view(np.complex128).reshape(n, n)
        v = finish_metrics(host[:R], host[R:2 * R], host[2 * R:3 * R], gram, R, cols, True,
                           defer_mdl=pending is not None)
        if pending is not None and host[:R].sum() > 0:
            pending.append((slot, gram.copy(), min(R, cols)))
        return v

    def metric(self, metric_idx):
        if self._metrics is None:
            return C.METRIC_UNSET if 0 <= metric_idx < C.METRIC_COUNT else 0.0
        return self._metrics.get(metric_idx)

    def metrics_array(self, metric_idx):
        if self._metrics is None:
            return np.full(self.config.wavelength_count() + 1, C.METRIC_UNSET, dtype=np.float32)
        return self._metrics.get_all(metric_idx)

    # ------------------------------------------------------- calibration
    def set_batch_calibration(self, cal, pol_count_cal, batch_count_cal):
        if cal is None or pol_count_cal < 1 or batch_count_cal < 1:
            self.batch_cal_enabled = 0
            return False
        self.batch_cal = np.asarray(cal, dtype=np.complex64).reshape(pol_count_cal, batch_count_cal).copy()
        self.batch_cal_enabled = 1
        return True
