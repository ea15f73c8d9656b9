"""AutoAlign driver over the GPU engine (holopipe/align.py).

The algorithm is the reference's: a coarse "snap" (tilt from the peak of the
batch-summed Fourier intensity, beam centre and waist from the field-plane
aggregate summary, |defocus| from the Fourier-lobe spread) followed by cyclic
coordinate descent with a three-point parabolic fit per parameter, halving
all steps after each cycle.  Every evaluation is one GPU pipeline run
(``Engine.run_pipeline(from_stage)``) plus the GPU metric reductions; the
batch-summed intensities come from the plane-summary and field-intensity
kernels.  Only scalar decisions stay on the host.
"""

from __future__ import annotations

import numpy as np

from . import constants as C
from . import geometry
from .errors import HoloError

MAX_TWEAK_CYCLES = 20          # holopipe/align.py:17


def _direction(goal):
    return -1.0 if goal == C.METRIC_MDL else 1.0


def _evaluate(eng, from_stage):
    """One pipeline run + metrics (holopipe/align.py:25-29)."""
    eng.run_pipeline(from_stage)
    eng.calc_metrics()
    g = eng.config.autoAlignGoalIdx
    val = eng.metric(g) * _direction(g)
    rec = getattr(eng, "eval_log", None)
    if rec is not None:
        c = eng.config
        rec.append((from_stage, val, [c.tilt[0][0], c.tilt[1][0], c.beamCentre[0][0], c.beamCentre[1][0],
                                      c.defocus[0], c.basisWaist[0]]))
    return val


def _refine_peak(inten, row, col, ny):
    """Wrap-aware centroid over a 5x5 neighbourhood (holopipe/align.py:102-123)."""
    h, w = inten.shape
    dyv = np.arange(-2, 3)
    rows = (row + dyv) % h
    cols = col + dyv
    ok = (cols >= 0) & (cols < w)
    blk = inten[np.ix_(rows, cols[ok])].astype(np.float64)
    tot = float(blk.sum())
    if tot <= 0:
        return float(col), float(row if row <= ny // 2 else row - ny)
    kx = col + float((blk.sum(axis=0) * dyv[ok]).sum()) / tot
    kyr = row + float((blk.sum(axis=1) * dyv).sum()) / tot
    return float(kx), float(kyr if kyr <= ny / 2 else kyr - ny)


def _set_max_radius(cfg, pol):
    """Largest admissible window radius for a pol's tilt (holopipe/align.py:126-135)."""
    wmax = geometry.max_resolvable_angle(cfg.wavelengthCentre, cfg.framePixelSize)
    tx, ty = abs(cfg.tilt[0][pol]), abs(cfg.tilt[1][pol])
    r = min(np.hypot(tx, ty) / 3.0, wmax - tx, wmax - ty)
    if r > 0:
        cfg.fourierWindowRadius = float(r)


def _spread(inten, ax, ay):
    """Mean per-axis second-moment std (holopipe/align.py:138-149)."""
    tot = inten.sum()
    if tot <= 0:
        return 0.0
    px, py = inten.sum(axis=0), inten.sum(axis=1)
    mx, my = (px * ax).sum() / tot, (py * ay).sum() / tot
    var = ((px * (ax - mx) ** 2).sum() + (py * (ay - my) ** 2).sum()) / (2.0 * tot)
    return float(np.sqrt(var))


def _defocus_magnitude(eng, pol, field_int, window_int):
    """|defocus| from excess Fourier-lobe spread (holopipe/align.py:152-189)."""
    cfg = eng.config
    x_axis, y_axis = eng._field_axes
    sx = _spread(field_int[pol], x_axis.astype(np.float64), y_axis.astype(np.float64))
    if sx <= 0:
        return 0.0
    wi = window_int[pol]
    wh, ww = wi.shape
    nx, ny, p = cfg.fftWindowSizeX, cfg.fftWindowSizeY, cfg.framePixelSize
    fx = (np.arange(ww) - ww // 2) / (nx * p)
    fy = (np.arange(wh) - wh // 2) / (ny * p)
    sf = _spread(wi, fx, fy)
    mbar = max(cfg.basisGroupCount - 1, 0) / 3.0
    floor = (mbar + 0.5) / (2.0 * np.pi * sx)
    excess = sf ** 2 - floor ** 2
    if excess <= 0:
        return 0.0
    return float(cfg.wavelengthCentre * np.sqrt(excess) / sx)


def snap_estimate(eng):
    """Coarse estimate of tilt, radius, centre, waist and |defocus| (holopipe/align.py:32-99)."""
    cfg = eng.config
    if eng._st0 is None:
        eng.process_fft()
    nx, ny, p, lam = cfg.fftWindowSizeX, cfg.fftWindowSizeY, cfg.framePixelSize, cfg.wavelengthCentre
    wmax = geometry.max_resolvable_angle(lam, p)
    eng._fourier_axes_pair()
    tx_ax, ty_ax = eng._fourier_axes
    excl = (tx_ax[None, :].astype(np.float64) ** 2 + ty_ax[:, None].astype(np.float64) ** 2) < (wmax / 3.0) ** 2
    inten_all = eng.fourier_intensity_per_pol() if cfg.autoAlignTilt else None
    for pol in range(cfg.polCount):
        if cfg.autoAlignTilt:
            masked = np.where(excl, 0.0, inten_all[pol])
            row, col = divmod(int(np.argmax(masked)), masked.shape[1])
            kx, ky = _refine_peak(masked, row, col, ny)
            cfg.tilt[0][pol] = float(geometry.bin_to_tilt(kx, nx, p, lam))
            cfg.tilt[1][pol] = float(geometry.bin_to_tilt(ky, ny, p, lam))
        if cfg.autoAlignFourierWindowRadius:
            _set_max_radius(cfg, pol)
    if cfg.polLockTilt and cfg.polCount == 2:
        cfg.tilt[0][1], cfg.tilt[1][1] = cfg.tilt[0][0], cfg.tilt[1][0]
    if not (cfg.autoAlignBeamCentre or cfg.autoAlignBasisWaist or cfg.autoAlignDefocus):
        return
    eng.process_ifft()
    eng.process_remove_tilt()
    summ = eng.batch_summary(C.PLANE_FIELD)
    agg = eng._plan["batch"]
    field_int = window_int = None
    if cfg.autoAlignDefocus:
        field_int = eng.field_intensity_per_pol()
        window_int = eng.window_intensity_per_pol()
    for pol in range(cfg.polCount):
        if cfg.autoAlignBeamCentre:
            cfg.beamCentre[0][pol] += float(summ.parameters[C.ANALYSIS_COMX, pol, agg])
            cfg.beamCentre[1][pol] += float(summ.parameters[C.ANALYSIS_COMY, pol, agg])
        if cfg.autoAlignBasisWaist and cfg.basisGroupCount >= 1:
            aeff = float(summ.parameters[C.ANALYSIS_AEFF, pol, agg])
            if aeff > 0:
                mean_order = 2.0 * (cfg.basisGroupCount - 1) / 3.0
                cfg.basisWaist[pol] = float(np.sqrt(aeff / np.pi) / np.sqrt(mean_order + 1.0))
        if cfg.autoAlignDefocus:
            cfg.defocus[pol] = _defocus_magnitude(eng, pol, field_int, window_int)
    if cfg.polCount == 2:
        if cfg.polLockBasisWaist:
            cfg.basisWaist[1] = cfg.basisWaist[0]
        if cfg.polLockDefocus:
            cfg.defocus[1] = cfg.defocus[0]
    if cfg.autoAlignBeamCentre:
        eng.process_fft()


class _Knob:
    """One tweakable parameter: getter, setter, initial step, restart stage."""

    def __init__(self, name, get, put, step, stage):
        self.name, self.get, self.put, self.step, self.stage = name, get, put, step, stage


def _knobs(eng):
    """Enabled parameters in the reference's order (holopipe/align.py:201-245)."""
    cfg = eng.config
    p = cfg.framePixelSize
    bin_deg = geometry.bin_width_deg(cfg.fftWindowSizeX, p, cfg.wavelengthCentre)
    out = []
    if cfg.autoAlignTilt:
        locked = bool(cfg.polLockTilt) or cfg.polCount == 1
        for pol in range(1 if locked else 2):
            for axis in (0, 1):
                def put(v, a=axis, q=pol, lk=locked):
                    cfg.tilt[a][q] = v
                    if lk:
                        cfg.tilt[a][1] = cfg.tilt[a][0]
                out.append(_Knob(f"tilt{'xy'[axis]}[{pol}]", lambda a=axis, q=pol: cfg.tilt[a][q],
                                 put, 0.25 * bin_deg, 1))
    if cfg.autoAlignBeamCentre:
        for pol in range(1 if cfg.polCount == 1 else 2):
            for axis in (0, 1):
                def put(v, a=axis, q=pol):
                    cfg.beamCentre[a][q] = v
                out.append(_Knob(f"centre{'xy'[axis]}[{pol}]", lambda a=axis, q=pol: cfg.beamCentre[a][q],
                                 put, 1.0 * p, 0))
    if cfg.autoAlignDefocus:
        locked = bool(cfg.polLockDefocus) or cfg.polCount == 1
        for pol in range(1 if locked else 2):
            def put(v, q=pol, lk=locked):
                cfg.defocus[q] = v
                if lk:
                    cfg.defocus[1] = cfg.defocus[0]
            out.append(_Knob(f"defocus[{pol}]", lambda q=pol: cfg.defocus[q], put, 0.05, 2))
    if cfg.autoAlignBasisWaist and cfg.basisGroupCount >= 1:
        def put(v):
            cfg.basisWaist[0] = cfg.basisWaist[1] = v
        out.append(_Knob("basisWaist", lambda: cfg.basisWaist[0], put, 0.05 * cfg.basisWaist[0], 3))
    return out


def tweak_optimise(eng):
    """Cyclic coordinate descent with parabolic line fits (holopipe/align.py:248-299)."""
    cfg = eng.config
    eng.tweak_cycles = 0
    if cfg.basisGroupCount < 1:
        return None
    knobs = _knobs(eng)
    best = _evaluate(eng, 0)
    if not knobs:
        return best
    sign_probed = False
    for _ in range(MAX_TWEAK_CYCLES):
        start = best
        for k in knobs:
            x0 = k.get()
            step = k.step
            if k.name.startswith("defocus") and not sign_probed and x0 != 0.0:
                sign_probed = True        # the snap cannot sign the defocus: probe -x0
                k.put(-x0)
                v_neg = _evaluate(eng, k.stage)
                if v_neg > best:
                    best, x0 = v_neg, -x0
                else:
                    k.put(x0)
                    best = _evaluate(eng, k.stage)
            cand = {}
            for x in (x0 - step, x0 + step):
                k.put(x)
                cand[x] = _evaluate(eng, k.stage)
            vm, vp = cand[x0 - step], cand[x0 + step]
            den = vm - 2.0 * best + vp
            if den < 0:
                vx = x0 + 0.5 * step * (vm - vp) / den
                vx = min(max(vx, x0 - 2 * step), x0 + 2 * step)
                k.put(vx)
                cand[vx] = _evaluate(eng, k.stage)
            cand[x0] = best
            xb = max(cand, key=cand.get)
            k.put(xb)
            best = _evaluate(eng, k.stage)
        eng.tweak_cycles += 1
        for k in knobs:
            k.step *= 0.5
        if best - start < max(cfg.autoAlignTol, 0.0) + 1e-12:
            break
    return best


def auto_align(eng):
    """Run the configured mode; returns the goal metric (0.0 on error), holopipe/align.py:302-319."""
    cfg = eng.config
    eng.tweak_cycles = 0
    try:
        # frames cannot change during one auto_align call: stage them on the device once
        # (full frames: the window origins move with the beam centre)
        plan = eng._batch_plan()
        frames = eng.source.staged(plan["frame_count"], cfg.frameWidth, cfg.frameHeight, eng.device)
        eng.source.freeze(frames[0].clone())
        try:
            if cfg.autoAlignMode in (C.AUTOALIGNMODE_FULL, C.AUTOALIGNMODE_ESTIMATE):
                snap_estimate(eng)
            if cfg.autoAlignMode in (C.AUTOALIGNMODE_FULL, C.AUTOALIGNMODE_TWEAK) and cfg.basisGroupCount >= 1:
                tweak_optimise(eng)
            else:
                eng.run_pipeline(0)
            if cfg.basisGroupCount >= 1:
                eng.calc_metrics()
                return eng.metric(cfg.autoAlignGoalIdx)
            return 0.0
        finally:
            eng.source.thaw()
    except HoloError:
        return 0.0
