"""CPU oracle for the digHolo batch hot path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  The
product package (``paper_2204_02348_b200``) never imports it and has no CPU
fallback: its compute path is the CUDA library behind ``include/holo_b200.h``.

It restates, in vectorised numpy, the algorithm of the reference package
``holopipe`` (``/root/reference/pkg/src/holopipe``) for the chain

    frame -> window -> R2C FFT -> Fourier-window crop -> reduced IFFT
          -> tilt/defocus removal -> field summary -> int16 field
          -> separable HG overlap -> coefficients -> transfer-matrix metrics

Every function cites the reference lines it follows.  The FFT and the small
SVD go through the same third-party libraries the reference calls
(``scipy.fft`` 1.18 / ducc0 for ``rfft2``/``ifft2``; numpy LAPACK for the SVD),
so numerical agreement with the reference is at float32 round-off.

Parity pin: ``tests/golden/make_golden.py`` runs the *reference itself*
(imported from /root/reference in the build container) on seeded frames and
stores its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this oracle against those fixtures.  The reference ships no golden
vectors of its own.

``cfg`` arguments are any object carrying the reference ``HoloConfig`` field
names (``holopipe/config.py:33-71``).
"""

from __future__ import annotations

import math

import numpy as np
import scipy.fft

PIXEL_QUANTA = 16                      # holopipe/constants.py:10
SINC_FLOOR = 1e-3                      # holopipe/pipeline.py:20
SNR_CAP_DB = 200.0                     # holopipe/analysis.py:23
UNSET = float(np.finfo(np.float32).min)  # holopipe/constants.py:59
N_ANALYSIS = 7                         # holopipe/constants.py:62-69
N_METRIC = 9                           # holopipe/constants.py:47-56


class OracleError(Exception):
    """Mirrors ``HoloError`` (holopipe/errors.py:25-30): carries an int code."""

    def __init__(self, code, msg=""):
        super().__init__(msg or str(code))
        self.code = int(code)


# --------------------------------------------------------------- geometry

def effective_params(cfg):
    """Tilt/defocus/waist after pol locks (holopipe/engine.py:79-92)."""
    tilt = [list(cfg.tilt[0]), list(cfg.tilt[1])]
    defocus = list(cfg.defocus)
    waist = list(cfg.basisWaist)
    if cfg.polLockTilt:
        tilt[0][1], tilt[1][1] = tilt[0][0], tilt[1][0]
    if cfg.polLockDefocus:
        defocus[1] = defocus[0]
    if cfg.polLockBasisWaist:
        waist[1] = waist[0]
    return tilt, defocus, waist


def origin_of(cfg, pol):
    """(col0, row0) and fractional centre (xi_x, xi_y) of one pol's window.

    holopipe/pipeline.py:23-44 (pol regions, half-even rounding, clamping) and
    holopipe/engine.py:147-150 (fractional centre).
    """
    W, H = cfg.frameWidth, cfg.frameHeight
    nx, ny, p = cfg.fftWindowSizeX, cfg.fftWindowSizeY, cfg.framePixelSize
    lo, hi = (0, W) if cfg.polCount == 1 else ((0, W // 2) if pol == 0 else (W // 2, W))
    if nx > hi - lo or ny > H:
        raise OracleError(5, "fft window does not fit")
    cx = cfg.beamCentre[0][pol] / p + W / 2.0
    cy = cfg.beamCentre[1][pol] / p + H / 2.0
    col0 = min(max(int(round(cx)) - nx // 2, lo), hi - nx)
    row0 = min(max(int(round(cy)) - ny // 2, 0), H - ny)
    return (col0, row0), (cx - col0, cy - row0)


def window_box(cfg):
    """(wh, ww, fr) of the Fourier window (holopipe/pipeline.py:62-69)."""
    fr = math.sin(math.radians(cfg.fourierWindowRadius)) / cfg.wavelengthCentre
    nx, ny, p = cfg.fftWindowSizeX, cfg.fftWindowSizeY, cfg.framePixelSize
    ww = min(2 * (int(np.floor(fr * nx * p)) + 1), nx)
    wh = min(2 * (int(np.floor(fr * ny * p)) + 1), ny)
    return wh, ww, fr


def circle(wh, ww, nx, ny, p, fr):
    """Boolean Fourier-window mask (holopipe/pipeline.py:72-76)."""
    fx = (np.arange(ww) - ww // 2) / (nx * p)
    fy = (np.arange(wh) - wh // 2) / (ny * p)
    return fy[:, None] ** 2 + fx[None, :] ** 2 <= fr * fr + 1e-30


def carrier_bin(tilt_deg, n, p, lam):
    """k0 = round_half_even(sin(tilt)*n*p/lam) (holopipe/engine.py:191-194)."""
    return int(round(float(np.sin(np.radians(tilt_deg)) * n * p / lam)))


def out_axes(cfg, wh, ww):
    """Field-plane axes in metres (holopipe/pipeline.py:152-160)."""
    nx, ny, p = cfg.fftWindowSizeX, cfg.fftWindowSizeY, cfg.framePixelSize
    if cfg.resolutionMode == 0:
        xa = (np.arange(nx) - nx // 2) * p
        ya = (np.arange(ny) - ny // 2) * p
    else:
        xa = (np.arange(ww) - ww // 2) * p * (nx / ww)
        ya = (np.arange(wh) - wh // 2) * p * (ny / wh)
    return xa.astype(np.float32), ya.astype(np.float32)


def wavelengths(cfg):
    return list(cfg.wavelengths) if cfg.wavelengths else [cfg.wavelengthCentre]


def batch_layout(cfg):
    """Averaging membership and wavelength of each batch row.

    holopipe/engine.py:94-120.
    """
    B, A = max(1, cfg.batchCount), max(1, cfg.avgCount)
    mode = cfg.avgMode if cfg.avgMode in (0, 1, 2) else 0
    lams = wavelengths(cfg)
    L = len(lams)
    rows = np.arange(B)
    if cfg.wavelengthOrdering[0] == 0 or L <= 1:
        wl = rows % L
    else:
        wl = np.minimum(rows * L // B, L - 1)
    a = np.arange(A)
    if mode == 1:
        members = rows[:, None] + a[None, :] * B
    elif mode == 2 and L > 1:
        members = ((rows // L) * A * L)[:, None] + a[None, :] * L + (rows % L)[:, None]
    else:
        members = rows[:, None] * A + a[None, :]
    return B, A, lams, wl.astype(np.int64), members.astype(np.int64)


def output_order(cfg, B, L):
    """Row permutation between wavelength orderings (holopipe/engine.py:22-34,122-131)."""
    o_in, o_out = cfg.wavelengthOrdering[0], cfg.wavelengthOrdering[1]
    if L <= 1 or B % L or o_in == o_out:
        return np.arange(B)
    idx = np.arange(B)
    if o_in == 0:
        return idx.reshape(B // L, L).T.reshape(-1)
    return idx.reshape(L, B // L).T.reshape(-1)


# ----------------------------------------------------------- FFT stages

def fourier_planes(frames, origins, nx, ny):
    """Windows then unnormalised rfft2 (holopipe/pipeline.py:47-59)."""
    F = frames.shape[0]
    win = np.empty((F, len(origins), ny, nx), np.float32)
    for k, (c0, r0) in enumerate(origins):
        win[:, k] = frames[:, r0:r0 + ny, c0:c0 + nx]
    return scipy.fft.rfft2(win, axes=(-2, -1)).astype(np.complex64)


def crop_window(plane, k0x, k0y, wh, ww, nx, ny, fill_factor):
    """Window of bins around (k0x, k0y), centred layout.

    Direct half-plane fetch or Hermitian partner, wrap modulo n, optional
    division by the pixel-sinc envelope (holopipe/pipeline.py:79-104).
    """
    bx = k0x + np.arange(ww) - ww // 2
    by = k0y + np.arange(wh) - wh // 2
    mx, my = np.mod(bx, nx), np.mod(by, ny)
    keep = mx <= nx // 2
    col = np.where(keep, mx, nx - mx)
    row = np.where(keep[None, :], my[:, None], np.mod(-by, ny)[:, None])
    got = plane[..., row, np.broadcast_to(col[None, :], (wh, ww))]
    got = np.where(keep[None, :], got, np.conj(got))
    if fill_factor:
        fy = np.where(my > ny // 2, my - ny, my) / float(ny)
        env = np.sinc(fy)[:, None] * np.sinc(col / float(nx))[None, :]
        env = np.where(np.abs(env) < SINC_FLOOR, SINC_FLOOR, env)
        got = got / env.astype(got.dtype)
    return got.astype(np.complex64)


def centre_shift(k0x, k0y, wh, ww, nx, ny, xi_x, xi_y):
    """Recentring phase (holopipe/pipeline.py:114-127)."""
    bx = k0x + np.arange(ww) - ww // 2
    by = k0y + np.arange(wh) - wh // 2
    ex = np.exp(2j * np.pi * bx * (xi_x - nx / 2.0) / nx)
    ey = np.exp(2j * np.pi * by * (xi_y - ny / 2.0) / ny)
    return (ey[:, None] * ex[None, :]).astype(np.complex64)


def constructive_mean(stack):
    """Phase-aligned mean over axis 1 of (R, A, h, w) (holopipe/engine.py:543-552)."""
    acc = stack[:, 0].astype(np.complex128)
    for k in range(1, stack.shape[1]):
        m = stack[:, k].astype(np.complex128)
        ip = np.sum(np.conj(acc) * m, axis=(-2, -1))
        rot = np.where(np.abs(ip) > 0, np.exp(-1j * np.angle(ip)), 1.0)
        acc = acc + m * rot[:, None, None]
    return (acc / stack.shape[1]).astype(np.complex64)


def inverse_window(win, mode, nx, ny):
    """ifftshift + ifft2, net 1/(nx*ny) (holopipe/pipeline.py:130-149)."""
    wh, ww = win.shape[-2:]
    if mode == 0 and (wh != ny or ww != nx):
        spec = np.zeros(win.shape[:-2] + (ny, nx), np.complex64)
        r0, c0 = ny // 2 - wh // 2, nx // 2 - ww // 2
        spec[..., r0:r0 + wh, c0:c0 + ww] = win
    else:
        spec = win
    spec = np.fft.ifftshift(spec, axes=(-2, -1))
    out = scipy.fft.ifft2(spec, axes=(-2, -1))
    return (out * (spec.shape[-2] * spec.shape[-1] / float(nx * ny))).astype(np.complex64)


def tilt_defocus_phase(xa, ya, tx_deg, ty_deg, defocus, lam, k0x, k0y,
                       nx, ny, p, bcx, bcy):
    """Conjugate residual reference phase (holopipe/pipeline.py:163-185)."""
    fx = np.sin(np.radians(tx_deg)) / lam
    fy = np.sin(np.radians(ty_deg)) / lam
    rx = fx - k0x / (nx * p)
    ry = fy - k0y / (ny * p)
    x = xa.astype(np.float64)
    y = ya.astype(np.float64)
    c = 2.0 * np.pi * (fx * bcx + fy * bcy) - np.pi * (k0x + k0y)
    phx = 2.0 * np.pi * rx * x + (np.pi * defocus / lam) * x * x
    phy = 2.0 * np.pi * ry * y + (np.pi * defocus / lam) * y * y
    return np.exp(-1j * (c + phx[None, :] + phy[:, None])).astype(np.complex64)


def pack_int16(fields):
    """Vectorised int16 packing of (..., h, w) complex64 fields.

    Same arithmetic as holopipe/pipeline.py:188-199 per (batch, pol): peak of
    |Re| and |Im|, scale = float32(32767/peak) (1 when peak is 0), float32
    product, round half to even.
    """
    re, im = fields.real, fields.imag
    peak = np.maximum(np.abs(re).max(axis=(-2, -1)), np.abs(im).max(axis=(-2, -1)))
    peak64 = peak.astype(np.float64)
    with np.errstate(divide="ignore"):
        scale = np.where(peak64 > 0, 32767.0 / np.where(peak64 > 0, peak64, 1.0), 1.0)
    scale = scale.astype(np.float32)
    fr = np.rint(re * scale[..., None, None]).astype(np.int16)
    fi = np.rint(im * scale[..., None, None]).astype(np.int16)
    return fr, fi, scale


# --------------------------------------------------------------- basis

def mode_list(G):
    """Group-major (m, n) with m descending in a group (holopipe/hgbasis.py:17-27)."""
    return [(g - n, n) for g in range(G) for n in range(g + 1)]


def group_of_mode(i):
    """holopipe/hgbasis.py:34-39."""
    g = 0
    while (g + 1) * (g + 2) // 2 <= i:
        g += 1
    return g


def hermite_gauss(G, axis, centre, waist):
    """Grid-renormalised HG profiles in fp64 (holopipe/hgbasis.py:42-70)."""
    axis = np.asarray(axis, np.float64)
    if axis.size == 0 or waist <= 0 or G < 1:
        raise OracleError(5, "bad basis")
    u = math.sqrt(2.0) * (axis - centre) / waist
    h = np.empty((G, axis.size))
    h[0] = np.pi ** -0.25 * np.exp(-0.5 * u * u)
    if G > 1:
        h[1] = math.sqrt(2.0) * u * h[0]
    for k in range(2, G):
        h[k] = math.sqrt(2.0 / k) * u * h[k - 1] - math.sqrt((k - 1.0) / k) * h[k - 2]
    d = abs(axis[1] - axis[0]) if axis.size > 1 else 1.0
    nrm = np.sqrt((h * h).sum(axis=1) * d)
    nrm[nrm == 0] = 1.0
    return h / nrm[:, None]


def quantised_profiles(G, axis, waist):
    """int16 profiles + per-order float32 scale (holopipe/hgbasis.py:76-93)."""
    h = hermite_gauss(G, axis, 0.0, waist)
    s = np.float32(32767.0) / np.abs(h).max(axis=1).astype(np.float32)
    q = np.round(h * s[:, None]).astype(np.int16)
    return q, s


def overlap(fields, xa, ya, G, waist):
    """HG coefficients of (..., h, w) complex64 fields.

    Separable contraction with the dequantised int16 basis and the grid
    measure dx*dy (holopipe/hgbasis.py:95-116).
    """
    qx, sx = quantised_profiles(G, xa, waist)
    qy, sy = quantised_profiles(G, ya, waist)
    hx = (qx.astype(np.float32) / sx[:, None]).astype(np.complex64)
    hy = (qy.astype(np.float32) / sy[:, None]).astype(np.complex64)
    dx = float(abs(xa[1] - xa[0])) if xa.size > 1 else 1.0
    dy = float(abs(ya[1] - ya[0])) if ya.size > 1 else 1.0
    t = np.tensordot(fields, hx.T, axes=([-1], [0]))
    t = np.moveaxis(np.tensordot(hy, t, axes=([1], [-2])), 0, -2)
    t = t * np.complex64(dx * dy)
    ms = mode_list(G)
    return t[..., [n for (_, n) in ms], [m for (m, _) in ms]]


def lg_matrix(G):
    """HG->LG unitary block matrix (holopipe/hgbasis.py:126-175)."""
    M = G * (G + 1) // 2
    T = np.zeros((M, M), np.complex128)
    off = 0
    for N in range(G):
        for row in range(N + 1):
            n, m = row, N - row
            sgn = (-1.0) ** min(n, m)
            den = math.factorial(n) * math.factorial(m) * 2 ** N
            for k in range(N + 1):
                poly = sum((-1) ** j * math.comb(n, j) * math.comb(m, k - j)
                           for j in range(max(0, k - m), min(n, k) + 1))
                b = math.sqrt(math.factorial(N - k) * math.factorial(k) / den) * poly
                T[off + row, off + k] = sgn * (1j ** k) * b
        off += N + 1
    return T


# ------------------------------------------------------------ analysis

def plane_stats(data, xa, ya):
    """Seven analysis parameters per (frame, pol) + aggregate slot.

    Vectorised restatement of holopipe/analysis.py:39-94.  ``data`` is
    (F, P, h, w) complex.  Returns (params (7, P, F+1) float32,
    total_intensity (h, w) float32).
    """
    data = np.asarray(data)
    if data.size == 0:
        raise OracleError(5, "empty plane")
    F, P = data.shape[:2]
    xa = np.asarray(xa, np.float64)
    ya = np.asarray(ya, np.float64)
    mag = np.abs(data)
    inten = mag.astype(np.float64) ** 2
    agg = inten.sum(axis=0)                                  # (P, h, w)
    I = np.concatenate([inten, agg[None]], axis=0)           # (F+1, P, h, w)
    A = np.concatenate([mag, np.sqrt(agg)[None]], axis=0)
    dx = float(abs(xa[1] - xa[0])) if xa.size > 1 else 1.0
    dy = float(abs(ya[1] - ya[0])) if ya.size > 1 else 1.0
    da = dx * dy
    tot = I.sum(axis=(-2, -1))
    colsum = I.sum(axis=-2)
    rowsum = I.sum(axis=-1)
    out = np.zeros((N_ANALYSIS, P, F + 1), np.float64)
    out[0] = (tot * da).T
    pos = tot > 0
    safe = np.where(pos, tot, 1.0)
    comx = (colsum * xa).sum(-1) / safe
    comy = (rowsum * ya).sum(-1) / safe
    aeff = (tot * da) ** 2 / np.where(pos, (I ** 2).sum(axis=(-2, -1)) * da, 1.0)
    span = dy * ya.size
    ang = 2.0 * np.pi * (ya - ya[0]) / span
    res = (rowsum * np.exp(1j * ang)).sum(-1)
    theta = np.mod(np.angle(res), 2.0 * np.pi)
    wrap = ya[0] + theta * span / (2.0 * np.pi)
    out[1] = np.where(pos, comx, 0.0).T
    out[2] = np.where(pos, comy, 0.0).T
    out[5] = np.where(pos, aeff, 0.0).T
    out[6] = np.where(pos, wrap, ya[0] if ya.size else 0.0).T
    flat = A.reshape(F + 1, P, -1)
    arg = flat.argmax(axis=-1)
    out[3] = np.take_along_axis(flat, arg[..., None], -1)[..., 0].T
    params = out.astype(np.float32)
    params[4] = arg.T.astype(np.int32).view(np.float32)
    return params, inten.sum(axis=(0, 1)).astype(np.float32)


def _db(x):
    return UNSET if x <= 0 else 10.0 * math.log10(x)


def _snr(sig, noise):
    if sig <= 0:
        return UNSET
    if noise <= 0:
        return SNR_CAP_DB
    return min(10.0 * math.log10(sig / noise), SNR_CAP_DB)


def transfer_matrix(coefs, M, P, pol_indep=0, conj_trans=0):
    """holopipe/analysis.py:104-126."""
    A = np.asarray(coefs, np.complex128).reshape(coefs.shape[0], P * M)
    if pol_indep and P > 1:
        B = A.shape[0]
        out = np.zeros((P * B, P * M), np.complex128)
        for q in range(P):
            out[q * B:(q + 1) * B, q * M:(q + 1) * M] = A[:, q * M:(q + 1) * M]
        A = out
    if conj_trans:
        A = A @ A.conj().T
    return A


def metrics_one(A, labels=None):
    """Nine metrics of one matrix (holopipe/analysis.py:143-188)."""
    v = np.full(N_METRIC, UNSET)
    if A.size == 0:
        return v
    pw = np.abs(A) ** 2
    R, Cn = A.shape
    nd = min(R, Cn)
    rowp = pw.sum(axis=1)
    v[0] = _db(float(rowp.mean()))
    if np.any(pw > 0):
        sv = np.linalg.svd(A, compute_uv=False)
        if sv.min() > 0:
            v[1] = 20.0 * math.log10(sv.max() / sv.min())
    d = pw[np.arange(nd), np.arange(nd)]
    dt = float(d.sum())
    ot = float(pw.sum() - dt)
    v[2] = _db(dt / nd)
    v[3] = _snr(dt, ot)
    with np.errstate(divide="ignore"):
        ddb = np.where(d > 0, 10.0 * np.log10(np.maximum(d, 1e-300)), UNSET)
    v[4], v[5] = float(ddb.max()), float(ddb.min())
    roff = rowp[:nd] - d
    snr = np.array([_snr(float(d[i]), float(roff[i])) for i in range(nd)])
    v[6] = float(snr.max()) if nd else UNSET
    v[7] = float(snr.min()) if nd else UNSET
    if labels is not None:
        lab = np.asarray(labels)
        same = lab[:nd, None] == lab[None, :]
        sig = float(np.where(same, pw[:nd], 0.0).sum())
        v[8] = _snr(sig, float(pw.sum() - sig))
    else:
        v[8] = v[3]
    return v


def metrics(coefs, M, P, wl_of_row, L, pol_indep=0, conj_trans=0, groups=None):
    """(9, L+1) float32 report (holopipe/analysis.py:213-248)."""
    rep = np.full((N_METRIC, L + 1), UNSET, np.float32)
    if coefs is None or coefs.size == 0:
        return rep
    labels = None
    if groups is not None:
        labels = [q * 1000 + g for q in range(P) for g in groups]
    per = np.full((N_METRIC, L), UNSET)
    for w in range(L):
        rows = np.nonzero(np.asarray(wl_of_row) == w)[0]
        if rows.size == 0:
            continue
        A = transfer_matrix(coefs[rows], M, P, pol_indep, conj_trans)
        per[:, w] = metrics_one(A, None if conj_trans else labels)
    rep[:, :L] = per.astype(np.float32)
    for m in range(N_METRIC):
        ok = per[m][per[m] > UNSET / 2]
        if ok.size:
            rep[m, L] = np.float32(ok.mean())
    return rep


# ------------------------------------------------------------ full chain

CAL_EPS = 1e-6   # holopipe/engine.py:332-333 (_CAL_EPS)


def ref_calibration(cfg, kind, raw, origins, xis, lams, wh, ww, mask, xa, ya):
    """Processed reference-wave calibration (holopipe/engine.py:276-335).

    kind 1 (intensity): sqrt of the max-normalised intensity window, carrier at DC,
    no removal phase; kind 2 (field): full complex FFT of conj(raw), window at the
    carrier k0 (no fill-factor envelope, pipeline.py:107-111), removal phase.
    Returns conj(proc) / max(|proc|^2, 1e-6), complex64 (Lc, P, gh, gw).
    """
    nx, ny, p = cfg.fftWindowSizeX, cfg.fftWindowSizeY, cfg.framePixelSize
    P = cfg.polCount
    tilt, defocus, _ = effective_params(cfg)
    if kind == 1:
        inten = np.asarray(raw, np.float32).astype(np.float64)
    else:
        inten = np.abs(np.asarray(raw, np.complex64).astype(np.complex128)) ** 2
    peak = inten.max()
    inten = np.ones_like(inten) if peak <= 0 else inten / peak     # frames.py:175-187
    Lc = inten.shape[0]
    out = np.empty((Lc, P, ya.size, xa.size), np.complex64)
    for ci in range(Lc):
        lam = lams[min(ci, len(lams) - 1)]
        for q in range(P):
            c0, r0 = origins[q]
            if kind == 1:
                amp = np.sqrt(inten[ci, r0:r0 + ny, c0:c0 + nx])
                spec = scipy.fft.rfft2(amp[None].astype(np.float32), axes=(-2, -1)).astype(np.complex64)[0]
                g = crop_window(spec, 0, 0, wh, ww, nx, ny, bool(cfg.fillFactorCorrectionEnabled))
                proc = inverse_window((g * mask * centre_shift(0, 0, wh, ww, nx, ny, *xis[q]))[None],
                                      cfg.resolutionMode, nx, ny)[0]
            else:
                ref = np.conj(np.asarray(raw, np.complex64)[ci, r0:r0 + ny, c0:c0 + nx])
                spec = np.fft.fft2(ref).astype(np.complex64)
                kx = carrier_bin(tilt[0][q], nx, p, lam)
                ky = carrier_bin(tilt[1][q], ny, p, lam)
                tx = np.mod(kx + np.arange(ww) - ww // 2, nx)
                ty = np.mod(ky + np.arange(wh) - wh // 2, ny)
                g = spec[ty[:, None], tx[None, :]].astype(np.complex64)
                proc = inverse_window((g * mask * centre_shift(kx, ky, wh, ww, nx, ny, *xis[q]))[None],
                                      cfg.resolutionMode, nx, ny)[0]
                proc = proc * tilt_defocus_phase(xa, ya, tilt[0][q], tilt[1][q], defocus[q], lam, kx, ky,
                                                 nx, ny, p, cfg.beamCentre[0][q], cfg.beamCentre[1][q])
            mag2 = np.maximum(np.abs(proc.astype(np.complex128)) ** 2, CAL_EPS)
            out[ci, q] = (np.conj(proc) / mag2).astype(np.complex64)
    return out


def run_chain(cfg, frames, batch_cal=None, stop_after=None, ref_cal=None, custom_transform=None):
    """Reference pipeline on host frames; returns a dict of stage products.

    Follows holopipe/engine.py:135-385 (process_fft, process_ifft,
    process_remove_tilt, extract_coefs) for float32 frames (B*A, H, W).
    ``ref_cal`` = (kind, raw) enables the reference-wave calibration
    (kind 1 intensity (Lc, H, W) float32, kind 2 field complex64).
    ``custom_transform`` (out x in complex) is the user matrix of basisType CUSTOM.
    """
    W, H = cfg.frameWidth, cfg.frameHeight
    nx, ny, p = cfg.fftWindowSizeX, cfg.fftWindowSizeY, cfg.framePixelSize
    P = cfg.polCount
    B, A, lams, wl, members = batch_layout(cfg)
    need = B * A * W * H
    flat = np.asarray(frames, np.float32).reshape(-1)
    if flat.size < need:
        raise OracleError(5, "frame buffer too short")
    fr = flat[:need].reshape(B * A, H, W)
    geo = [origin_of(cfg, q) for q in range(P)]
    origins = [g[0] for g in geo]
    xis = [g[1] for g in geo]
    plane = fourier_planes(fr, origins, nx, ny)
    out = {"plane": plane, "origins": origins, "xis": xis, "wl": wl}
    if stop_after == "fft":
        return out
    tilt, defocus, waist = effective_params(cfg)
    wh, ww, frad = window_box(cfg)
    mask = circle(wh, ww, nx, ny, p, frad)
    win = np.zeros((B, P, wh, ww), np.complex64)
    k0 = np.zeros((B, P, 2), np.int64)
    for q in range(P):
        for w, lam in enumerate(lams):
            rows = np.nonzero(wl == w)[0]
            if rows.size == 0:
                continue
            kx = carrier_bin(tilt[0][q], nx, p, lam)
            ky = carrier_bin(tilt[1][q], ny, p, lam)
            k0[rows, q] = (kx, ky)
            g = crop_window(plane[members[rows].reshape(-1), q], kx, ky, wh, ww,
                            nx, ny, bool(cfg.fillFactorCorrectionEnabled))
            g = g.reshape(rows.size, A, wh, ww)
            g = g * (mask * centre_shift(kx, ky, wh, ww, nx, ny, *xis[q]))[None, None]
            win[rows, q] = constructive_mean(g) if A > 1 else g[:, 0]
    raw = inverse_window(win, cfg.resolutionMode, nx, ny)
    xa, ya = out_axes(cfg, wh, ww)
    out.update(window=win, k0=k0, raw=raw, xa=xa, ya=ya, wh=wh, ww=ww)
    applied = None
    if ref_cal is not None:
        applied = ref_calibration(cfg, ref_cal[0], ref_cal[1], origins, xis, lams, wh, ww, mask, xa, ya)
        out["ref_applied"] = applied
    if stop_after == "ifft":
        return out
    fields = raw.copy()
    for q in range(P):
        for w, lam in enumerate(lams):
            rows = np.nonzero(wl == w)[0]
            if rows.size == 0:
                continue
            ph = tilt_defocus_phase(xa, ya, tilt[0][q], tilt[1][q], defocus[q], lam,
                                    int(k0[rows[0], q, 0]), int(k0[rows[0], q, 1]),
                                    nx, ny, p, cfg.beamCentre[0][q], cfg.beamCentre[1][q])
            fields[rows, q] *= ph[None]
    if batch_cal is not None:
        cal = np.asarray(batch_cal, np.complex64)
        for b in range(B):
            for q in range(P):
                fields[b, q] *= cal[min(q, cal.shape[0] - 1), b % cal.shape[1]]
    if applied is not None:   # engine.py:250-255
        for b in range(B):
            fields[b] *= applied[int(wl[b]) % applied.shape[0]]
    params, inten = plane_stats(fields, xa, ya)
    full = np.zeros((N_ANALYSIS, P, B * A + 1), np.float32)
    full[:, :, :B] = params[:, :, :B]
    full[:, :, B] = params[:, :, B]
    f16r, f16i, scale = pack_int16(fields)
    out.update(fields=fields, field_params=full, field_inten=inten,
               fr=f16r, fi=f16i, scale=scale)
    if cfg.basisGroupCount < 1 or stop_after == "tilt":
        out["coefs"] = None
        return out
    G = cfg.basisGroupCount
    M = G * (G + 1) // 2
    hg = np.empty((B, P, M), np.complex64)
    for q in range(P):
        deq = ((f16r[:, q].astype(np.float32) + 1j * f16i[:, q].astype(np.float32))
               / scale[:, q, None, None])
        hg[:, q] = overlap(deq, xa, ya, G, waist[q])
    transform = None   # engine.py:371-382: LG = conj(T_LG); CUSTOM = the user matrix (None -> HG)
    if getattr(cfg, "basisType", 0) == 1:
        transform = np.conj(lg_matrix(G))
    elif getattr(cfg, "basisType", 0) == 2:
        transform = custom_transform
    if transform is not None:
        use = min(M, transform.shape[1])
        hg = np.einsum("om,bpm->bpo", transform[:, :use], hg[:, :, :use].astype(np.complex128)).astype(np.complex64)
        M = hg.shape[-1]
    out["coefs"] = hg.reshape(B, P * M)
    out["coefs_out"] = out["coefs"][output_order(cfg, B, len(lams))]   # engine.py:408-417
    out["mode_count"] = M
    return out


def chain_metrics(cfg, coefs, M):
    """calc_metrics (holopipe/engine.py:503-515)."""
    _, _, lams, wl, _ = batch_layout(cfg)
    groups = [group_of_mode(i) for i in range(M)]
    return metrics(coefs, M, cfg.polCount, wl, len(lams),
                   cfg.autoAlignPolIndependence, cfg.autoAlignBasisMulConjTrans, groups)


# ----------------------------------------------------- plain config object

class Cfg:
    """Minimal stand-in with the reference HoloConfig defaults (holopipe/config.py:33-71)."""

    def __init__(self, **kw):
        lam, p = 1565e-9, 20e-6
        wmax = math.degrees(lam / (2 * p))
        wc = 0.320513 * wmax
        t = 3.0 * wc / math.sqrt(2.0)
        self.frameWidth, self.frameHeight, self.framePixelSize = 320, 256, p
        self.polCount = 1
        self.fftWindowSizeX = self.fftWindowSizeY = 128
        self.fourierWindowRadius = wc
        self.beamCentre = [[0.0, 0.0], [0.0, 0.0]]
        self.tilt = [[t, t], [t, t]]
        self.defocus = [0.0, 0.0]
        self.basisWaist = [4.2667e-4, 4.2667e-4]
        self.basisGroupCount = 0
        self.basisType = 0
        self.wavelengthCentre = lam
        self.wavelengths = []
        self.wavelengthOrdering = [0, 0]
        self.resolutionMode = 1
        self.fillFactorCorrectionEnabled = 0
        self.polLockTilt = self.polLockDefocus = self.polLockBasisWaist = 0
        self.autoAlignPolIndependence = 0
        self.autoAlignBasisMulConjTrans = 0
        self.batchCount = 1
        self.avgCount = 1
        self.avgMode = 0
        for k, v in kw.items():
            setattr(self, k, v)
