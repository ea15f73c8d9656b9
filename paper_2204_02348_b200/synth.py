"""Seeded synthetic off-axis hologram frames.

Not part of the processing path: this generates the camera frames the bench
and the parity tests feed to both the oracle and the CUDA path.  The
conventions follow the reference simulator (holopipe/simulate.py:164-190):
signal S is a Hermite-Gaussian superposition on each polarisation's half of
the frame, the reference is R = exp(-2 pi i (fx x + fy y)) on absolute frame
coordinates, S is scaled to 1:1 power with R over the whole batch, and the
frame is |S + R|^2.  BASELINE.md adds the camera model: scale to a 4095
maximum, then either additive Gaussian noise (sigma = 1% of max, no clip) or
Poisson shot noise clipped to [0, 4095] (12-bit).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class FrameSpec:
    width: int = 256
    height: int = 256
    pol_count: int = 1
    batch: int = 16
    group_count: int = 9          # synthesis HG groups
    waist: float = 200e-6
    tilt: tuple = (1.0, 1.0)      # degrees (x, y), same for both pols
    pixel: float = 20e-6
    wavelength: float = 1565e-9
    noise: str = "gauss"          # "gauss" | "poisson" | "none"
    zernike_terms: int = 0        # config 3: Noll 2..11 phase screen
    zernike_radius_px: float = 256.0
    seed: int = 1
    beam_centres: list = field(default_factory=list)  # per pol (x, y) metres


def _hg(G, axis, centre, waist):
    u = math.sqrt(2.0) * (np.asarray(axis, np.float64) - centre) / waist
    h = np.empty((G, u.size))
    h[0] = np.pi ** -0.25 * np.exp(-0.5 * u * u)
    if G > 1:
        h[1] = math.sqrt(2.0) * u * h[0]
    for k in range(2, G):
        h[k] = math.sqrt(2.0 / k) * u * h[k - 1] - math.sqrt((k - 1.0) / k) * h[k - 2]
    d = abs(axis[1] - axis[0]) if len(axis) > 1 else 1.0
    return h / np.sqrt((h * h).sum(axis=1) * d)[:, None]


def _zernike_noll_2_11(rho, th):
    s3, s5, s6, s8 = math.sqrt(3), math.sqrt(5), math.sqrt(6), math.sqrt(8)
    return [
        2 * rho * np.cos(th), 2 * rho * np.sin(th),
        s3 * (2 * rho ** 2 - 1),
        s6 * rho ** 2 * np.sin(2 * th), s6 * rho ** 2 * np.cos(2 * th),
        s8 * (3 * rho ** 3 - 2 * rho) * np.sin(th), s8 * (3 * rho ** 3 - 2 * rho) * np.cos(th),
        s8 * rho ** 3 * np.sin(3 * th), s8 * rho ** 3 * np.cos(3 * th),
        s5 * (6 * rho ** 4 - 6 * rho ** 2 + 1),
    ]


def default_centres(spec):
    """Beam centre of each pol at the middle of its region (metres)."""
    if spec.beam_centres:
        return list(spec.beam_centres)
    if spec.pol_count == 1:
        return [(0.0, 0.0)]
    q = spec.width // 4
    return [(-q * spec.pixel, 0.0), (q * spec.pixel, 0.0)]


def make_frames(spec: FrameSpec, chunk: int = 64, return_truth: bool = False):
    """(batch, height, width) float32 frames; optionally the true coefficients."""
    rng = np.random.default_rng(spec.seed)
    W, H, P, G = spec.width, spec.height, spec.pol_count, spec.group_count
    M = G * (G + 1) // 2
    p, lam = spec.pixel, spec.wavelength
    x_full = (np.arange(W) - W // 2) * p
    y = (np.arange(H) - H // 2) * p
    regions = [(0, W)] if P == 1 else [(0, W // 2), (W // 2, W)]
    centres = default_centres(spec)
    fx = math.sin(math.radians(spec.tilt[0])) / lam
    fy = math.sin(math.radians(spec.tilt[1])) / lam
    # coefficients: i.i.d. complex Gaussian, unit power per (frame, pol)
    c = rng.standard_normal((spec.batch, P, M)) + 1j * rng.standard_normal((spec.batch, P, M))
    c /= np.sqrt((np.abs(c) ** 2).sum(axis=-1, keepdims=True))
    zern = None
    if spec.zernike_terms:
        zc = rng.normal(0.0, 0.5, (spec.batch, spec.zernike_terms))
        X, Y = np.meshgrid(x_full / p, y / p)
        rho = np.hypot(X, Y) / spec.zernike_radius_px
        th = np.arctan2(Y, X)
        zern = (np.stack(_zernike_noll_2_11(rho, th)[:spec.zernike_terms]), zc)
    mode_idx = [(g - n, n) for g in range(G) for n in range(g + 1)]
    S = np.zeros((spec.batch, H, W), np.complex128)
    R = np.zeros((H, W), np.complex128)
    for q, (x0, x1) in enumerate(regions):
        xs = x_full[x0:x1]
        hx = _hg(G, xs, centres[q][0], spec.waist)
        hy = _hg(G, y, centres[q][1], spec.waist)
        C = np.zeros((spec.batch, G, G), np.complex128)        # C[b, n, m]
        for k, (m, n) in enumerate(mode_idx):
            C[:, n, m] = c[:, q, k]
        for b0 in range(0, spec.batch, chunk):
            b1 = min(spec.batch, b0 + chunk)
            S[b0:b1, :, x0:x1] = hy.T[None] @ C[b0:b1] @ hx[None]
        R[:, x0:x1] = np.exp(-2j * np.pi * (fx * xs[None, :] + fy * y[:, None]))
    if zern is not None:
        basis, zc = zern
        for b in range(spec.batch):
            S[b] *= np.exp(1j * np.tensordot(zc[b], basis, axes=(0, 0)))
    scale = math.sqrt(spec.batch * float((np.abs(R) ** 2).sum()) / float((np.abs(S) ** 2).sum()))
    frames = np.empty((spec.batch, H, W), np.float32)
    peak = 0.0
    for b0 in range(0, spec.batch, chunk):
        b1 = min(spec.batch, b0 + chunk)
        blk = np.abs(S[b0:b1] * scale + R[None]) ** 2
        peak = max(peak, float(blk.max()))
        frames[b0:b1] = blk
    frames *= np.float32(4095.0 / peak)
    if spec.noise == "gauss":
        frames += rng.normal(0.0, 0.01 * 4095.0, frames.shape).astype(np.float32)
    elif spec.noise == "poisson":
        frames = np.clip(rng.poisson(frames.astype(np.float64)), 0, 4095).astype(np.float32)
    if return_truth:
        return frames, c
    return frames


def frames_digest(frames) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(frames, np.float32).tobytes()).hexdigest()


# BASELINE.json configs, normalised as in BASELINE.md section 3.
CONFIGS = {
    "pr1": FrameSpec(256, 256, 1, 16, 9, 200e-6, (1.0, 1.0), noise="gauss", seed=1),
    "dualpol": FrameSpec(640, 256, 2, 1000, 14, 200e-6, (1.2, 0.9), noise="poisson", seed=2),
    "largeframe": FrameSpec(1024, 1024, 1, 256, 20, 1e-3, (1.5, 1.5), noise="gauss",
                            zernike_terms=10, seed=3),
    "autoalign": FrameSpec(320, 256, 1, 128, 9, 200e-6, (1.0, 1.0), noise="gauss", seed=4),
    "largebasis": FrameSpec(320, 256, 1, 65536, 45, 200e-6, (1.0, 1.0), noise="poisson", seed=5),
}
