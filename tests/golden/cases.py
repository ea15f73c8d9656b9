"""Golden parity cases: frame spec + engine config (reference HoloConfig names).

Shared by tests/golden/make_golden.py (which runs the reference on them) and
the parity tests (which run the oracle and the CUDA path on the same frames).
Sizes are chosen so the reference finishes each case in about a second.
"""

import math

LAM, PIX = 1565e-9, 20e-6
WMAX = math.degrees(LAM / (2 * PIX))        # holopipe/geometry.py:29-37
RADIUS = 0.32 * WMAX
WRAP_FRAC = (-2.0 + math.sqrt(68.0)) / 16.0     # holopipe/geometry.py:23
WC_WRAP = WRAP_FRAC * WMAX * 0.98


def _cfg(**kw):
    base = dict(framePixelSize=PIX, wavelengthCentre=LAM, fourierWindowRadius=RADIUS,
                fftWindowSizeX=128, fftWindowSizeY=128, resolutionMode=1)
    base.update(kw)
    return base


CASES = {
    # BASELINE config 1 (PR1), 4-frame subset
    "pr1": dict(
        frames=dict(width=256, height=256, pol_count=1, batch=4, group_count=9,
                    waist=200e-6, tilt=(1.0, 1.0), noise="gauss", seed=1),
        config=_cfg(frameWidth=256, frameHeight=256, polCount=1, batchCount=4,
                    tilt=[[1.0, 1.0], [1.0, 1.0]], basisGroupCount=9,
                    basisWaist=[200e-6, 200e-6]),
        store_fourier=True),
    # BASELINE config 2 (dual polarisation), 3-frame subset
    "dualpol": dict(
        frames=dict(width=640, height=256, pol_count=2, batch=3, group_count=14,
                    waist=200e-6, tilt=(1.2, 0.9), noise="poisson", seed=2),
        config=_cfg(frameWidth=640, frameHeight=256, polCount=2, batchCount=3,
                    tilt=[[1.2, 1.2], [0.9, 0.9]], basisGroupCount=14,
                    basisWaist=[200e-6, 200e-6],
                    beamCentre=[[-160 * PIX, 160 * PIX], [0.0, 0.0]])),
    # BASELINE config 5 (1035-mode basis), 2-frame subset
    "largebasis": dict(
        frames=dict(width=320, height=256, pol_count=1, batch=2, group_count=45,
                    waist=200e-6, tilt=(1.0, 1.0), noise="poisson", seed=5),
        config=_cfg(frameWidth=320, frameHeight=256, polCount=1, batchCount=2,
                    tilt=[[1.0, 1.0], [1.0, 1.0]], basisGroupCount=45,
                    basisWaist=[200e-6, 200e-6])),
    # BASELINE config 3 (512 window, fields only), 1-frame subset
    "largeframe": dict(
        frames=dict(width=1024, height=1024, pol_count=1, batch=1, group_count=20,
                    waist=1e-3, tilt=(1.5, 1.5), noise="gauss", zernike_terms=10, seed=3),
        config=_cfg(frameWidth=1024, frameHeight=1024, polCount=1, batchCount=1,
                    fftWindowSizeX=512, fftWindowSizeY=512,
                    tilt=[[1.5, 1.5], [1.5, 1.5]], basisGroupCount=0)),
    # off-centre fractional beam centre, defocus, unequal tilts, 64x96 window
    "offcentre": dict(
        frames=dict(width=320, height=256, pol_count=1, batch=3, group_count=6,
                    waist=150e-6, tilt=(1.1, 0.8), noise="gauss", seed=11,
                    beam_centres=[(3.3e-4, -2.1e-4)]),
        config=_cfg(frameWidth=320, frameHeight=256, polCount=1, batchCount=3,
                    fftWindowSizeX=96, fftWindowSizeY=64,
                    beamCentre=[[3.3e-4, 0.0], [-2.1e-4, 0.0]],
                    tilt=[[1.1, 1.1], [0.8, 0.8]], defocus=[0.35, 0.0],
                    basisGroupCount=6, basisWaist=[150e-6, 150e-6])),
    # wrap-around window at the +-ky Nyquist edge (holopipe tests/test_pipeline.py:263-281)
    "wrap": dict(
        frames=dict(width=256, height=256, pol_count=1, batch=3, group_count=5,
                    waist=128 * PIX / 5, tilt=(WMAX - WC_WRAP, WMAX),
                    noise="gauss", seed=12),
        config=_cfg(frameWidth=256, frameHeight=256, polCount=1, batchCount=3,
                    fourierWindowRadius=WC_WRAP,
                    tilt=[[WMAX - WC_WRAP] * 2, [WMAX] * 2],
                    basisGroupCount=5, basisWaist=[128 * PIX / 5] * 2)),
    # fill-factor correction, full-frame 64x64 window (reference unit-test geometry)
    "fillfactor": dict(
        frames=dict(width=64, height=64, pol_count=1, batch=2, group_count=3,
                    waist=64 * PIX / 6, tilt=(1.5, 1.5), noise="gauss", seed=13),
        config=_cfg(frameWidth=64, frameHeight=64, polCount=1, batchCount=2,
                    fftWindowSizeX=64, fftWindowSizeY=64, fillFactorCorrectionEnabled=1,
                    tilt=[[1.5, 1.5], [1.5, 1.5]], basisGroupCount=3,
                    basisWaist=[64 * PIX / 6] * 2)),
    # IFFT resolution mode 0 (full-size band-limited interpolation)
    "mode0": dict(
        frames=dict(width=128, height=128, pol_count=1, batch=2, group_count=4,
                    waist=128 * PIX / 6, tilt=(1.5, 1.5), noise="gauss", seed=14),
        config=_cfg(frameWidth=128, frameHeight=128, polCount=1, batchCount=2,
                    resolutionMode=0, tilt=[[1.5, 1.5], [1.5, 1.5]], basisGroupCount=4,
                    basisWaist=[128 * PIX / 6] * 2)),
    # two wavelengths, slow input ordering, fast output ordering
    "multiwl": dict(
        frames=dict(width=256, height=256, pol_count=1, batch=4, group_count=4,
                    waist=200e-6, tilt=(1.0, 1.0), noise="gauss", seed=15),
        config=_cfg(frameWidth=256, frameHeight=256, polCount=1, batchCount=4,
                    wavelengths=[1550e-9, 1580e-9], wavelengthOrdering=[1, 0],
                    tilt=[[1.0, 1.0], [1.0, 1.0]], basisGroupCount=4,
                    basisWaist=[200e-6, 200e-6])),
    # constructive averaging, interlaced, 3 groups of 2
    "average": dict(
        frames=dict(width=256, height=256, pol_count=1, batch=6, group_count=4,
                    waist=200e-6, tilt=(1.0, 1.0), noise="gauss", seed=16),
        config=_cfg(frameWidth=256, frameHeight=256, polCount=1, batchCount=3,
                    avgCount=2, avgMode=1, tilt=[[1.0, 1.0], [1.0, 1.0]],
                    basisGroupCount=4, basisWaist=[200e-6, 200e-6])),
    # dual-pol with pol locks off, different per-pol tilts and a batch calibration
    "dualpol_cal": dict(
        frames=dict(width=320, height=128, pol_count=2, batch=2, group_count=4,
                    waist=120e-6, tilt=(1.0, 1.0), noise="gauss", seed=17),
        config=_cfg(frameWidth=320, frameHeight=128, polCount=2, batchCount=2,
                    fftWindowSizeX=128, fftWindowSizeY=128,
                    tilt=[[1.0, 0.95], [1.0, 1.05]], basisGroupCount=4,
                    basisWaist=[120e-6, 120e-6], defocus=[0.0, -0.2],
                    beamCentre=[[-80 * PIX, 80 * PIX], [0.0, 0.0]]),
        batch_cal=[[1.0 + 0.0j, 0.5 - 0.5j], [0.0 + 1.0j, 2.0 + 0.0j]]),
    # 256-point window (reference unit-test size), ww = 82
    "n256": dict(
        frames=dict(width=256, height=256, pol_count=1, batch=2, group_count=6,
                    waist=256 * PIX / 6, tilt=(1.0, 1.0), noise="gauss", seed=18),
        config=_cfg(frameWidth=256, frameHeight=256, polCount=1, batchCount=2,
                    fftWindowSizeX=256, fftWindowSizeY=256, tilt=[[1.0, 1.0], [1.0, 1.0]],
                    basisGroupCount=6, basisWaist=[256 * PIX / 6] * 2)),
    # dual-pol with a 24-group basis (300 modes/pol): the tensor-core overlap with per-pol basis operands
    "dualpol_g24": dict(
        frames=dict(width=640, height=256, pol_count=2, batch=2, group_count=24,
                    waist=200e-6, tilt=(1.2, 0.9), noise="poisson", seed=23),
        config=_cfg(frameWidth=640, frameHeight=256, polCount=2, batchCount=2,
                    tilt=[[1.2, 1.2], [0.9, 0.9]], basisGroupCount=24,
                    basisWaist=[200e-6, 180e-6], polLockBasisWaist=0,
                    beamCentre=[[-160 * PIX, 160 * PIX], [0.0, 0.0]])),
    # LG basis: conj(T_LG) applied after the HG overlap (holopipe/engine.py:371-382, hgbasis.py:126-175)
    "lg": dict(
        frames=dict(width=640, height=256, pol_count=2, batch=2, group_count=6,
                    waist=200e-6, tilt=(1.2, 0.9), noise="poisson", seed=31),
        config=_cfg(frameWidth=640, frameHeight=256, polCount=2, batchCount=2,
                    tilt=[[1.2, 1.2], [0.9, 0.9]], basisGroupCount=6, basisType=1,
                    basisWaist=[200e-6, 200e-6], beamCentre=[[-160 * PIX, 160 * PIX], [0.0, 0.0]])),
    # user transform (12 out x 10 in) narrower than the 15 HG modes: only the first 10 enter
    # (holopipe/engine.py:375-380, use = min(hg_count, transform.shape[1]))
    "custom": dict(
        frames=dict(width=320, height=256, pol_count=1, batch=3, group_count=5,
                    waist=200e-6, tilt=(1.0, 1.0), noise="gauss", seed=32),
        config=_cfg(frameWidth=320, frameHeight=256, polCount=1, batchCount=3,
                    tilt=[[1.0, 1.0], [1.0, 1.0]], basisGroupCount=5, basisType=2,
                    basisWaist=[200e-6, 200e-6]),
        custom=dict(seed=33, out=12, inp=10)),
    # SEQUENTIALSWEEP averaging over two wavelengths (holopipe/engine.py:111-113)
    "avg_sweep": dict(
        frames=dict(width=256, height=256, pol_count=1, batch=8, group_count=4,
                    waist=200e-6, tilt=(1.0, 1.0), noise="gauss", seed=34),
        config=_cfg(frameWidth=256, frameHeight=256, polCount=1, batchCount=4, avgCount=2, avgMode=2,
                    wavelengths=[1550e-9, 1580e-9], tilt=[[1.0, 1.0], [1.0, 1.0]],
                    basisGroupCount=4, basisWaist=[200e-6, 200e-6])),
    # process_batch_frequency_sweep_linear (holopipe/engine.py:419-431), output ordering swapped
    "sweep_linear": dict(
        frames=dict(width=256, height=256, pol_count=1, batch=6, group_count=4,
                    waist=200e-6, tilt=(1.0, 1.0), noise="gauss", seed=35),
        config=_cfg(frameWidth=256, frameHeight=256, polCount=1, batchCount=6, wavelengthOrdering=[0, 1],
                    tilt=[[1.0, 1.0], [1.0, 1.0]], basisGroupCount=4, basisWaist=[200e-6, 200e-6]),
        sweep=dict(kind="linear", start=1540e-9, stop=1590e-9, count=3)),
    # process_batch_wavelength_sweep_arbitrary (holopipe/engine.py:433-442)
    "sweep_arbitrary": dict(
        frames=dict(width=320, height=128, pol_count=2, batch=4, group_count=4,
                    waist=120e-6, tilt=(1.0, 1.0), noise="gauss", seed=36),
        config=_cfg(frameWidth=320, frameHeight=128, polCount=2, batchCount=4, wavelengthOrdering=[1, 0],
                    tilt=[[1.0, 1.0], [1.0, 1.0]], basisGroupCount=4, basisWaist=[120e-6, 120e-6],
                    beamCentre=[[-80 * PIX, 80 * PIX], [0.0, 0.0]]),
        sweep=dict(kind="arbitrary", wavelengths=[1575e-9, 1555e-9], count=2)),
    # reference-wave calibration, intensity kind (holopipe/engine.py:276-335)
    "refcal_int": dict(
        frames=dict(width=256, height=256, pol_count=1, batch=3, group_count=6,
                    waist=200e-6, tilt=(1.0, 1.0), noise="gauss", seed=19),
        config=_cfg(frameWidth=256, frameHeight=256, polCount=1, batchCount=3,
                    tilt=[[1.0, 1.0], [1.0, 1.0]], basisGroupCount=6,
                    basisWaist=[200e-6, 200e-6]),
        ref_cal=dict(kind=1, wavelengths=[LAM], seed=21)),
    # reference-wave calibration, field kind, dual-pol, two wavelengths
    "refcal_field": dict(
        frames=dict(width=320, height=128, pol_count=2, batch=4, group_count=4,
                    waist=120e-6, tilt=(1.0, 1.0), noise="gauss", seed=20),
        config=_cfg(frameWidth=320, frameHeight=128, polCount=2, batchCount=4,
                    wavelengths=[1550e-9, 1580e-9],
                    tilt=[[1.0, 1.0], [1.0, 1.0]], defocus=[0.1, 0.1], basisGroupCount=4,
                    basisWaist=[120e-6, 120e-6],
                    beamCentre=[[-80 * PIX, 80 * PIX], [0.0, 0.0]]),
        ref_cal=dict(kind=2, wavelengths=[1550e-9, 1580e-9], seed=22, tilt=(1.0, 1.0))),
}


def make_ref_cal(case):
    """Seeded calibration frames for a case's ``ref_cal`` spec: (kind, raw).

    kind 1: a broad Gaussian beam intensity with 1 % multiplicative noise,
    float32 (Lc, H, W); kind 2: a reference-wave field -- Gaussian amplitude,
    carrier exp(-2 pi i (fx x + fy y)) at the configured tilt and a weak
    low-order phase -- complex64 (Lc, H, W)."""
    import numpy as np
    spec = case["ref_cal"]
    cfg = case["config"]
    W, H = cfg["frameWidth"], cfg["frameHeight"]
    rng = np.random.default_rng(spec["seed"])
    x = (np.arange(W) - W / 2.0) * PIX
    y = (np.arange(H) - H / 2.0) * PIX
    X, Y = np.meshgrid(x, y)
    out = []
    for lam in spec["wavelengths"]:
        x0, y0 = rng.uniform(-0.2, 0.2, 2) * W * PIX / 4
        w0 = W * PIX * rng.uniform(0.6, 0.9)
        amp = np.exp(-((X - x0) ** 2 + (Y - y0) ** 2) / w0 ** 2)
        if spec["kind"] == 1:
            out.append((amp ** 2 * (1.0 + 0.01 * rng.standard_normal(X.shape))).astype(np.float32))
        else:
            tx, ty = spec["tilt"]
            fx, fy = math.sin(math.radians(tx)) / lam, math.sin(math.radians(ty)) / lam
            a, b, c = rng.normal(0.0, 0.5, 3)
            phi = a * (X / w0) + b * (Y / w0) + c * ((X ** 2 + Y ** 2) / w0 ** 2)
            out.append((amp * np.exp(-2j * np.pi * (fx * X + fy * Y) + 1j * phi)).astype(np.complex64))
    return spec["kind"], np.stack(out)


def make_custom(case):
    """Seeded user transform (out x in, complex64) of a case's ``custom`` spec."""
    import numpy as np
    spec = case["custom"]
    rng = np.random.default_rng(spec["seed"])
    t = rng.standard_normal((spec["out"], spec["inp"])) + 1j * rng.standard_normal((spec["out"], spec["inp"]))
    return (t / np.sqrt(spec["inp"])).astype(np.complex64)


def sweep_wavelengths(case):
    """The wavelength list a case's ``sweep`` sets (holopipe/engine.py:419-442)."""
    import numpy as np
    sw = case["sweep"]
    if sw["kind"] == "linear":
        if sw["count"] == 1:
            return [float(sw["start"])]
        f0, f1 = 1.0 / sw["start"], 1.0 / sw["stop"]
        return list(1.0 / (f0 + np.arange(sw["count"]) * (f1 - f0) / (sw["count"] - 1)))
    return [float(v) for v in sw["wavelengths"][:sw["count"]]]
