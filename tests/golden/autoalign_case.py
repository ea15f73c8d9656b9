"""BASELINE config 4 (AutoAlign), normalised as in BASELINE.md section 3 / SURVEY 8(d).

128 frames of 320x256; truth centre (0,0), tilt (1,1) deg, waist 200 um, no
defocus; the starting configuration is perturbed by seeded draws (centre
+-10 px, tilt +-0.1 deg, waist x U(0.9,1.1), defocus U(-0.2,0.2) D); FULL
mode with tilt, centre, defocus and waist enabled.
"""

import math

import numpy as np

LAM, PIX = 1565e-9, 20e-6
WMAX = math.degrees(LAM / (2 * PIX))
FRAMES = dict(width=320, height=256, pol_count=1, batch=128, group_count=9, waist=200e-6,
              tilt=(1.0, 1.0), noise="gauss", seed=4)


def start_config():
    r = np.random.default_rng(44)
    dc = r.uniform(-10, 10, 2) * PIX
    dt = r.uniform(-0.1, 0.1, 2)
    wk = r.uniform(0.9, 1.1)
    df = r.uniform(-0.2, 0.2)
    return dict(frameWidth=320, frameHeight=256, framePixelSize=PIX, polCount=1, batchCount=128,
                wavelengthCentre=LAM, fourierWindowRadius=0.32 * WMAX, fftWindowSizeX=128, fftWindowSizeY=128,
                beamCentre=[[float(dc[0]), 0.0], [float(dc[1]), 0.0]],
                tilt=[[1.0 + float(dt[0])] * 2, [1.0 + float(dt[1])] * 2],
                defocus=[float(df), 0.0], basisGroupCount=9, basisWaist=[200e-6 * float(wk)] * 2,
                autoAlignTilt=1, autoAlignBeamCentre=1, autoAlignDefocus=1, autoAlignBasisWaist=1,
                autoAlignMode=0)
