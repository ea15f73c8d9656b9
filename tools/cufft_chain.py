"""Library comparison row: the same per-frame chain as fast128_kernel written with cuFFT (torch.fft) and
cuBLAS (torch.matmul) on device-resident frames -- window extraction, rfft2, crop of the off-axis window
(wrap + Hermitian partner, holopipe/pipeline.py:79-104), mask x recentring phase (:72-127), ifftshift + ifft2
at 42 x 42 (:130-149), removal phase (:163-185), int16 packing (:188-199) and the separable HG overlap
(hgbasis.py:101-116).  Tables come from the engine's native plan (origins, k0, axes, quantised basis) plus
the reference formulas restated here; the int16 fields / coefficients are checked against the fused kernel,
then both are timed the same way as bench.py (CUDA events, L2 flushed before every step).

    python tools/cufft_chain.py [--steps 20] [--warmup 5]
"""
import argparse
import json
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_02348_b200 import api  # noqa: E402
from paper_2204_02348_b200.synth import FrameSpec, make_frames  # noqa: E402


def tables(eng, cfg):
    """Per-pol constant tables of the chain (device tensors)."""
    plan = eng._native_plan(eng._plan_key(cfg["basisGroupCount"], eng._effective()[2]))
    info = plan.info
    P, nx, ny, p = cfg["polCount"], cfg["fftWindowSizeX"], cfg["fftWindowSizeY"], cfg["framePixelSize"]
    W, H, lam = cfg["frameWidth"], cfg["frameHeight"], cfg["wavelengthCentre"]
    wh, ww = info.wh, info.ww
    fr = math.sin(math.radians(cfg["fourierWindowRadius"])) / lam
    xa, ya = plan.axes()
    G = cfg["basisGroupCount"]
    hx, hy = plan.basis(P, G) if G > 0 else (np.zeros((P, 0, info.gw)), np.zeros((P, 0, info.gh)))
    dev = torch.device("cuda", 0)
    T = {"origins": [], "rows": [], "cols": [], "conj": [], "win": [], "rem": [], "wh": wh, "ww": ww, "G": G,
         "hx": torch.as_tensor(hx, dtype=torch.complex64, device=dev),
         "hy": torch.as_tensor(hy, dtype=torch.complex64, device=dev)}
    fx = (np.arange(ww) - ww // 2) / (nx * p)
    fy = (np.arange(wh) - wh // 2) / (ny * p)
    mask = fy[:, None] ** 2 + fx[None, :] ** 2 <= fr * fr + 1e-30
    for q in range(P):
        col0, row0 = int(info.col0[q]), int(info.row0[q])
        k0x, k0y = int(info.k0[q][0][0]), int(info.k0[q][0][1])
        bcx, bcy = cfg["beamCentre"][0][q], cfg["beamCentre"][1][q]
        xi_x, xi_y = bcx / p + W / 2.0 - col0, bcy / p + H / 2.0 - row0
        bx = k0x + np.arange(ww) - ww // 2
        by = k0y + np.arange(wh) - wh // 2
        mx, my = np.mod(bx, nx), np.mod(by, ny)
        keep = mx <= nx // 2
        col = np.broadcast_to(np.where(keep, mx, nx - mx)[None, :], (wh, ww))
        row = np.where(keep[None, :], my[:, None], np.mod(-by, ny)[:, None])
        ex = np.exp(2j * np.pi * bx * (xi_x - nx / 2.0) / nx)
        ey = np.exp(2j * np.pi * by * (xi_y - ny / 2.0) / ny)
        win = (mask * (ey[:, None] * ex[None, :]).astype(np.complex64)).astype(np.complex64)
        tx, ty = cfg["tilt"][0][q], cfg["tilt"][1][q]
        fxl, fyl = np.sin(np.radians(tx)) / lam, np.sin(np.radians(ty)) / lam
        rx, ry = fxl - k0x / (nx * p), fyl - k0y / (ny * p)
        c = 2.0 * np.pi * (fxl * bcx + fyl * bcy) - np.pi * (k0x + k0y)
        x, y = xa.astype(np.float64), ya.astype(np.float64)
        rem = np.exp(-1j * (c + (2 * np.pi * rx * x)[None, :] + (2 * np.pi * ry * y)[:, None])).astype(np.complex64)
        T["origins"].append((col0, row0))
        T["rows"].append(torch.as_tensor(row, device=dev))
        T["cols"].append(torch.as_tensor(np.ascontiguousarray(col), device=dev))
        T["conj"].append(torch.as_tensor(np.broadcast_to(~keep[None, :], (wh, ww)).copy(), device=dev))
        T["win"].append(torch.as_tensor(win, device=dev))
        T["rem"].append(torch.as_tensor(rem, device=dev))
    dxdy = np.complex64(float(abs(xa[1] - xa[0])) * float(abs(ya[1] - ya[0])))
    T["dxdy"] = complex(dxdy)
    ms = [(g - n, n) for g in range(G) for n in range(g + 1)]
    T["mi"] = torch.as_tensor([m for m, _ in ms], device=dev)
    T["ni"] = torch.as_tensor([n for _, n in ms], device=dev)
    return T


def chain(frames, T, nx, ny):
    """One pass over a device batch [B][H][W] float32 -> (fr, fi, scale, coefs)."""
    outs = []
    for q, (c0, r0) in enumerate(T["origins"]):
        plane = torch.fft.rfft2(frames[:, r0:r0 + ny, c0:c0 + nx])                 # (B, ny, nx/2+1)
        crop = plane[:, T["rows"][q], T["cols"][q]]                                 # (B, wh, ww)
        crop = torch.where(T["conj"][q], crop.conj(), crop) * T["win"][q]
        field = torch.fft.ifft2(torch.fft.ifftshift(crop, dim=(-2, -1))) * (crop.shape[-1] * crop.shape[-2]
                                                                          / float(nx * ny))
        field = field * T["rem"][q]
        peak = torch.maximum(field.real.abs().amax(dim=(-2, -1)), field.imag.abs().amax(dim=(-2, -1)))
        scale = torch.where(peak > 0, (32767.0 / peak.double()).float(), torch.ones_like(peak))
        fr = torch.round(field.real * scale[:, None, None]).to(torch.int16)
        fi = torch.round(field.imag * scale[:, None, None]).to(torch.int16)
        if T["G"] > 0:
            deq = torch.complex(fr.float(), fi.float()) / scale[:, None, None]
            t = torch.matmul(torch.matmul(T["hy"][q], deq), T["hx"][q].transpose(0, 1)) * T["dxdy"]   # (B, G, G)
            coefs = t[:, T["ni"], T["mi"]]
        else:
            coefs = fr.new_zeros((fr.shape[0], 0), dtype=torch.complex64)
        outs.append((fr, fi, scale, coefs))
    fr = torch.stack([o[0] for o in outs], 1)
    fi = torch.stack([o[1] for o in outs], 1)
    sc = torch.stack([o[2] for o in outs], 1)
    co = torch.cat([o[3] for o in outs], 1)
    return fr, fi, sc, co


def timed(fn, steps, warmup, flush):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.mean(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="dualpol")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    fspec, cfg = bench.config_for(args.config)
    B = fspec["batch"]
    frames = torch.from_numpy(make_frames(FrameSpec(**fspec))).cuda()
    h = api.create_handle()
    eng = api.engine(h)
    for k, v in cfg.items():
        setattr(eng.config, k, v)
    cfg = dict(cfg, framePixelSize=bench.PIX, wavelengthCentre=bench.LAM)
    api.set_batch(h, B, frames)
    eng.run_pipeline(0)
    T = tables(eng, cfg)
    nx, ny = cfg["fftWindowSizeX"], cfg["fftWindowSizeY"]
    lib = chain(frames, T, nx, ny)
    fr, fi, sc = (t.cpu().numpy() for t in eng.fields16_device())
    co = eng.coefs_device().cpu().numpy() if T["G"] > 0 else None
    lfr, lfi, lsc, lco = (t.cpu().numpy() for t in lib)
    dq = lambda r, i, s: (r.astype(np.float32) + 1j * i.astype(np.float32)) / s[..., None, None]   # noqa: E731
    P = len(T["origins"])
    a, b = dq(fr, fi, sc).reshape(B * P, -1), dq(lfr, lfi, lsc).reshape(B * P, -1)
    field_err = float(np.max(np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)))
    coef_err = float(np.max(np.linalg.norm(co - lco, axis=1) / np.linalg.norm(lco, axis=1))) if co is not None else None
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    launch = eng.prepare_launch()
    t_fused = timed(lambda: launch.launch(), args.steps, args.warmup, flush)
    t_lib = timed(lambda: chain(frames, T, nx, ny), args.steps, args.warmup, flush)
    print(json.dumps({"config": args.config, "frames": B, "fields_rel_l2_max": field_err, "coefs_rel_l2_max": coef_err,
                      "fused_ms": t_fused, "cufft_cublas_ms": t_lib, "fused_frames_per_s": B / t_fused * 1e3,
                      "cufft_cublas_frames_per_s": B / t_lib * 1e3, "speedup": t_lib / t_fused}))


if __name__ == "__main__":
    main()
