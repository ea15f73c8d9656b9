"""Benchmark: camera frames/s of the fused FFT -> window -> IFFT -> HG-coefficient
hot path (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config dualpol]
    python bench.py --impl reference ...      # the reference CPU path (holopipe from baseline/_ref)
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one pass of the hot path over one batch of synthetic frames already
resident in HBM (``value``); ``e2e`` is the same metric through the public
API with pinned HOST frames (host->device copy of the step's frames and the
device->host read of its coefficients inside the timed region).  Each rank
processes its own batch (weak scaling; frames are independent, no collective
on the data path).  L2 is flushed (256 MB write) before every timed step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LAM, PIX = 1565e-9, 20e-6
WMAX = np.degrees(LAM / (2 * PIX))

# BASELINE.json configs normalised as in BASELINE.md section 3
WORKLOADS = {
    "pr1": dict(frames=dict(width=256, height=256, pol_count=1, batch=16, group_count=9, waist=200e-6,
                            tilt=(1.0, 1.0), noise="gauss", seed=1),
                G=9, centres=[[0.0, 0.0], [0.0, 0.0]], nx=128),
    "dualpol": dict(frames=dict(width=640, height=256, pol_count=2, batch=1000, group_count=14, waist=200e-6,
                                tilt=(1.2, 0.9), noise="poisson", seed=2),
                    G=14, centres=[[-160 * PIX, 160 * PIX], [0.0, 0.0]], nx=128),
    "largeframe": dict(frames=dict(width=1024, height=1024, pol_count=1, batch=256, group_count=20, waist=1e-3,
                                   tilt=(1.5, 1.5), noise="gauss", zernike_terms=10, seed=3),
                       G=0, centres=[[0.0, 0.0], [0.0, 0.0]], nx=512),
    "autoalign": dict(frames=dict(width=320, height=256, pol_count=1, batch=128, group_count=9, waist=200e-6,
                                  tilt=(1.0, 1.0), noise="gauss", seed=4),
                      G=9, centres=[[0.0, 0.0], [0.0, 0.0]], nx=128),
    "largebasis": dict(frames=dict(width=320, height=256, pol_count=1, batch=8192, group_count=45, waist=200e-6,
                                   tilt=(1.0, 1.0), noise="poisson", seed=5),
                       G=45, centres=[[0.0, 0.0], [0.0, 0.0]], nx=128),
}


def time_autoalign(api, reps=3):
    """BASELINE config 4: AutoAlign time-to-converge from the seeded perturbed start (FULL mode,
    tilt / centre / defocus / waist, IL goal, autoAlignTol 1e-4), best of `reps` on fresh handles."""
    import copy
    import torch
    from paper_2204_02348_b200 import align
    from paper_2204_02348_b200.synth import FrameSpec, make_frames
    from tests.golden.autoalign_case import FRAMES, start_config
    frames = make_frames(FrameSpec(**FRAMES))
    best = None
    for _ in range(reps + 1):   # first run warms the allocator / module state
        h = api.create_handle()
        eng = api.engine(h)
        for k, v in start_config().items():
            setattr(eng.config, k, copy.deepcopy(v))
        eng.config.autoAlignTol = 1e-4
        eng.source.set_float32(frames)
        eng.eval_log = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        goal = align.auto_align(eng)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        api.destroy_handle(h)
        if _ == 0:
            continue
        if best is None or t < best[0]:
            best = (t, len(eng.eval_log), goal)
    t, n, goal = best
    return {"time_to_converge_ms": t * 1e3, "evaluations": n, "us_per_eval": t / max(n, 1) * 1e6,
            "goal": "METRIC_IL", "goal_db": goal, "tol_db": 1e-4,
            "note": "wall clock of api auto_align on the GPU engine (host decisions + GPU evaluations)"}


def config_for(name, batch=None):
    w = WORKLOADS[name]
    f = dict(w["frames"])
    if batch:
        f["batch"] = batch
    tx, ty = f["tilt"]
    cfg = dict(frameWidth=f["width"], frameHeight=f["height"], polCount=f["pol_count"], batchCount=f["batch"],
               framePixelSize=PIX, wavelengthCentre=LAM, fourierWindowRadius=0.32 * WMAX,
               fftWindowSizeX=w["nx"], fftWindowSizeY=w["nx"], tilt=[[tx, tx], [ty, ty]],
               beamCentre=w["centres"], basisGroupCount=w["G"], basisWaist=[f["waist"], f["waist"]])
    return f, cfg


def algorithmic_bytes_per_frame(P, nx, ny, gh, gw, M):
    # window read (f32) + int16 field pair + f32 scale + complex64 coefs
    return P * (nx * ny * 4 + gh * gw * 4 + 4) + P * M * 8


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (B200_PROFILING.md clocks line).

    NVML (nvidia-ml-py) is read every ~0.2 ms from a thread, so a few-millisecond timed region still gets
    a median under load; nvidia-smi (one process per sample) is the fallback."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device):
        """``device``: the CUDA ordinal this rank runs on.  NVML and nvidia-smi number GPUs in PCI order
        and ignore CUDA_VISIBLE_DEVICES, so the GPU is looked up by the UUID torch reports for it."""
        import torch
        self.uuid = None
        try:
            u = str(torch.cuda.get_device_properties(device).uuid)
            self.uuid = u if u.startswith("GPU-") else "GPU-" + u
        except Exception:
            pass
        self.index = self.uuid or str(device)
        self.rows = []      # (sm_mhz, sm_max_mhz, {reason names})
        self.source = "nvml"
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self, nv):
        h, mx = self._nvml
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        while not self._stop.is_set():
            sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((sm, mx, {n for n, b in zip(self.NAMES, bits) if r & b}))
            self._stop.wait(0.0002)

    def _run_smi(self):
        self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    c = [x.strip() for x in out.split(",")]
                    if c[1].replace(".", "").isdigit() and c[2].replace(".", "").isdigit():
                        self.rows.append((float(c[1]), float(c[2]),
                                          {n for n, v in zip(self.NAMES, c[5:9]) if v == "Active"}))
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        if self._nvml is None:
            self._run_smi()
            return
        try:
            import pynvml as nv
            self._run_nvml(nv)
        except Exception:
            self._run_smi()

    def __enter__(self):
        self._nvml = None
        try:   # NVML set up before the timed region starts, so sampling begins with it
            import pynvml as nv
            nv.nvmlInit()
            h = (nv.nvmlDeviceGetHandleByUUID(self.uuid) if self.uuid
                 else nv.nvmlDeviceGetHandleByIndex(int(self.index)))
            self._nvml = (h, float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))
        except Exception:
            self._nvml = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted(set().union(*(r[2] for r in self.rows)))
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": self.source, "gpu_uuid": self.uuid}


def dist_init(n_gpus, need_group=False):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
        if need_group:   # --split on one GPU: the same NCCL code path over a 1-rank group
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
            sk.close()
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                    device_id=torch.device("cuda", 0))
    return rank, world, local


def max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_reference(cfg_dict, frames, min_seconds=10.0, threads=None):
    """Oracle (reference algorithm restated on numpy/scipy) on a bounded host sample."""
    import scipy.fft
    from oracle import holo_oracle as O
    threads = threads or os.cpu_count() or 1
    cfg = O.Cfg(**cfg_dict)
    n = frames.shape[0]
    with scipy.fft.set_workers(threads):
        O.run_chain(cfg, frames)  # warm-up (plans, caches)
        reps, t0 = 0, time.perf_counter()
        while True:
            O.run_chain(cfg, frames)
            reps += 1
            el = time.perf_counter() - t0
            if el >= min_seconds:
                break
    return reps * n / el, threads, reps, el


def holopipe_api():
    """The reference itself -- holopipe, installed UNMODIFIED into baseline/_ref --
    or None when that install is absent (then the oracle port stands in, kind "port")."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "holopipe")):
        return None
    if ref not in sys.path:
        sys.path.append(ref)
    import holopipe.api as R
    return R


def holopipe_rate(R, cfg, frames, threads, steps, warmup):
    """Frames/s of the reference's public API on the host: holopipe.api.process_batch (= Engine.run_pipeline(0)
    + coef_view, holopipe/api.py:854-861) with threadCount = ``threads``; mean over ``steps`` after ``warmup``."""
    B = frames.shape[0]
    h = R.create_handle()
    eng = R.engine(h)
    for k, v in (cfg | {"batchCount": B}).items():
        setattr(eng.config, k, v)
    eng.config.threadCount = threads
    R.set_batch(h, B, frames)
    for _ in range(max(warmup, 1)):
        R.process_batch(h)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        out = R.process_batch(h)
        times.append(time.perf_counter() - t0)
        assert out[1] == B, "reference process_batch failed"
    R.destroy_handle(h)
    return B / float(np.mean(times)), float(np.mean(times))


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation of the path on this box's host cores,
    same workload / metric / unit as the B200 arm.  Rank 0 only (the other ranks exit without work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2204_02348_b200.synth import FrameSpec, make_frames
    B = args.batch or WORKLOADS[args.config]["frames"]["batch"]
    sample = min(args.ref_sample or 1000, B)
    fspec, cfg = config_for(args.config, batch=sample)
    frames = make_frames(FrameSpec(**fspec))
    threads = os.cpu_count() or 1
    R = holopipe_api()
    if R is not None:
        value, sec = holopipe_rate(R, cfg, frames, threads, args.steps, args.warmup)
        kind = "reference"
        what = "holopipe.api.process_batch (baseline/_ref, unmodified reference)"
        # the single-thread row BASELINE.md section 4 promises (threadCount = 1), on a bounded sample
        n1 = min(sample, 64)
        v1, _ = holopipe_rate(R, cfg, frames[:n1], 1, 2, 1)
        single = {"value": v1, "unit": "frames/s", "cores": 1, "sample": f"{n1} frames x 2 steps, threadCount=1"}
    else:
        import scipy.fft
        from oracle import holo_oracle as O
        ocfg = O.Cfg(**cfg)
        with scipy.fft.set_workers(threads):
            for _ in range(max(args.warmup, 1)):
                O.run_chain(ocfg, frames)
            times = []
            for _ in range(args.steps):
                t0 = time.perf_counter()
                O.run_chain(ocfg, frames)
                times.append(time.perf_counter() - t0)
        sec = float(np.mean(times))
        value, kind, single = sample / sec, "port", None
        what = "oracle/holo_oracle.py (numpy+scipy restatement of holopipe; baseline/_ref absent)"
    desc = f"{sample} frames of the '{args.config}' workload per step, {what}, threadCount={threads}"
    line = {
        "impl": "reference", "metric": "camera frames/sec (FFT->IFFT->HG coefs)", "value": value,
        "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.config, "frames_per_step": sample, "same_config": sample == B,
                   "host_cores": threads},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": kind, "sample": desc},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if single is not None:
        line["cpu_baseline"]["threadcount_1"] = single
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="dualpol", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=0, help="override frames per step (per GPU)")
    ap.add_argument("--ref-sample", type=int, default=0, help="reference-arm frames per step (default min(B, 1000))")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tc", action="store_true", help="use the tcgen05 row-pass kernel (HPG_FLAG_TC)")
    ap.add_argument("--simt", action="store_true", help="keep the fused SIMT kernel (HPG_FLAG_SIMT) where the two-kernel "
                    "tensor-core path would be chosen")
    ap.add_argument("--tc2", action="store_true", help="use the two-kernel tensor-core path (HPG_FLAG_TC2)")
    ap.add_argument("--split", action="store_true",
                    help="strong scaling: divide the batch over WORLD_SIZE and include distributed.calc_metrics "
                         "(NCCL all-reduce of the Gram, all-gather of the row sums) in every timed step")
    ap.add_argument("--tile", type=int, default=0,
                    help="generate this many distinct frames and tile them in HBM up to the batch (config 5: 1024)")
    ap.add_argument("--traffic-bytes", type=float, default=None,
                    help="dram read+write bytes per launch from an ncu --set full capture")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    rank, world, local = dist_init(args.gpus, need_group=args.split)
    from paper_2204_02348_b200 import api, native
    from paper_2204_02348_b200.synth import FrameSpec, make_frames

    fspec, cfg = config_for(args.config, batch=args.batch or None)
    B_total = fspec["batch"]
    if args.split:   # strong scaling: the batch is divided over the ranks (distributed.shard)
        from paper_2204_02348_b200 import distributed as D
        r0, r1 = D.shard(B_total, world, rank)
        B = r1 - r0
    else:            # weak scaling: every rank processes its own full batch
        B = B_total
    cfg = dict(cfg, batchCount=B)
    n_distinct = min(B, args.tile) if args.tile else B
    fspec = dict(fspec, batch=n_distinct, seed=fspec["seed"] * 1000 + rank)
    frames_host = make_frames(FrameSpec(**fspec))
    dev = torch.device("cuda", torch.cuda.current_device())

    h = api.create_handle()
    eng = api.engine(h)
    eng.use_tc = args.tc
    eng.force_simt = args.simt
    eng.use_tc2 = args.tc2
    for k, v in cfg.items():
        setattr(eng.config, k, v)
    frames_dev = torch.from_numpy(frames_host).to(dev)
    if n_distinct < B:   # BASELINE config 5 at its full size: distinct frames tiled in HBM (21.5 GB at 65,536)
        reps = -(-B // n_distinct)
        frames_dev = frames_dev.repeat(reps, 1, 1)[:B].contiguous()
    api.set_batch(h, B, frames_dev)
    eng.run_pipeline(0)
    torch.cuda.synchronize()

    # the timed unit: one fused kernel launch through the C ABI (hpg_run) on device frames
    P, nx, ny = cfg["polCount"], cfg["fftWindowSizeX"], cfg["fftWindowSizeY"]
    gh, gw = eng._field_r.shape[-2:]
    M = eng._mode_count
    bpf = algorithmic_bytes_per_frame(P, nx, ny, gh, gw, M)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    launch = eng.prepare_launch()   # one hpg_run on the resident frames, arguments pre-built
    stream_h = native.stream_handle()

    metric_launches = 0
    if args.split:   # the step includes the metric reduction over the process group (NCCL)
        from paper_2204_02348_b200 import distributed as D
        L_wl = len(eng.config.wavelength_list())
        metric_launches = 2 * L_wl   # hpg_metric_partials: row + Gram kernels per wavelength

        def step():
            launch.launch(stream_h)
            D.calc_metrics(eng, defer_mdl=True)
    else:
        def step():
            launch.launch(stream_h)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clocks:
        for i in range(args.steps):
            flush.zero_()
            starts[i].record()
            step()
            ends[i].record()
        torch.cuda.synchronize()
    barrier(world)
    launches_per_step = int(native.lib().hpg_last_launch_count())   # kernels the last hpg_run launched
    per_step = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_local = float(np.mean(per_step))
    ms = max_over_ranks(ms_local, world)
    value = (B_total if args.split else B * world) / (ms / 1e3)
    achieved = bpf * B / (ms_local / 1e3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))

    # DRAM traffic of the dominant kernel per launch, from the committed `ncu --set full`
    # capture of the same command (profiles/ncu_traffic.json); rescaled per launch size
    fast_geom = nx == 128 and ny == 128 and gh == 42 and gw == 42
    if args.tc2 or (fast_geom and not args.tc and launches_per_step == 2):
        # the two-kernel tensor-core path (chosen by hpg_run for large batches): the roofline is taken over
        # the whole step (both kernels), against the same algorithmic bytes
        kernel_name = "holo::fourier128_tc2_kernel+holo::tail42p_kernel"
    elif args.tc:
        kernel_name = "holo::fast128tc_kernel<42,42>"
    elif fast_geom:
        kernel_name = "holo::fast128_kernel<42,42>"
    elif nx == 512 and ny == 512:
        # one hpg_run = the five L2-chunked large-window kernels; the roofline is taken over all of them
        kernel_name = "holo::lw_rows512+lw_cols512+lw_ifft_y+lw_field+lw_pack (large-window path)"
    else:
        kernel_name = "holo::fused_kernel"
    traffic = args.traffic_bytes
    if traffic is None:
        try:
            with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")) as fh:
                rec = json.load(fh).get(f"{args.config}/{kernel_name}")
            if rec:
                traffic = rec["dram_bytes_per_launch"] * B / rec["frames_per_launch"]
        except (OSError, ValueError, KeyError):
            traffic = None

    # ---------------- e2e through the public API with host frames (H2D + kernel + D2H in the timed region)
    def time_e2e(setter, host, reps):
        setter(host)
        for _ in range(2):
            api.process_batch(h)
        torch.cuda.synchronize()
        e_ms = []
        barrier(world)
        for i in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            coefs, b, m, p = api.process_batch(h)       # H2D frames, kernel, D2H coefs
            if coefs is None:                            # fields-only workload: read the int16 fields back
                out = api.get_fields16(h)
                d2h = int(out[0].nbytes + out[1].nbytes + out[2].nbytes)
            else:
                d2h = int(coefs.nbytes)
            e.record()
            e.synchronize()
            e_ms.append(s.elapsed_time(e))
        barrier(world)
        em = max_over_ranks(float(np.median(e_ms)), world)   # median step (host scheduling jitter)
        return {"value": B * world / (em / 1e3), "unit": "frames/s",
                "h2d_bytes_per_step": int(eng.last_h2d_bytes), "d2h_bytes_per_step": d2h,
                "ms_per_step": em, "steps": len(e_ms), "stat": "median"}

    e2e = None
    e2e_variants = {}
    host_bytes = B * frames_host[0].nbytes
    if not args.no_e2e and (host_bytes > 8e9 or args.split):
        e2e_variants["skipped"] = (f"{host_bytes / 1e9:.1f} GB of host frames per step (device-tiled workload)"
                                   if host_bytes > 8e9 else "split mode times the sharded device path")
    elif not args.no_e2e:
        reps = max(5, min(args.steps, 20))
        pinned = torch.from_numpy(frames_host).pin_memory()
        e2e = time_e2e(lambda x: api.set_batch(h, B, x), pinned, reps)
        e2e["path"] = ("api.process_batch on pinned host frames: window-only H2D (hpg_upload_windows), "
                       "fused kernel, D2H of the coefficients (of the int16 fields when there is no basis)")
        del pinned
        # the drop-in caller's buffer: a pageable numpy array, exactly as holopipe.api.set_batch receives it
        v = time_e2e(lambda x: api.set_batch(h, B, x), frames_host, reps)
        v["path"] = "api.set_batch(numpy float32, pageable) + api.process_batch"
        e2e_variants["pageable_numpy_f32"] = v
        if np.array_equal(frames_host, np.round(frames_host)) and frames_host.min() >= 0 and frames_host.max() < 65536:
            # camera format (holopipe/frames.py:49-59): the same integer frames as uint16, half the PCIe bytes
            u16 = torch.from_numpy(frames_host.astype(np.uint16)).pin_memory()
            v = time_e2e(lambda x: api.set_batch_uint16(h, B, x), u16, reps)
            v["path"] = "api.set_batch_uint16(pinned uint16 frames) + api.process_batch"
            e2e_variants["pinned_u16"] = v
            u16np = frames_host.astype(np.uint16)
            v = time_e2e(lambda x: api.set_batch_uint16(h, B, x), u16np, reps)
            v["path"] = "api.set_batch_uint16(numpy uint16, pageable) + api.process_batch"
            e2e_variants["pageable_numpy_u16"] = v
            del u16, u16np
        api.set_batch(h, B, frames_dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = min(B, 256)
        R = holopipe_api()
        if R is not None:   # the reference itself, ~cpu_seconds of host work
            threads = os.cpu_count() or 1
            v0, sec0 = holopipe_rate(R, cfg, frames_host[:sample], threads, 1, 1)
            reps = max(1, int(args.cpu_seconds / max(sec0, 1e-3)))
            v, sec = holopipe_rate(R, cfg, frames_host[:sample], threads, reps, 0)
            cpu = {"value": v, "unit": "frames/s", "cores": threads, "kind": "reference",
                   "sample": f"{sample} frames x {reps} steps ({reps * sec:.1f} s) of the same workload; "
                             f"holopipe.api.process_batch from baseline/_ref, threadCount={threads}"}
        else:
            v, threads, reps, el = cpu_reference(cfg | {"batchCount": sample}, frames_host[:sample],
                                                 min_seconds=args.cpu_seconds)
            cpu = {"value": v, "unit": "frames/s", "cores": threads, "kind": "port",
                   "sample": f"{sample} frames x {reps} reps ({el:.1f} s) of the same workload; "
                             f"oracle/holo_oracle.py (numpy+scipy restatement of holopipe)"}

    autoalign = None
    if rank == 0 and args.config == "autoalign":
        autoalign = time_autoalign(api)

    if rank == 0:
        line = {
            "metric": "camera frames/sec (FFT->IFFT->HG coefs)", "value": value, "unit": "frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if args.split else "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded HG superposition holograms, BASELINE.md section 3)",
            "config": {"workload": args.config, "frames_per_step_per_gpu": B, "frame": [fspec["height"], fspec["width"]],
                       "pols": P, "fft_window": [ny, nx], "field": [int(gh), int(gw)], "modes_per_pol": int(M),
                       "l2": "flushed (256 MB write) before every timed step", "parallelism": f"dp{world}",
                       "frames_total": B_total if args.split else B * world,
                       "distinct_frames_per_gpu": n_distinct,
                       "metrics_in_step": "distributed.calc_metrics over NCCL (MDL deferred)" if args.split else None},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kernel_name, "bytes_per_frame": bpf,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_variants": e2e_variants or None,
            "gpu_launches": (launches_per_step + metric_launches) * args.steps,
            "clocks": clocks.summary(),
        }
        if autoalign is not None:
            line["autoalign"] = autoalign
        print(json.dumps(line), flush=True)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
