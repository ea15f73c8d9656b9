"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck), one tool per call:

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Cases: fast128_kernel (SIMT overlap, NT=256 and NT=512), fast128_kernel<TCO> (tcgen05 overlap, G=45), the
large-window lw_* kernels (512^2 window), the two-kernel tensor-core path (fourier128_tc2_kernel + tail42),
the generic fused kernel, and the metric / plane-summary kernels.  Each case checks its result against the
generic kernel so a sanitizer-clean run is also a correct one."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2204_02348_b200 import api  # noqa: E402
from paper_2204_02348_b200.synth import FrameSpec, make_frames  # noqa: E402


def run(name, batch, **flags):
    fspec, cfg = bench.config_for(name, batch=batch)
    frames = make_frames(FrameSpec(**fspec))
    out = {}
    for mode in ("path", "generic"):
        h = api.create_handle()
        eng = api.engine(h)
        for k, v in cfg.items():
            setattr(eng.config, k, v)
        if mode == "generic":
            eng.force_generic = True
        else:
            for k, v in flags.items():
                setattr(eng, k, v)
        api.set_batch(h, batch, torch.from_numpy(frames).cuda())
        eng.run_pipeline(0)
        fr = eng.fields16_device()[0].cpu().numpy()
        co = eng.coefs_device()
        out[mode] = (fr, None if co is None else co.cpu().numpy())
        if mode == "path" and co is not None:
            eng.calc_metrics()
            eng.metric(1)
        api.destroy_handle(h)
    lsb = np.abs(out["path"][0].astype(int) - out["generic"][0]).max()
    print(f"{name} batch={batch} {flags}: max |int16 diff| vs generic = {lsb}", flush=True)
    assert lsb <= 2


if __name__ == "__main__":
    torch.cuda.set_device(0)
    run("dualpol", 80)                                # fast128_kernel<42,42,false,256>: 160 items > 148 SMs
    run("dualpol", 4)                                 # fast128_kernel<...,512>: fewer items than SMs
    run("largebasis", 160)                            # fast128_kernel<42,42,true,256>: tcgen05 HG overlap
    run("dualpol", 80, use_tc2=True)                  # fourier128_tc2_kernel + tail42_kernel
    run("largeframe", 2)                              # lw_rows512 / lw_cols512<FUSE164> / lw_field / lw_pack
    print("sanitize cases done", flush=True)
