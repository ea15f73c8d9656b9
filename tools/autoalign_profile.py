"""cProfile of api-level AutoAlign (config 4 start, device-resident frames): where the host time goes."""
import cProfile, pstats, sys, copy, time
sys.path.insert(0,'.')
import numpy as np, torch
from paper_2204_02348_b200 import align
from paper_2204_02348_b200.engine import Engine
from paper_2204_02348_b200.synth import FrameSpec, make_frames
from tests.golden.autoalign_case import FRAMES, start_config
frames = make_frames(FrameSpec(**FRAMES))
fd = torch.from_numpy(frames).cuda()
def run():
    eng = Engine()
    for k, v in start_config().items(): setattr(eng.config, k, copy.deepcopy(v))
    eng.config.autoAlignTol = 1e-4
    eng.source.set_float32(fd)
    t0=time.perf_counter(); align.auto_align(eng); return time.perf_counter()-t0
run()
print("plain", run())
pr = cProfile.Profile(); pr.enable(); run(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
