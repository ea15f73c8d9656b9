"""api.benchmark: per-stage throughput of the GPU engine (holopipe/bench.py:30-54).

Same contract as the reference: ``(batchesPerSecond, info[6])`` with one rate per
BENCHMARK_* slot (FFT, IFFT, APPLYTILT, BASIS, OVERLAP, TOTAL), every rate a whole
batch per second, TOTAL a full ``run_pipeline(0)``.  Each stage runs back to back on
the engine's stream for about ``goal_duration / 6`` seconds and is timed with CUDA
events recorded on that stream around the loop (the events also capture the host
work a stage does between its launches, e.g. plan construction for BASIS).
"""

from __future__ import annotations

import time

import numpy as np

from . import constants as C


def _rate(eng, func, budget):
    """Stage calls per second, device time between CUDA events bracketing the loop."""
    import torch
    func()   # warm-up outside the timed region
    with torch.cuda.device(eng.device):
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        start.record()
        calls = 0
        t0 = time.perf_counter()
        while True:
            func()
            calls += 1
            if calls >= 2 and time.perf_counter() - t0 >= budget:
                break
        stop.record()
        stop.synchronize()
        ms = start.elapsed_time(stop)
    return calls / max(ms * 1e-3, 1e-9)


def benchmark(eng, goal_duration=1.0):
    if goal_duration <= 0:
        goal_duration = 1.0
    eng.run_pipeline(0)   # plans, buffers and device products in place
    budget = goal_duration / C.BENCHMARK_COUNT

    def regenerate_basis():
        # holopipe rebuilds the HG tables (engine.py:339-351); here they live in the native plan
        if eng.config.basisGroupCount >= 1:
            key = eng._plan_key(eng.config.basisGroupCount, eng._effective()[2])
            eng._plans.pop(key, None)   # the dropped plan frees its tables when released
            eng._native_plan(key)

    stages = {
        C.BENCHMARK_FFT: eng.process_fft,
        C.BENCHMARK_IFFT: eng.process_ifft,
        C.BENCHMARK_APPLYTILT: eng.process_remove_tilt,
        C.BENCHMARK_BASIS: regenerate_basis,
        C.BENCHMARK_OVERLAP: eng.extract_coefs,
        C.BENCHMARK_TOTAL: lambda: eng.run_pipeline(0),
    }
    info = np.zeros(C.BENCHMARK_COUNT, dtype=np.float32)
    for idx, func in stages.items():
        info[idx] = _rate(eng, func, budget)
    return float(info[C.BENCHMARK_TOTAL]), info
