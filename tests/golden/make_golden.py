"""Generate golden fixtures by running the REFERENCE (holopipe) itself.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

For every case below, seeded frames are generated with
``paper_2204_02348_b200.synth`` (their sha256 is stored so the GPU box can
check it regenerated identical inputs), the reference ``holopipe.engine.Engine``
is configured exactly like the case's config, ``run_pipeline(0)`` +
``calc_metrics`` are run, and the reference's own outputs are saved to
``tests/golden/<case>.npz``.  Nothing here is used at run time on the GPU box:
only the .npz files travel.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from paper_2204_02348_b200.synth import FrameSpec, make_frames, frames_digest  # noqa: E402
from tests.golden.cases import CASES, make_custom, make_ref_cal  # noqa: E402


def run_reference(case):
    from holopipe.engine import Engine
    spec = FrameSpec(**case["frames"])
    frames = make_frames(spec)
    eng = Engine()
    cfg = eng.config
    for k, v in case["config"].items():
        setattr(cfg, k, v)
    cfg.threadCount = 1
    eng.source.set_float32(frames)
    batch_cal = case.get("batch_cal")
    if batch_cal is not None:
        arr = np.asarray(batch_cal, np.complex64)
        eng.set_batch_calibration(arr.reshape(-1), arr.shape[0], arr.shape[1])
    if case.get("ref_cal") is not None:
        kind, raw = make_ref_cal(case)
        Lc, Hc, Wc = raw.shape
        if kind == 1:
            eng.ref_cal.set_intensity(raw, Lc, Wc, Hc)
        else:
            eng.ref_cal.set_field(raw, Lc, Wc, Hc)
    if case.get("custom") is not None:
        eng.custom_transform = make_custom(case)
    sweep = case.get("sweep")
    if sweep is None:
        eng.run_pipeline(0)
    elif sweep["kind"] == "linear":
        eng.process_batch_frequency_sweep_linear(sweep["start"], sweep["stop"], sweep["count"])
    else:
        eng.process_batch_wavelength_sweep_arbitrary(np.asarray(sweep["wavelengths"]), sweep["count"])
    out = {
        "frames_sha256": np.array(frames_digest(frames)),
        "fr": eng._field_r, "fi": eng._field_i, "scale": eng._field_scale,
        "x_axis": eng._field_axes[0], "y_axis": eng._field_axes[1],
        "field_params": eng._summary_field.parameters,
        "field_inten": eng._summary_field.total_intensity,
        "k0": eng._window_meta["k0"],
        "origins": np.array(eng._plan["origins"]),
    }
    if case.get("ref_cal") is not None:
        out["ref_applied"] = eng._ref_applied
    if case.get("store_fourier"):
        out["fourier_params"] = eng._summary_fourier.parameters
        out["fourier_inten"] = eng._summary_fourier.total_intensity
        out["window"] = eng._window
    if cfg.basisGroupCount >= 1:
        coefs, b, m, p = eng.coef_view()
        out["coefs"] = coefs
        eng.calc_metrics()
        out["metrics"] = np.stack([eng.metrics_array(i) for i in range(9)])
    return out


def main(names=None):
    import scipy
    meta = {"numpy": np.__version__, "scipy": scipy.__version__, "cases": {}}
    for name, case in CASES.items():
        if names and name not in names:
            continue
        out = run_reference(case)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        meta["cases"][name] = {k: list(np.shape(v)) for k, v in out.items()}
        print(name, {k: np.shape(v) for k, v in out.items()})
    path = os.path.join(HERE, "golden_meta.json")
    if names and os.path.exists(path):
        old = json.load(open(path))
        old["cases"].update(meta["cases"])
        meta["cases"] = old["cases"]
    with open(path, "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or None)
