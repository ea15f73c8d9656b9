"""Reference output files (holopipe/settings.py:195-293: write_fields / write_coefs / write_summary) for the
'pr1' golden case, written by the REFERENCE itself.  Run in the build container:

    python tests/golden/make_writer_golden.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from holopipe import api as R  # noqa: E402
from holopipe import settings as S  # noqa: E402

from paper_2204_02348_b200.synth import FrameSpec, make_frames  # noqa: E402
from tests.golden.cases import CASES  # noqa: E402


def main():
    case = CASES["pr1"]
    frames = make_frames(FrameSpec(**case["frames"]))
    h = R.create_handle()
    eng = R.engine(h)
    for k, v in case["config"].items():
        setattr(eng.config, k, v)
    eng.config.threadCount = 1
    R.set_batch(h, case["config"]["batchCount"], frames)
    R.process_batch(h)
    R.auto_align_calc_metrics(h)
    out = os.path.join(HERE, "writers")
    os.makedirs(out, exist_ok=True)
    S.write_fields(h, os.path.join(out, "pr1_fields.bin"))
    S.write_coefs(h, os.path.join(out, "pr1_coefs.bin"))
    S.write_summary(h, os.path.join(out, "pr1_summary.txt"))
    R.destroy_handle(h)


if __name__ == "__main__":
    main()
