"""The C-ABI library loads and exports every symbol include/holo_b200.h declares (CPU)."""

import ctypes
import os
import re

from paper_2204_02348_b200 import native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "holo_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(hpg_\w+)\s*\(", src, re.M)))


def test_header_declares_expected_entry_points():
    assert set(_declared()) == set(native.EXPORTS)


def test_library_loads_and_exports_all_symbols():
    lib = native.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.hpg_version() >= 1


def test_struct_sizes_match_header_layout():
    # 8-byte alignment of the double block after 10 int32 fields
    assert ctypes.sizeof(native.PlanDesc) == 10 * 4 + 3 * 8 + 8 + 4 * 4 * 8 + 2 * 8 * 2
    assert native.Batch.frame_count.offset == 16
