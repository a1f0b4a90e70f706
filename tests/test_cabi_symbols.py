"""The C-ABI library loads and exports every symbol include/lvx.h declares (no compute calls)."""
import ctypes
import os
import re

import pytest

from paper_2510_09081_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(ROOT, "include", "lvx.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lvx_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_functions():
    names = declared()
    assert "lvx_voxelize" in names and "lvx_render" in names and len(names) >= 20


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.fail(f"{_native.LIB_PATH} missing: run __graft_entry__.build()")
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert sorted(_native.SIGNATURES) == declared()


def test_pure_host_entry_points():
    lib = _native.lib()
    assert lib.lvx_version() >= 100
    assert lib.lvx_num_levels(256) == 9 and lib.lvx_num_levels(100) < 0
    assert lib.lvx_pyramid_elems(64) == sum((64 >> l) ** 3 for l in range(7))
    assert lib.lvx_scan_scratch_bytes(64 ** 3) > 0 and lib.lvx_list_words(8) == 8 + 16
    assert lib.lvx_cull_scratch_words(7) < 0


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2510_09081_b200 as lvx
    with pytest.raises(_native.LvxError):
        lvx.voxelize(lvx.generate("helix"), None, lvx.GridDesc(8, np.zeros(3), 1.0))
