"""CPU: the C-ABI library loads and exports every symbol include/dse_b200.h
declares; without a GPU the product fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2012_03667_b200 import _native


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "dse_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dse_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_header_symbols():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_native.EXPORTED_SYMBOLS) == syms


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_native.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_no_gpu_fails_loudly(gpu_available):
    if gpu_available:
        pytest.skip("GPU present")
    import paper_2012_03667_b200 as p
    g = p.build_grid(8, 8, 4, 1e-6, 1e4)
    with pytest.raises(p.ExecutionEnvironmentError):
        p.iterate_once(g, np.ones(8), np.ones(8), p.ModelParams(), p.VARIANTS["indexed-gpu"])
    with pytest.raises(p.ExecutionEnvironmentError):
        p.interp_search_many(np.array([1.0, 2.0]), np.array([1.0, 2.0]), np.array([1.5]))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2012_03667_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"import\s+oracle|from\s+oracle|liboracle_dse|dse_oracle", txt), f
