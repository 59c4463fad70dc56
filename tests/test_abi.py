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
                # any import or load of the checker: oracle, mu_oracle, cubic_oracle,
                # mu_dirac, liboracle_*.so, the C restatement's symbols
                assert not re.search(r"import\s+[\w.]*(oracle|mu_dirac)|from\s+[\w.]*(oracle|mu_dirac)\b|"
                                     r"liboracle|dse_oracle|oracle_(sweep|solve|mu)|(mu|cubic)_oracle\.(?!py)|"
                                     r"sys\.path[^\n]*oracle|CDLL\([^)]*oracle", txt), f


def test_anderson_state_argument_validation_without_gpu():
    """dse_mu_aa_residual / dse_mu_aa_update reject bad shapes before any CUDA
    call (DSE_EPARAM -> ParameterError), and the Python state checks the
    depth the kernels support (1..16)."""
    from paper_2012_03667_b200.errors import ParameterError
    from paper_2012_03667_b200.finite_mu import _DeviceAnderson
    lib = _native.load()
    err = _native.DseErr()
    cols = (ctypes.c_int32 * 4)(0, 1, 2, 3)
    host = np.zeros(64)
    hp = host.ctypes.data_as(_native.f64p)
    # S = 5 solves (max 4), depth 17 (max 16), ncols > depth
    for S, depth, slot, ncols in ((5, 4, 0, 1), (1, 17, 0, 1), (1, 2, 0, 3), (1, 2, 0, 4)):
        rc = lib.dse_mu_aa_residual(S, 8, 1, 1, 1, 1, 1, 1, 1, depth, slot, cols, ncols, 1, hp, 0, ctypes.byref(err))
        assert rc == _native.DSE_EPARAM, (S, depth, ncols)
        rc = lib.dse_mu_aa_update(S, 8, 1, 1, 1, 1, depth, cols, ncols, hp, 1.0, 0, ctypes.byref(err))
        assert rc == _native.DSE_EPARAM
    bad_cols = (ctypes.c_int32 * 2)(0, 5)  # slot 5 of a depth-2 ring
    rc = lib.dse_mu_aa_residual(1, 8, 1, 1, 1, 1, 1, 1, 1, 2, 0, bad_cols, 2, 1, hp, 0, ctypes.byref(err))
    assert rc == _native.DSE_EPARAM and b"slot" in err.msg
    # null state pointers
    rc = lib.dse_mu_aa_residual(1, 8, None, 1, 1, 1, 1, 1, 1, 2, -1, cols, 0, 1, hp, 0, ctypes.byref(err))
    assert rc == _native.DSE_EPARAM and err.msg
    for depth in (0, 17):
        with pytest.raises(ParameterError):
            _DeviceAnderson(1, 8, depth, 1.0, "cpu", 0)
