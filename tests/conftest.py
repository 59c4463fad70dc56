import os
import sys
import types

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libdse_b200.so)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_grid(tag):
    """MomentumGrid-like object holding the reference's own grid arrays."""
    z = golden(f"grid_{tag}.npz")
    d = {k: z[k] for k in z.files if k not in ("args", "p2_range", "call")}
    g = types.SimpleNamespace(**d)
    g.n_ext, g.m_rad, g.m_ang = g.p2_ext.size, g.q2_int.size, g.z_nodes.size
    return g


def params_ns(D=0.55, omega=0.678, m0=0.0, z1=1.0, xi=1e-10, relaxation=1.0, max_iterations=1, coeff=None):
    from paper_2012_03667_b200 import ModelParams
    p = ModelParams(D=D, omega=omega, m0=m0, z1=z1, xi=xi, relaxation=relaxation, max_iterations=max_iterations)
    if coeff is not None:
        assert p.interaction_coeff == coeff
    return p


def hybrid_rel(x, ref, floor=1e-6):
    """SURVEY.md §8c parity measure: relative error where |ref| >= floor*max|ref|,
    else absolute error / max|ref|."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    m = float(np.max(np.abs(ref)))
    if m == 0.0:
        return float(np.max(np.abs(x - ref)))
    big = np.abs(ref) >= floor * m
    err = np.abs(x - ref)
    r = np.where(big, err / np.where(big, np.abs(ref), 1.0), err / m)
    return float(np.max(r))


@pytest.fixture(scope="session")
def gpu_available():
    try:
        from paper_2012_03667_b200 import _native
        _native.device_info(0)
        return True
    except Exception:  # noqa: BLE001
        return False
