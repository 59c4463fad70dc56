"""Cubic half of BASELINE config 1 (no reference routine): the
host spline coefficients against scipy's natural CubicSpline (CPU), and the
GPU kernel against the numpy restatement bitwise (values and brackets)."""
import numpy as np
import pytest
from scipy.interpolate import CubicSpline

import cubic_oracle
from paper_2012_03667_b200.interpolation import interp_cubic_batch, natural_cubic_coefficients


def _table(n=512):
    x = np.logspace(-4, 4, n)
    return x, 1.0 / (1.0 + x) + 0.1 * np.log1p(x)


@pytest.mark.parametrize("n", [2, 3, 4, 7, 512])
def test_coefficients_match_scipy_natural_spline(n):
    x, v = _table(n)
    cf = natural_cubic_coefficients(x, v)
    cs = CubicSpline(x, v, bc_type="natural")
    q = np.exp(np.random.default_rng(n).uniform(np.log(x[0]), np.log(x[-1]), 20000))
    got, _ = cubic_oracle.interp_cubic(x, v, cf, q)
    # few knots over 8 decades: t reaches 1e4 and the Horner terms cancel, so
    # two correct evaluations differ by ~1e-11; 512 knots agree to 1e-13
    tol = 1e-13 if n >= 64 else 1e-10
    assert np.max(np.abs(got - cs(q)) / np.abs(cs(q))) < tol
    assert np.array_equal(cf[:, 0], v[:-1])


def test_oracle_clamps_and_brackets():
    x, v = _table(16)
    cf = natural_cubic_coefficients(x, v)
    q = np.array([x[0] / 2, x[0], x[3], x[-1], 2 * x[-1]])
    val, idx = cubic_oracle.interp_cubic(x, v, cf, q)
    assert list(idx) == [-1, 0, 3, 15, 15]
    # the reference's _bracket_search on NaN ends at 0 (interpolation.py:47-68)
    nv, ni = cubic_oracle.interp_cubic(x, v, cf, np.array([np.nan]))
    assert ni[0] == 0 and np.isnan(nv[0])
    assert val[0] == v[0] and val[1] == v[0] and val[2] == v[3] and val[3] == v[-1] and val[4] == v[-1]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["direct", "search"])
def test_gpu_cubic_bitwise(mode):
    x, v = _table()
    rng = np.random.default_rng(0)
    q = np.exp(rng.uniform(np.log(1e-4), np.log(1e4), 1 << 18))
    q = np.concatenate([q, x, [x[0] / 3, 1e5, x[-1], np.nextafter(x[-1], 0), np.nextafter(x[0], 1),
                               np.nan, np.inf, -np.inf, 0.0]])
    cf = natural_cubic_coefficients(x, v)
    got, gidx = interp_cubic_batch(x, v, q, mode=mode, with_index=True)
    ref, ridx = cubic_oracle.interp_cubic(x, v, cf, q)
    assert np.array_equal(gidx, ridx)
    assert np.array_equal(got, ref, equal_nan=True)


@pytest.mark.gpu
def test_gpu_cubic_non_uniform_knots():
    rng = np.random.default_rng(3)
    x = np.sort(rng.uniform(-5, 5, 300))
    v = np.sin(x)
    q = rng.uniform(-6, 6, 50001)
    cf = natural_cubic_coefficients(x, v)
    got, gidx = interp_cubic_batch(x, v, q, mode="direct", with_index=True)
    ref, ridx = cubic_oracle.interp_cubic(x, v, cf, q)
    assert np.array_equal(gidx, ridx) and np.array_equal(got, ref)
