"""CPU oracle of the batched cubic interpolation (BASELINE config 1, cubic half).

TEST INFRASTRUCTURE ONLY (tests/, bench.py's cpu leg).  The reference has no
cubic routine: parity is against this numpy restatement of the
kernel's arithmetic (bitwise: same brackets as interpolation.py:47-68, same
clamping as :84-97, Horner order a + t (b + t (c + t d))) and, for the
spline itself, scipy.interpolate.CubicSpline(bc_type="natural").
"""
from __future__ import annotations

import numpy as np


def brackets(x, q):
    """_bracket_search semantics (interpolation.py:47-68): searchsorted(right) - 1,
    clamped to [-1, n-1]; a NaN query fails both range tests and every
    bisection compare, so the search ends at 0."""
    q = np.asarray(q, np.float64)
    i = np.clip(np.searchsorted(x, q, side="right") - 1, -1, x.size - 1)
    return np.where(np.isnan(q), 0, i)


def interp_cubic(x, v, coef, q):
    x = np.asarray(x, np.float64)
    q = np.asarray(q, np.float64)
    i = brackets(x, q)
    ii = np.clip(i, 0, x.size - 2)
    a, b, c, d = (coef[ii, k] for k in range(4))
    t = q - x[ii]
    val = a + t * (b + t * (c + t * d))
    val = np.where(i < 0, v[0], val)
    val = np.where(i >= x.size - 1, v[-1], val)
    return val, i.astype(np.int32)
