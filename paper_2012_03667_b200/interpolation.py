"""Piecewise-linear interpolation in p2 (reference interpolation.py:1-154), on the GPU.

Both strategies apply the identical formula v[i] + (q - x[i]) * (v[i+1] -
v[i]) / (x[i+1] - x[i]) with IEEE fp64 and no FMA contraction, so results
are bitwise equal to the reference's (tests/test_interp_gpu.py).

  search   : per-query binary search (_bracket_search, interpolation.py:47-68)
  indexed  : precomputed bracket (grid.bracket_idx, interpolation.py:135-154)
  direct   : batch mode of interp_search_many(..., mode="direct"): the bracket
             is computed arithmetically from a log2/linear bucket table and
             fixed with at most a few exact compares (the paper's "modified
             interpolation"); bitwise equal to search.
"""
from __future__ import annotations

import ctypes
import enum

import numpy as np

from . import _native as nat
from .errors import ParameterError

__all__ = ["InterpStrategy", "ComparisonCounter", "interp_search", "interp_search_many",
           "interp_indexed", "interp_indexed_many", "interp_linear_batch", "natural_cubic_coefficients",
           "interp_cubic_batch"]


class InterpStrategy(enum.Enum):
    SEARCH_BASED = "search"
    PRECOMPUTED_INDEX = "indexed"


class ComparisonCounter:
    """Counts comparisons made against grid entries during bracket location
    (2 per query + 1 per bisection step, interpolation.py:38-63)."""

    __slots__ = ("count",)

    def __init__(self):
        self.count = 0


def _validate_grid(x, v):
    if len(x) < 2:
        raise ParameterError("interpolation grid needs at least 2 knots")
    if len(x) != len(v):
        raise ParameterError(f"grid/value length mismatch: {len(x)} vs {len(v)}")
    if not np.all(np.diff(x) > 0):
        raise ParameterError("interpolation grid must be strictly increasing")


def interp_linear_batch(x, v, queries, mode: str = "search", with_index: bool = False,
                        counter: ComparisonCounter | None = None):
    """Batched interpolation through dse_interp_linear_batch (host arrays).

    mode "search" = interp_search_many semantics with a per-query binary
    search; "direct" = arithmetic bracket + compare-fix (no search).  Returns
    values, or (values, int32 bracket indices) with with_index=True.
    """
    _validate_grid(x, v)
    xs, px = nat.as_f64(x)
    vs, pv = nat.as_f64(v)
    qs, pq = nat.as_f64(np.ravel(np.asarray(queries, dtype=np.float64)))
    out = np.empty(qs.size)
    idx = np.empty(qs.size, np.int32) if with_index else None
    cmp = ctypes.c_int64(0)
    err = nat.DseErr()
    m = {"search": nat.BATCH_SEARCH, "direct": nat.BATCH_DIRECT}.get(mode)
    if m is None:
        raise ParameterError(f"unknown interpolation mode {mode!r}")
    rc = nat.load().dse_interp_linear_batch(
        px, pv, xs.size, pq, qs.size, m, out.ctypes.data_as(nat.f64p),
        idx.ctypes.data_as(nat.i32p) if with_index else None,
        ctypes.byref(cmp) if counter is not None else None, ctypes.byref(err))
    nat.raise_for(rc, err)
    if counter is not None:
        counter.count += int(cmp.value)
    return (out, idx) if with_index else out


def natural_cubic_coefficients(x, v) -> np.ndarray:
    """Natural cubic spline through (x_i, v_i) (second derivative 0 at both
    ends), as rows (a, b, c, d) of a + t (b + t (c + t d)), t = x - x_i, per
    interval [x_i, x_i+1].  Host-side input producer of interp_cubic_batch
    (like the grid builder): the tridiagonal system for the knot second
    derivatives M is solved once per table by the Thomas algorithm.  The
    reference has no cubic routine; tests pin this against
    scipy.interpolate.CubicSpline(bc_type="natural")."""
    x = np.asarray(x, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    _validate_grid(x, v)
    n = x.size
    h = np.diff(x)
    M = np.zeros(n)
    if n > 2:
        sl = np.diff(v) / h
        rhs = 6.0 * np.diff(sl)                  # rows 1..n-2
        diag = 2.0 * (h[:-1] + h[1:])
        sub = h[1:-1].copy()                     # h_i couples M_i and M_{i+1}
        cp = np.empty(n - 2)
        dp = np.empty(n - 2)
        cp[0] = sub[0] / diag[0] if n > 3 else 0.0
        dp[0] = rhs[0] / diag[0]
        for i in range(1, n - 2):
            den = diag[i] - h[i] * cp[i - 1]
            cp[i] = sub[i] / den if i < n - 3 else 0.0
            dp[i] = (rhs[i] - h[i] * dp[i - 1]) / den
        m_in = np.empty(n - 2)
        m_in[-1] = dp[-1]
        for i in range(n - 4, -1, -1):
            m_in[i] = dp[i] - cp[i] * m_in[i + 1]
        M[1:-1] = m_in
    coef = np.empty((n - 1, 4))
    coef[:, 0] = v[:-1]
    coef[:, 1] = np.diff(v) / h - h * (2.0 * M[:-1] + M[1:]) / 6.0
    coef[:, 2] = 0.5 * M[:-1]
    coef[:, 3] = np.diff(M) / (6.0 * h)
    return coef


def interp_cubic_batch(x, v, queries, mode: str = "direct", with_index: bool = False, coef=None):
    """Batched natural-cubic-spline interpolation through dse_interp_cubic_batch
    (BASELINE config 1's cubic half): the same brackets ("search" or "direct")
    and clamping as interp_linear_batch, value from the interval's cubic."""
    _validate_grid(x, v)
    xs, px = nat.as_f64(x)
    vs, pv = nat.as_f64(v)
    cf, pc = nat.as_f64(natural_cubic_coefficients(xs, vs) if coef is None else coef)
    if cf.shape != (xs.size - 1, 4):
        raise ParameterError(f"coefficient table must be ({xs.size - 1}, 4), got {cf.shape}")
    qs, pq = nat.as_f64(np.ravel(np.asarray(queries, dtype=np.float64)))
    out = np.empty(qs.size)
    idx = np.empty(qs.size, np.int32) if with_index else None
    err = nat.DseErr()
    m = {"search": nat.BATCH_SEARCH, "direct": nat.BATCH_DIRECT}.get(mode)
    if m is None:
        raise ParameterError(f"unknown interpolation mode {mode!r}")
    rc = nat.load().dse_interp_cubic_batch(px, pv, pc, xs.size, pq, qs.size, m, out.ctypes.data_as(nat.f64p),
                                           idx.ctypes.data_as(nat.i32p) if with_index else None, ctypes.byref(err))
    nat.raise_for(rc, err)
    return (out, idx) if with_index else out


def interp_search(x, v, q, counter: ComparisonCounter | None = None) -> float:
    """Scalar search-based interpolation (interpolation.py:84-97)."""
    return float(interp_linear_batch(x, v, [q], "search", counter=counter)[0])


def interp_search_many(x, v, queries, counter: ComparisonCounter | None = None) -> np.ndarray:
    """Search-based interpolation of every query (interpolation.py:100-113)."""
    return interp_linear_batch(x, v, queries, "search", counter=counter)


def _indexed(grid, values, js):
    n = grid.n_ext
    if len(values) != n:
        raise ParameterError(f"values length {len(values)} != external grid size {n}")
    xs, px = nat.as_f64(grid.p2_ext)
    vs, pv = nat.as_f64(values)
    qs, pq = nat.as_f64(np.asarray(grid.q2_int)[js])
    ix, pi = nat.as_i64(np.asarray(grid.bracket_idx)[js])
    out = np.empty(qs.size)
    err = nat.DseErr()
    rc = nat.load().dse_interp_indexed_batch(px, pv, n, pq, pi, qs.size, out.ctypes.data_as(nat.f64p),
                                             ctypes.byref(err))
    nat.raise_for(rc, err)
    return out


def interp_indexed(grid, values, j: int) -> float:
    """Interpolation at internal node j with the precomputed bracket (interpolation.py:116-132)."""
    if not 0 <= j < grid.m_rad:
        raise ParameterError(f"internal node index {j} out of range [0, {grid.m_rad})")
    return float(_indexed(grid, values, np.array([j]))[0])


def interp_indexed_many(grid, values) -> np.ndarray:
    """Precomputed-index interpolation at all internal nodes (interpolation.py:135-154)."""
    return _indexed(grid, values, np.arange(grid.m_rad))
