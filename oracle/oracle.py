"""ctypes front end of the CPU oracle (dse_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline / --impl reference leg.  The product
package paper_2012_03667_b200 never imports this module.

Every function mirrors one reference entry point (file:line under
/root/reference/pkg/src/dsegap) and takes plain numpy arrays.  The grid is
any object with the MomentumGrid attributes (grid.py:29-64).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_dse.so")

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


class _Grid(ctypes.Structure):
    _fields_ = [("p2_ext", _f64p), ("q2_int", _f64p), ("sqrt_q2_int", _f64p),
                ("radial_measure", _f64p), ("bracket_idx", _i64p), ("z_nodes", _f64p),
                ("z_weights", _f64p), ("n_ext", ctypes.c_int64), ("m_rad", ctypes.c_int64),
                ("m_ang", ctypes.c_int64)]


class _Params(ctypes.Structure):
    _fields_ = [("coeff", ctypes.c_double), ("omega", ctypes.c_double), ("m0", ctypes.c_double),
                ("z1", ctypes.c_double), ("xi", ctypes.c_double), ("relaxation", ctypes.c_double),
                ("max_iterations", ctypes.c_int64)]


def build(force: bool = False) -> str:
    """Compile liboracle_dse.so with oracle/Makefile (gcc, -ffp-contract=off)."""
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "dse_oracle.c")):
        subprocess.run(["make", "-s", "-C", HERE, "-B" if force else "all"], check=True)
    return LIB_PATH


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_pairwise_sum.restype = ctypes.c_double
        L.oracle_pairwise_sum.argtypes = [_f64p, ctypes.c_int64]
        L.oracle_bracket_search.restype = ctypes.c_int64
        L.oracle_interp_search_many.restype = ctypes.c_int64
        L.oracle_interp_search_many.argtypes = [_f64p, _f64p, ctypes.c_int64, _f64p, ctypes.c_int64,
                                                _f64p, _i64p, ctypes.c_int]
        L.oracle_merge_bracket_indices.argtypes = [_f64p, ctypes.c_int64, _f64p, ctypes.c_int64, _i64p]
        L.oracle_sweep.restype = ctypes.c_int
        L.oracle_sweep.argtypes = [ctypes.POINTER(_Grid), ctypes.POINTER(_Params), ctypes.c_int,
                                   _f64p, _f64p, _f64p, _f64p, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_int, _i64p]
        L.oracle_solve.restype = ctypes.c_int
        L.oracle_solve.argtypes = [ctypes.POINTER(_Grid), ctypes.POINTER(_Params), ctypes.c_int,
                                   _f64p, ctypes.c_int64, _f64p, _f64p, _i64p,
                                   ctypes.POINTER(ctypes.c_int), _f64p, ctypes.c_int, _i64p]
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_set_per_row_interp.argtypes = [ctypes.c_int]
        _LIB = L
    return _LIB


def _p(a, dt=np.float64):
    a = np.ascontiguousarray(a, dtype=dt)
    return a, a.ctypes.data_as(_i64p if dt == np.int64 else _f64p)


class OracleError(RuntimeError):
    def __init__(self, msg, loc):
        super().__init__(msg)
        self.loc = loc


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def pairwise_sum(a) -> float:
    a, pa = _p(np.ravel(a))
    return float(lib().oracle_pairwise_sum(pa, a.size))


def merge_bracket_indices(p2_ext, q2_int):
    x, px = _p(p2_ext)
    q, pq = _p(q2_int)
    out = np.empty(q.size, np.int64)
    lib().oracle_merge_bracket_indices(px, x.size, pq, q.size, out.ctypes.data_as(_i64p))
    return out


def interp_search_many(x, v, queries, threads: int = 1, with_index: bool = False):
    """interpolation.py:100-113; returns values (and bracket indices, comparison count)."""
    x, px = _p(x)
    v, pv = _p(v)
    q, pq = _p(queries)
    out = np.empty(q.size)
    idx = np.empty(q.size, np.int64) if with_index else None
    cmp = lib().oracle_interp_search_many(px, pv, x.size, pq, q.size, out.ctypes.data_as(_f64p),
                                          idx.ctypes.data_as(_i64p) if with_index else None,
                                          int(threads))
    if with_index:
        return out, idx, int(cmp)
    return out


class _Keep:
    """Holds the contiguous arrays alive for the C struct."""

    def __init__(self, grid):
        self.arrs = []

        def f(a, dt=np.float64):
            a, p = _p(a, dt)
            self.arrs.append(a)
            return p
        self.g = _Grid(f(grid.p2_ext), f(grid.q2_int), f(grid.sqrt_q2_int), f(grid.radial_measure),
                       f(grid.bracket_idx, np.int64), f(grid.z_nodes), f(grid.z_weights),
                       grid.p2_ext.size, grid.q2_int.size, grid.z_nodes.size)


def _params(params):
    return _Params(float(params.interaction_coeff), float(params.omega), float(params.m0),
                   float(params.z1), float(params.xi), float(params.relaxation),
                   int(params.max_iterations))


def sweep(grid, a, b, params, strategy: int = 1, threads: int = 1, rows=None):
    """solver.py:117-128 _eval_rows (strategy 0 = search, 1 = indexed).

    rows = (start, stop) evaluates a sub-range (the reference's worker chunk).
    Raises OracleError(loc=(row, radial, angular)) like row_rhs.
    """
    keep = _Keep(grid)
    prm = _params(params)
    a, pa = _p(a)
    b, pb = _p(b)
    start, stop = (0, a.size) if rows is None else rows
    ao = np.empty(stop - start)
    bo = np.empty(stop - start)
    err = np.full(3, -1, np.int64)
    rc = lib().oracle_sweep(ctypes.byref(keep.g), ctypes.byref(prm), int(strategy), pa, pb,
                            ao.ctypes.data_as(_f64p), bo.ctypes.data_as(_f64p), start, stop,
                            int(threads), err.ctypes.data_as(_i64p))
    if rc:
        raise OracleError(f"non-finite integrand at row={err[0]}, radial={err[1]}, angular={err[2]}",
                          tuple(int(e) for e in err))
    return ao, bo


def set_per_row_interp(on: bool) -> None:
    """Interpolate A, B at the internal nodes once per ROW, as the reference's
    _eval_rows does (solver.py:123-125; same bits, the reference's cost)."""
    lib().oracle_set_per_row_interp(int(bool(on)))


def solve(grid, params, a0, b0, probes_p2=(), strategy: int = 1, threads: int = 1):
    """solver.py:221-266 + iteration.py:18-40.  Returns (A, B, iterations, converged, history)."""
    keep = _Keep(grid)
    prm = _params(params)
    a = np.array(a0, dtype=np.float64, copy=True)
    b = np.array(b0, dtype=np.float64, copy=True)
    pr, ppr = _p(np.asarray(probes_p2, dtype=np.float64).reshape(-1))
    cap = int(params.max_iterations)
    hist = np.full((cap + 1, 3 + 2 * pr.size), np.nan)
    it = np.zeros(1, np.int64)
    conv = ctypes.c_int(0)
    err = np.full(4, -1, np.int64)
    rc = lib().oracle_solve(ctypes.byref(keep.g), ctypes.byref(prm), int(strategy), ppr, pr.size,
                            a.ctypes.data_as(_f64p), b.ctypes.data_as(_f64p),
                            it.ctypes.data_as(_i64p), ctypes.byref(conv), hist.ctypes.data_as(_f64p),
                            int(threads), err.ctypes.data_as(_i64p))
    if rc:
        raise OracleError(f"non-finite integrand at iteration={err[0]} row={err[1]}",
                          tuple(int(e) for e in err))
    n = int(it[0])
    return a, b, n, bool(conv.value), hist[: n + 1]
