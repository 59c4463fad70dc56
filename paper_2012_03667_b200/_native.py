"""ctypes binding of libdse_b200.so (include/dse_b200.h).

The library is built in-tree by paper_2012_03667_b200._build (nvcc, sm_100a).
There is no CPU fallback: if the library or a B200 is missing, every call
raises ExecutionEnvironmentError.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import ExecutionEnvironmentError, NumericalFailureError, ParameterError

LIB_NAME = "libdse_b200.so"
LIB_PATH = os.environ.get("DSE_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

DSE_OK, DSE_EPARAM, DSE_ENUMERIC, DSE_EENV = 0, 1, 2, 3
INTERP_SEARCH, INTERP_INDEXED = 0, 1
BATCH_SEARCH, BATCH_DIRECT = 0, 1
ARITH_EXACT, ARITH_FAST, ARITH_MOMENTS, ARITH_PAIRS = 0, 1, 2, 3

f64p = ctypes.POINTER(ctypes.c_double)
i64p = ctypes.POINTER(ctypes.c_int64)
i32p = ctypes.POINTER(ctypes.c_int32)


class DseGrid(ctypes.Structure):
    _fields_ = [("p2_ext", f64p), ("q2_int", f64p), ("sqrt_q2_int", f64p), ("radial_measure", f64p),
                ("bracket_idx", i64p), ("z_nodes", f64p), ("z_weights", f64p),
                ("n_ext", ctypes.c_int64), ("m_rad", ctypes.c_int64), ("m_ang", ctypes.c_int64)]


class DseParams(ctypes.Structure):
    _fields_ = [("coeff", ctypes.c_double), ("omega", ctypes.c_double), ("m0", ctypes.c_double),
                ("z1", ctypes.c_double), ("xi", ctypes.c_double), ("relaxation", ctypes.c_double),
                ("max_iterations", ctypes.c_int64)]


class DseErr(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("iteration", ctypes.c_int64), ("row", ctypes.c_int64),
                ("radial", ctypes.c_int64), ("angular", ctypes.c_int64), ("msg", ctypes.c_char * 256)]


class DseLayout(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("threads", "lanes_per_leaf", "static_items", "cluster2",
                                              "split_rows", "node_chunk")]


class DseMuGrid(ctypes.Structure):
    _fields_ = [(n, f64p) for n in ("p_ext", "ps2_ext", "p4_ext", "q_int", "qs2_int", "q4_int", "meas_s", "meas_4",
                                    "z_nodes", "z_weights")] + \
               [("brk_s", i64p), ("brk_4", i64p)] + [(n, ctypes.c_int64) for n in ("n_s", "n_4", "m_s", "m_4", "m_ang")]


class DseMuParams(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("coeff", "omega", "m0", "z1", "mu", "xi", "relaxation")] + \
               [("max_iterations", ctypes.c_int64), ("vertex", ctypes.c_int64), ("mode", ctypes.c_int64)]


_LIB = None

# (name, restype, argtypes) -- one row per declaration in include/dse_b200.h
_PROTOS = [
    ("dse_device_info", ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(DseErr)]),
    ("dse_sweeper_create", ctypes.c_int, [ctypes.POINTER(DseGrid), ctypes.POINTER(DseParams), ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(DseErr)]),
    ("dse_sweeper_destroy", ctypes.c_int, [ctypes.c_void_p]),
    ("dse_sweeper_sweep", ctypes.c_int, [ctypes.c_void_p, f64p, f64p, f64p, f64p, ctypes.POINTER(DseErr)]),
    ("dse_sweeper_sweep_device", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                                ctypes.POINTER(DseErr)]),
    ("dse_sweeper_check", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(DseErr)]),
    ("dse_sharded_sweep_pack", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t,
                                              ctypes.POINTER(DseErr)]),
    ("dse_sharded_assemble", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t,
                                            ctypes.POINTER(DseErr)]),
    ("dse_sharded_sweep_push", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int64, ctypes.c_size_t,
                                              ctypes.POINTER(DseErr)]),
    ("dse_p2p_barrier", ctypes.c_int, [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(DseErr)]),
    ("dse_p2p_alloc", ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p,
                                     ctypes.POINTER(DseErr)]),
    ("dse_p2p_open", ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p),
                                    ctypes.POINTER(DseErr)]),
    ("dse_p2p_close", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    ("dse_sweeper_state", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
                                         ctypes.POINTER(ctypes.c_void_p)]),
    ("dse_solve", ctypes.c_int, [ctypes.c_void_p, f64p, ctypes.c_int64, f64p, f64p, i64p,
                                 ctypes.POINTER(ctypes.c_int), f64p, ctypes.POINTER(DseErr)]),
    ("dse_solve_device", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        i64p, ctypes.POINTER(ctypes.c_int), ctypes.c_size_t,
                                        ctypes.POINTER(DseErr)]),
    ("dse_interp_indexed_batch", ctypes.c_int, [f64p, f64p, ctypes.c_int64, f64p, i64p, ctypes.c_int64, f64p,
                                                ctypes.POINTER(DseErr)]),
    ("dse_interp_linear_batch", ctypes.c_int, [f64p, f64p, ctypes.c_int64, f64p, ctypes.c_int64, ctypes.c_int,
                                               f64p, i32p, i64p, ctypes.POINTER(DseErr)]),
    ("dse_interp_linear_batch_device", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                                      ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                                      ctypes.POINTER(DseErr)]),
    ("dse_interp_cubic_batch", ctypes.c_int, [f64p, f64p, f64p, ctypes.c_int64, f64p, ctypes.c_int64, ctypes.c_int,
                                              f64p, i32p, ctypes.POINTER(DseErr)]),
    ("dse_interp_cubic_batch_device", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                     ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                                     ctypes.POINTER(DseErr)]),
    ("dse_solve_load", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                      ctypes.POINTER(DseErr)]),
    ("dse_solve_resume", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t, ctypes.POINTER(DseErr)]),
    ("dse_sweeper_stats", ctypes.c_int, [ctypes.c_void_p, i64p, i64p, i64p, i32p, i64p]),
    ("dse_sweeper_layout", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    ("dse_fp64_peak", ctypes.c_int, [ctypes.c_int, f64p, ctypes.POINTER(DseErr)]),
    ("dse_solve_batch", ctypes.c_int, [ctypes.POINTER(DseGrid), ctypes.POINTER(DseParams), ctypes.c_int64,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int, f64p, ctypes.c_int64, f64p, f64p,
                                       i64p, ctypes.POINTER(ctypes.c_int), f64p, ctypes.c_int64,
                                       ctypes.POINTER(DseErr)]),
    ("dse_row_rhs", ctypes.c_int, [ctypes.POINTER(DseGrid), ctypes.POINTER(DseParams), ctypes.c_int, ctypes.c_int,
                                   ctypes.c_double, ctypes.c_double, ctypes.c_double, f64p, f64p, ctypes.c_int64,
                                   f64p, f64p, ctypes.POINTER(DseErr)]),
    ("dse_debug_pairwise_sum", ctypes.c_int, [ctypes.c_int, f64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_int64, f64p, f64p, ctypes.POINTER(DseErr)]),
    ("dse_sharded_set_stop", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    ("dse_sharded_assemble_step", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                                 ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p,
                                                 ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                 ctypes.POINTER(DseErr)]),
    ("dse_debug_exp_neg_k2", ctypes.c_int, [ctypes.c_int, ctypes.c_double, f64p, ctypes.c_int64, f64p, f64p,
                                            ctypes.POINTER(DseErr)]),
    ("dse_debug_exp_exact", ctypes.c_int, [ctypes.c_int, f64p, ctypes.c_int64, f64p, f64p, i32p,
                                           ctypes.POINTER(DseErr)]),
    ("dse_debug_qdiv_ext", ctypes.c_int, [ctypes.c_int, f64p, f64p, ctypes.c_int64, f64p, f64p, i32p,
                                          ctypes.POINTER(DseErr)]),
    ("dse_plan_info", ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, i32p, i32p, ctypes.c_int64, i32p, i32p, i32p,
                                     ctypes.c_int64, i64p, i64p]),
    ("dse_debug_check_flags", ctypes.c_int, [ctypes.POINTER(ctypes.c_uint32)]),
    ("dse_mu_sweeper_create", ctypes.c_int, [ctypes.POINTER(DseMuGrid), ctypes.POINTER(DseMuParams), ctypes.c_int,
                                             ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p),
                                             ctypes.POINTER(DseErr)]),
    ("dse_mu_sweeper_destroy", ctypes.c_int, [ctypes.c_void_p]),
    ("dse_mu_solve", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(DseMuParams), f64p, f64p, f64p, i64p,
                                    ctypes.POINTER(ctypes.c_int), f64p, ctypes.POINTER(DseErr)]),
    ("dse_mu_sweep", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(DseMuParams), f64p, f64p, f64p, f64p, f64p, f64p,
                                    ctypes.POINTER(DseErr)]),
    ("dse_mu_solve_load", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_size_t, ctypes.POINTER(DseErr)]),
    ("dse_mu_solve_resume", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t, ctypes.POINTER(DseErr)]),
    ("dse_mu_interp", ctypes.c_int, [ctypes.c_void_p, f64p, f64p, ctypes.POINTER(DseErr)]),
    ("dse_mu_sharded_sweep_pack", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(DseMuParams), ctypes.c_void_p,
                                                 ctypes.c_int64, ctypes.c_size_t, ctypes.POINTER(DseErr)]),
    ("dse_mu_sharded_assemble", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                               ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t,
                                               ctypes.POINTER(DseErr)]),
    ("dse_mu_sharded_failure", ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(DseErr)]),
    ("dse_mu_sweeper_state", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    ("dse_mu_batch_sweep", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(DseMuParams), ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, i64p,
                                          ctypes.POINTER(DseErr)]),
    ("dse_mu_batch_solve", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(DseMuParams), ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, i64p,
                                          i32p, i64p, i64p, ctypes.c_size_t, ctypes.POINTER(DseErr)]),
    ("dse_mu_sweeper_stats", ctypes.c_int, [ctypes.c_void_p, i64p, i64p, i32p, i64p]),
    ("dse_mu_aa_residual", ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, i32p, ctypes.c_int32,
                                          ctypes.c_void_p, f64p, ctypes.c_size_t, ctypes.POINTER(DseErr)]),
    ("dse_mu_aa_update", ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, i32p, ctypes.c_int32, f64p,
                                        ctypes.c_double, ctypes.c_size_t, ctypes.POINTER(DseErr)]),
    ("dse_launch_count", ctypes.c_int64, []),
]

EXPORTED_SYMBOLS = tuple(p[0] for p in _PROTOS)


def load(path: str = LIB_PATH):
    """Load the CUDA library (once).  Raises ExecutionEnvironmentError if absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise ExecutionEnvironmentError(
            f"{LIB_NAME} is not built ({path}); run `python -c \"import __graft_entry__ as g; g.build()\"`")
    try:
        lib = ctypes.CDLL(path)
    except OSError as exc:
        raise ExecutionEnvironmentError(f"cannot load {path}: {exc}") from exc
    for name, res, args in _PROTOS:
        if not hasattr(lib, name) and os.environ.get("DSE_LIB"):
            continue  # an older library under A/B test
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def raise_for(rc: int, err: DseErr) -> None:
    """Map a C-ABI return code onto the reference's exception classes."""
    if rc == DSE_OK:
        return
    msg = err.msg.decode(errors="replace")
    if rc == DSE_EPARAM:
        raise ParameterError(msg)
    if rc == DSE_ENUMERIC:
        raise NumericalFailureError(msg, row=int(err.row), radial=int(err.radial), angular=int(err.angular),
                                    iteration=int(err.iteration) or None)
    raise ExecutionEnvironmentError(msg or f"CUDA library error {rc}")


def device_info(device: int = 0):
    lib = load()
    name = ctypes.create_string_buffer(128)
    sms = ctypes.c_int(0)
    err = DseErr()
    raise_for(lib.dse_device_info(device, name, 128, ctypes.byref(sms), ctypes.byref(err)), err)
    return name.value.decode(), sms.value


_SWEEP_RAW = []


def sweep_raw():
    """dse_sweeper_sweep bound with raw integer addresses (no pointer objects
    per call): the prototype of include/dse_b200.h with void* arguments."""
    if not _SWEEP_RAW:
        vp = ctypes.c_void_p
        fn = ctypes.CFUNCTYPE(ctypes.c_int, vp, vp, vp, vp, vp, vp)(("dse_sweeper_sweep", load()))
        _SWEEP_RAW.append(fn)
    return _SWEEP_RAW[0]


def as_f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(f64p)


def as_i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(i64p)


def launch_count() -> int:
    return int(load().dse_launch_count())


def debug_pairwise_sum(vals, chunk_leaves: int = 0, device: int = 0):
    """Test hook (dse_debug_pairwise_sum): the production kernel's reduction of
    vals[rows, m, k] per row; returns (sum(v), sum(-2 v)) per row."""
    import ctypes as _ct
    v = np.ascontiguousarray(vals, dtype=np.float64)
    rows, m, k = v.shape
    oa, ob = np.empty(rows), np.empty(rows)
    err = DseErr()
    rc = load().dse_debug_pairwise_sum(device, v.ctypes.data_as(f64p), rows, m, k, int(chunk_leaves),
                                       oa.ctypes.data_as(f64p), ob.ctypes.data_as(f64p), _ct.byref(err))
    raise_for(rc, err)
    return oa, ob


def debug_exp_neg_k2(k2, omega: float, device: int = 0):
    """Test hook (dse_debug_exp_neg_k2): (table exp, CUDA exp) of -k2/omega^2."""
    import ctypes as _ct
    k = np.ascontiguousarray(k2, dtype=np.float64)
    t, e = np.empty(k.size), np.empty(k.size)
    err = DseErr()
    rc = load().dse_debug_exp_neg_k2(device, float(omega), k.ctypes.data_as(f64p), k.size, t.ctypes.data_as(f64p),
                                     e.ctypes.data_as(f64p), _ct.byref(err))
    raise_for(rc, err)
    return t, e


def debug_exp_exact(x, device: int = 0):
    """Test hook (dse_debug_exp_exact): (exp_rep, CUDA exp, exp_rep valid) of x."""
    import ctypes as _ct
    v = np.ascontiguousarray(x, dtype=np.float64)
    r, e, k = np.empty(v.size), np.empty(v.size), np.empty(v.size, dtype=np.int32)
    err = DseErr()
    rc = load().dse_debug_exp_exact(device, v.ctypes.data_as(f64p), v.size, r.ctypes.data_as(f64p),
                                    e.ctypes.data_as(f64p), k.ctypes.data_as(i32p), _ct.byref(err))
    raise_for(rc, err)
    return r, e, k.astype(bool)


def debug_qdiv_ext(a, b, device: int = 0):
    """Test hook (dse_debug_qdiv_ext): (qdiv_ext, __ddiv_rn, ext valid) of a / b."""
    import ctypes as _ct
    va = np.ascontiguousarray(a, dtype=np.float64)
    vb = np.ascontiguousarray(b, dtype=np.float64)
    e, r, k = np.empty(va.size), np.empty(va.size), np.empty(va.size, dtype=np.int32)
    err = DseErr()
    rc = load().dse_debug_qdiv_ext(device, va.ctypes.data_as(f64p), vb.ctypes.data_as(f64p), va.size,
                                   e.ctypes.data_as(f64p), r.ctypes.data_as(f64p), k.ctypes.data_as(i32p),
                                   _ct.byref(err))
    raise_for(rc, err)
    return e, r, k.astype(bool)


def plan_info(n: int, chunk_leaves: int = 1 << 30):
    """The kernels' reduction plan for an n-element block (host only)."""
    import ctypes as _ct
    cap = n // 64 + 8
    ls, ll = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
    lo, hi, tp = np.zeros(cap, np.int32), np.zeros(cap, np.int32), np.zeros(2 * cap, np.int32)
    nl, nc = _ct.c_int64(), _ct.c_int64()
    rc = load().dse_plan_info(n, chunk_leaves, ls.ctypes.data_as(i32p), ll.ctypes.data_as(i32p), cap,
                              lo.ctypes.data_as(i32p), hi.ctypes.data_as(i32p), tp.ctypes.data_as(i32p), cap,
                              _ct.byref(nl), _ct.byref(nc))
    if rc:
        raise ValueError(f"dse_plan_info failed ({rc})")
    return (ls[:nl.value], ll[:nl.value], lo[:nc.value], hi[:nc.value], tp[:2 * max(nc.value - 1, 0)].reshape(-1, 2))
