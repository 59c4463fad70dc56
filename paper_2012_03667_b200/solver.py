"""Gap-equation solver on the GPU (drop-in for reference solver.py:1-266).

Same entry points, signatures and return types as the reference:

  solve(params, variant, grid=None, probes_log10p=(-2.5, 0.0), a0=None, b0=None)
      -> PropagatorSolution                                   (solver.py:221-266)
  iterate_once(grid, a, b, params, variant) -> (A', B')      (solver.py:201-212)
  _eval_rows(grid, params, strategy, a, b, start, stop)       (solver.py:117-128)

The strategy seam is kept: AlgorithmVariant(interp, execution, threads) and
_make_sweeper (solver.py:53-74, 195-198).  The reference's execution modes
SEQUENTIAL and PARALLEL are kept with the reference's meaning of `threads`
(host workers, variant.threads else $SOLVER_THREADS else the CPU count,
solver.py:100-108): both run the sweep on one GPU in the reference's
operation order (Arithmetic.EXACT), and -- exactly as the reference promises
for its worker pools (test_solver.py:67-71) -- the worker count cannot
change a single bit, because no per-row work is left on the host.
ExecutionMode.GPU adds the device arithmetics (FAST, PAIRS, MOMENTS).

The GPU count is a separate, explicit knob: AlgorithmVariant.gpus, else
$DSE_GPUS, else 1 (resolve_gpus).  gpus > 1 runs the row-sharded solve of
paper_2012_03667_b200.distributed under torchrun (one process per GPU);
`threads` never selects GPUs.

`solve` hands the whole successive-approximation loop to the device
(dse_solve): relaxation, max-norm deltas, the strict stopping rule, history
and probes all happen in the persistent kernel, with no host round trip per
iteration.
"""
from __future__ import annotations

import ctypes
import enum
import os
import threading
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import ParameterError
from .grid import MomentumGrid, build_grid
from .interpolation import InterpStrategy
from .kernels import ModelParams

__all__ = [
    "ExecutionMode",
    "Arithmetic",
    "AlgorithmVariant",
    "VARIANTS",
    "IterationRecord",
    "PropagatorSolution",
    "resolve_threads",
    "resolve_gpus",
    "iterate_once",
    "solve",
    "solve_batch",
    "GpuSweeper",
    "DEFAULT_PROBES_LOG10P",
]

THREADS_ENV_VAR = "SOLVER_THREADS"
GPUS_ENV_VAR = "DSE_GPUS"
DEVICE_ENV_VAR = "DSE_DEVICE"

DEFAULT_PROBES_LOG10P = (-2.5, 0.0)


class ExecutionMode(enum.Enum):
    """SEQUENTIAL / PARALLEL: the reference's modes (solver.py:48-50), same
    values; both sweep on one GPU in the reference's operation order, and
    PARALLEL's worker count (threads) is a host-side knob that cannot change
    a bit.  GPU: the device arithmetics (AlgorithmVariant.arith)."""

    SEQUENTIAL = "seq"
    PARALLEL = "par"
    GPU = "gpu"


class Arithmetic(enum.Enum):
    """How the integrand is evaluated on the device.

    EXACT: the reference's operation order (kernels.py:188-218), one rounding
           per numpy op, IEEE divides; differs from the reference only by the
           device exp (<= 1 ulp).  The arithmetic of the reference's own
           execution modes (SEQUENTIAL, PARALLEL).
    FAST:  algebraically reduced, FMA-contracted, one reciprocal of k2 per
           point (csrc/dse_device.cuh point_fast).
    MOMENTS: the angular-moment factorisation: six
           theta-moments per (row, radial node) built once per sweeper from
           the grid and omega, then O(N*M) work per iteration
           (dse_moment_kernel).  A different summation order: parity with the
           reference to the fast tolerance, not bitwise.
    PAIRS: fast arithmetic, every integrand point evaluated every iteration,
           with the angular sum of each (row, node) pair accumulated as five
           moments and contracted once per pair (dse_pairs_kernel).  Parity
           gated like FAST.
    """

    EXACT = "exact"
    FAST = "fast"
    MOMENTS = "moments"
    PAIRS = "pairs"


def _arith_code(arith: Arithmetic) -> int:
    return {Arithmetic.EXACT: nat.ARITH_EXACT, Arithmetic.FAST: nat.ARITH_FAST,
            Arithmetic.MOMENTS: nat.ARITH_MOMENTS, Arithmetic.PAIRS: nat.ARITH_PAIRS}[arith]


_HOST_MODES = (ExecutionMode.SEQUENTIAL, ExecutionMode.PARALLEL)


@dataclass(frozen=True)
class AlgorithmVariant:
    """(interpolation strategy x execution) cell (solver.py:53-66).

    The first three fields are the reference's, positionally and by meaning:
    threads = host workers (resolve_threads).  arith defaults to EXACT for
    the reference's modes and FAST for ExecutionMode.GPU; gpus = GPUs per
    solve (resolve_gpus)."""

    interp: InterpStrategy
    execution: ExecutionMode = ExecutionMode.GPU
    threads: int | None = None
    arith: Arithmetic | None = None
    gpus: int | None = None

    def __post_init__(self):
        if self.arith is None:
            object.__setattr__(self, "arith", Arithmetic.EXACT if self.execution in _HOST_MODES
                               else Arithmetic.FAST)

    @property
    def name(self) -> str:
        base = f"{self.interp.value}-{self.execution.value}"
        default = Arithmetic.EXACT if self.execution in _HOST_MODES else Arithmetic.FAST
        return base if self.arith is default else f"{base}-{self.arith.value}"

    def with_threads(self, threads: int | None) -> "AlgorithmVariant":
        return AlgorithmVariant(self.interp, self.execution, threads, self.arith, self.gpus)

    def with_arith(self, arith: Arithmetic) -> "AlgorithmVariant":
        return AlgorithmVariant(self.interp, self.execution, self.threads, arith, self.gpus)

    def with_gpus(self, gpus: int | None) -> "AlgorithmVariant":
        return AlgorithmVariant(self.interp, self.execution, self.threads, self.arith, gpus)


_SEARCH = AlgorithmVariant(InterpStrategy.SEARCH_BASED)
_INDEXED = AlgorithmVariant(InterpStrategy.PRECOMPUTED_INDEX)

VARIANTS = {
    # GPU variants: fast arithmetic (parity-gated: <=1e-12 per sweep, exact
    # iteration counts and <=1e-9 on every golden solve)
    "search-gpu": _SEARCH,
    "indexed-gpu": _INDEXED,
    # the reference's operation order, one rounding per numpy op
    "search-gpu-exact": _SEARCH.with_arith(Arithmetic.EXACT),
    "indexed-gpu-exact": _INDEXED.with_arith(Arithmetic.EXACT),
    # the angular-moment factorisation: O(N M) per iteration after a one-off
    # O(N M K) moment build (for solves; parity gated like the fast variants)
    "search-gpu-moments": _SEARCH.with_arith(Arithmetic.MOMENTS),
    "indexed-gpu-moments": _INDEXED.with_arith(Arithmetic.MOMENTS),
    # fast arithmetic in the pair-moment form (same points per iteration)
    "search-gpu-pairs": _SEARCH.with_arith(Arithmetic.PAIRS),
    "indexed-gpu-pairs": _INDEXED.with_arith(Arithmetic.PAIRS),
    # the reference's names and cells (solver.py:69-74): same execution
    # modes, swept on one GPU in the reference's operation order
    "search-seq": AlgorithmVariant(InterpStrategy.SEARCH_BASED, ExecutionMode.SEQUENTIAL),
    "indexed-seq": AlgorithmVariant(InterpStrategy.PRECOMPUTED_INDEX, ExecutionMode.SEQUENTIAL),
    "search-par": AlgorithmVariant(InterpStrategy.SEARCH_BASED, ExecutionMode.PARALLEL),
    "indexed-par": AlgorithmVariant(InterpStrategy.PRECOMPUTED_INDEX, ExecutionMode.PARALLEL),
}


@dataclass(frozen=True)
class IterationRecord:
    iteration: int
    max_delta_a: float
    max_delta_b: float
    probe_a: tuple[float, ...]
    probe_b: tuple[float, ...]


def _records(hist: np.ndarray, P: int) -> list:
    """History rows (n, |dA|, |dB|, P probes of A, P of B) -> IterationRecords
    (one tolist() instead of a float() per element: ~3x faster for the long
    histories of batched scans)."""
    return [IterationRecord(int(r[0]), r[1], r[2], tuple(r[3:3 + P]), tuple(r[3 + P:3 + 2 * P]))
            for r in hist.tolist()]


@dataclass
class PropagatorSolution:
    A: np.ndarray
    B: np.ndarray
    iterations: int
    converged: bool
    history: list[IterationRecord]
    grid: MomentumGrid
    params: ModelParams
    probes_log10p: tuple[float, ...] = field(default=DEFAULT_PROBES_LOG10P)


_CPU_COUNT = os.cpu_count() or 1  # (os.cpu_count() costs ~3 us: read once, not per iterate_once call)


def resolve_threads(variant: AlgorithmVariant) -> int:
    """Host worker count, the reference's rule (solver.py:100-108):
    variant.threads, else $SOLVER_THREADS, else the CPU count.  It never
    changes a result (no per-row work runs on the host) and never selects
    GPUs (resolve_gpus does)."""
    if variant.threads is not None:
        n = variant.threads
    else:
        env = os.environ.get(THREADS_ENV_VAR)
        n = int(env) if env else _CPU_COUNT
    if n < 1:
        raise ParameterError(f"thread count must be >= 1, got {n}")
    return n


def resolve_gpus(variant: AlgorithmVariant) -> int:
    """GPUs per solve: variant.gpus, else $DSE_GPUS, else 1.  More than one
    needs torch.distributed initialised with that many ranks (one per GPU)."""
    if variant.gpus is not None:
        n = variant.gpus
    else:
        env = os.environ.get(GPUS_ENV_VAR)
        n = int(env) if env else 1
    if n < 1:
        raise ParameterError(f"GPU count must be >= 1, got {n}")
    return n


_TORCH_CUDA = []  # [torch.cuda] once it is known to be importable and available (checked once per process)


def _device() -> int:
    env = os.environ.get(DEVICE_ENV_VAR)
    if env:
        return int(env)
    if not _TORCH_CUDA:
        try:
            import torch  # optional: follow the caller's current device when torch is in use
            _TORCH_CUDA.append(torch.cuda if torch.cuda.is_available() else None)
        except Exception:  # noqa: BLE001
            _TORCH_CUDA.append(None)
    tc = _TORCH_CUDA[0]
    if tc is not None and tc.is_initialized():
        return tc.current_device()
    return int(os.environ.get("LOCAL_RANK", "0"))


def _c_params(params: ModelParams) -> nat.DseParams:
    return nat.DseParams(float(params.interaction_coeff), float(params.omega), float(params.m0),
                         float(params.z1), float(params.xi), float(params.relaxation),
                         int(params.max_iterations))


class GpuSweeper:
    """Device-resident sweeper (the _SequentialSweeper/_ParallelSweeper seam,
    solver.py:148-192): grid uploaded once, sweep(a, b) -> (a', b'), close().

    rows = (start, stride) restricts the sweeper to external rows
    start, start+stride, ... (multi-GPU row sharding)."""

    def __init__(self, grid, params: ModelParams, strategy: InterpStrategy,
                 arith: Arithmetic = Arithmetic.FAST, device: int | None = None,
                 rows: tuple[int, int] = (0, 1)):
        self.lib = nat.load()
        self.grid = grid
        self.params = params
        self.n = grid.n_ext
        self.device = _device() if device is None else device
        keep = [nat.as_f64(grid.p2_ext), nat.as_f64(grid.q2_int), nat.as_f64(grid.sqrt_q2_int),
                nat.as_f64(grid.radial_measure), nat.as_i64(grid.bracket_idx), nat.as_f64(grid.z_nodes),
                nat.as_f64(grid.z_weights)]
        g = nat.DseGrid(*(p for _, p in keep), grid.n_ext, grid.m_rad, grid.m_ang)
        prm = _c_params(params)
        handle = ctypes.c_void_p()
        err = nat.DseErr()
        strat = nat.INTERP_INDEXED if strategy is InterpStrategy.PRECOMPUTED_INDEX else nat.INTERP_SEARCH
        ar = _arith_code(arith)
        self.arith_code = ar
        rc = self.lib.dse_sweeper_create(ctypes.byref(g), ctypes.byref(prm), strat, ar, self.device,
                                         int(rows[0]), int(rows[1]), ctypes.byref(handle), ctypes.byref(err))
        nat.raise_for(rc, err)
        self.handle = handle
        self._lock = threading.Lock()

    def sweep(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        ao = np.empty(self.n)
        bo = np.empty(self.n)
        err = nat.DseErr()
        with self._lock:  # raw addresses: the per-call hot path (iterate_once)
            rc = nat.sweep_raw()(self.handle, a.ctypes.data, b.ctypes.data, ao.ctypes.data, bo.ctypes.data,
                                 ctypes.byref(err))
        nat.raise_for(rc, err)
        return ao, bo

    def sweep_device(self, dA: int, dB: int, dA_out: int, dB_out: int, stream: int = 0) -> None:
        """One sweep on device buffers (raw pointers, e.g. torch .data_ptr())."""
        err = nat.DseErr()
        rc = self.lib.dse_sweeper_sweep_device(self.handle, dA, dB, dA_out, dB_out, stream, ctypes.byref(err))
        nat.raise_for(rc, err)

    def check(self) -> None:
        err = nat.DseErr()
        nat.raise_for(self.lib.dse_sweeper_check(self.handle, ctypes.byref(err)), err)

    def solve(self, a0, b0, probes_p2=()):
        """Whole successive-approximation loop on the device (dse_solve)."""
        a = np.array(a0, dtype=np.float64, copy=True)
        b = np.array(b0, dtype=np.float64, copy=True)
        pr, ppr = nat.as_f64(np.asarray(probes_p2, dtype=np.float64).reshape(-1))
        cap = int(self.params.max_iterations)
        hist = np.empty((cap + 1, 3 + 2 * pr.size))
        it = ctypes.c_int64(0)
        conv = ctypes.c_int(0)
        err = nat.DseErr()
        with self._lock:
            rc = self.lib.dse_solve(self.handle, ppr, pr.size, a.ctypes.data_as(nat.f64p),
                                    b.ctypes.data_as(nat.f64p), ctypes.byref(it), ctypes.byref(conv),
                                    hist.ctypes.data_as(nat.f64p), ctypes.byref(err))
        nat.raise_for(rc, err)
        n = int(it.value)
        return a, b, n, bool(conv.value), hist[: n + 1]

    def solve_device(self, dA: int, dB: int, max_iterations: int, stream: int = 0, wait: bool = True):
        """Device-resident loop on raw device pointers (benchmarks)."""
        err = nat.DseErr()
        it = ctypes.c_int64(0)
        conv = ctypes.c_int(0)
        rc = self.lib.dse_solve_device(self.handle, dA, dB, int(max_iterations),
                                       ctypes.byref(it) if wait else None, ctypes.byref(conv) if wait else None,
                                       stream, ctypes.byref(err))
        nat.raise_for(rc, err)
        return (int(it.value), bool(conv.value)) if wait else None

    def load_device(self, dA: int, dB: int, stream: int = 0) -> None:
        """Copy device A/B into the resident state and rewind to iteration 0."""
        err = nat.DseErr()
        nat.raise_for(self.lib.dse_solve_load(self.handle, dA, dB, stream, ctypes.byref(err)), err)

    def resume(self, n_iterations: int, stream: int = 0) -> None:
        """Run the next n_iterations of the on-device loop (one launch, async)."""
        err = nat.DseErr()
        nat.raise_for(self.lib.dse_solve_resume(self.handle, int(n_iterations), stream, ctypes.byref(err)), err)

    def stats(self) -> dict:
        nom, ev, rows, smem = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        blocks = ctypes.c_int32()
        self.lib.dse_sweeper_stats(self.handle, ctypes.byref(nom), ctypes.byref(ev), ctypes.byref(rows),
                                   ctypes.byref(blocks), ctypes.byref(smem))
        return {"nominal_points": nom.value, "evaluated_points": ev.value, "rows": rows.value,
                "blocks": blocks.value, "smem_bytes": smem.value}

    def layout(self) -> dict:
        """The execution layout the library chose (dse_sweeper_layout)."""
        out = nat.DseLayout()
        self.lib.dse_sweeper_layout(self.handle, ctypes.byref(out))
        return {n: getattr(out, n) for n, _ in out._fields_}

    def close(self):
        # under the call lock: a thread that took this sweeper from the cache
        # just before it was evicted finishes its call on a live handle
        lock = getattr(self, "_lock", None)
        if lock is None:
            self._destroy()
            return
        with lock:
            self._destroy()

    def _destroy(self):
        if getattr(self, "handle", None):
            self.lib.dse_sweeper_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


# iterate_once builds a sweeper per call in the reference (solver.py:208); the
# device upload is cached per (grid, params, strategy) so repeated calls only
# move A and B.
_CACHE: "OrderedDict[tuple, GpuSweeper]" = OrderedDict()
_CACHE_MAX = 4
_CACHE_LOCK = threading.Lock()


def _params_key(p: ModelParams):
    return (p.D, p.omega, p.m0, p.z1, p.xi, p.relaxation, p.max_iterations)


def _make_sweeper(grid, params, variant: AlgorithmVariant) -> GpuSweeper:
    if not isinstance(variant.execution, ExecutionMode):
        raise ParameterError(f"unsupported execution mode {variant.execution}")
    resolve_threads(variant)  # validated like the reference (a bad count is a ParameterError)
    dev = _device()
    key = (id(grid), _params_key(params), variant.interp, variant.arith, dev)
    with _CACHE_LOCK:
        hit = _CACHE.get(key)
        if hit is not None and hit.grid is grid:
            _CACHE.move_to_end(key)
            return hit
        sw = GpuSweeper(grid, params, variant.interp, variant.arith, dev)
        _CACHE[key] = sw
        while len(_CACHE) > _CACHE_MAX:
            # no explicit close(): a thread that took the evicted sweeper from
            # the cache may still be about to call it; the handle is destroyed
            # by __del__ once the last reference is dropped (reference counting)
            _CACHE.popitem(last=False)
        return sw


def clear_sweeper_cache() -> None:
    with _CACHE_LOCK:
        while _CACHE:
            _CACHE.popitem()[1].close()


def _interp_at_internal(grid: MomentumGrid, values: np.ndarray, strategy: InterpStrategy) -> np.ndarray:
    """values interpolated at the M internal nodes with the strategy's
    bracket source (solver.py:111-114), on the GPU."""
    from .interpolation import interp_indexed_many, interp_search_many
    if strategy is InterpStrategy.PRECOMPUTED_INDEX:
        return interp_indexed_many(grid, values)
    return interp_search_many(grid.p2_ext, values, grid.q2_int)


def _eval_rows(grid: MomentumGrid, params: ModelParams, strategy: InterpStrategy,
               a: np.ndarray, b: np.ndarray, start: int, stop: int):
    """Rows [start, stop) of the sweep in the reference's arithmetic
    (solver.py:117-128); reads only (a, b).  Rows are Jacobi-independent and
    each is reduced by one CTA in a fixed order, so the rows of the cached
    device sweep ARE the rows of any row range (bitwise).  A numerical
    failure outside the range does not concern this range: the range is
    then evaluated row by row (dse_row_rhs), which raises only for its own
    rows, with the reference's (row, radial, angular) location."""
    from .errors import NumericalFailureError
    if not 0 <= start <= stop <= grid.n_ext:
        raise ParameterError(f"row range [{start}, {stop}) outside [0, {grid.n_ext})")
    variant = AlgorithmVariant(strategy, ExecutionMode.SEQUENTIAL)
    try:
        full_a, full_b = iterate_once(grid, a, b, params, variant)
        return full_a[start:stop].copy(), full_b[start:stop].copy()
    except NumericalFailureError as exc:
        if exc.row is not None and start <= exc.row < stop:
            raise
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    a_q = _interp_at_internal(grid, a, strategy)
    b_q = _interp_at_internal(grid, b, strategy)
    a_out = np.empty(stop - start)
    b_out = np.empty(stop - start)
    for i in range(start, stop):
        a_out[i - start], b_out[i - start] = _row_rhs_gpu(grid.p2_ext[i], a[i], b[i], a_q, b_q, grid, params, i)
    return a_out, b_out


def iterate_once(grid: MomentumGrid, a: np.ndarray, b: np.ndarray, params: ModelParams,
                 variant: AlgorithmVariant):
    """One Jacobi sweep (A', B') from (A, B) on the GPU (solver.py:201-212)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if a.shape != (grid.n_ext,) or b.shape != (grid.n_ext,):
        raise ParameterError("A and B must match the external grid size")
    if resolve_gpus(variant) > 1:
        from .distributed import iterate_once_sharded
        return iterate_once_sharded(grid, a, b, params, variant)
    return _make_sweeper(grid, params, variant).sweep(a, b)


def solve(params: ModelParams, variant: AlgorithmVariant, grid: MomentumGrid | None = None,
          probes_log10p: tuple[float, ...] = DEFAULT_PROBES_LOG10P, a0: np.ndarray | None = None,
          b0: np.ndarray | None = None) -> PropagatorSolution:
    """Iterate from A = B = 1 (or a0/b0) until both max-norm updates drop below
    xi, on the device; converged=False (not an error) at the iteration cap
    (solver.py:221-266, iteration.py:18-40)."""
    params.validate()
    if grid is None:
        grid = build_grid(params.N, params.m_rad, params.m_ang, params.p2_min, params.p2_max)
    probes_p2 = tuple(10.0 ** (2.0 * lp) for lp in probes_log10p)
    a = np.ones(grid.n_ext) if a0 is None else np.asarray(a0, dtype=float).copy()
    b = np.ones(grid.n_ext) if b0 is None else np.asarray(b0, dtype=float).copy()
    if a.shape != (grid.n_ext,) or b.shape != (grid.n_ext,):
        raise ParameterError("a0 and b0 must match the external grid size")
    if resolve_gpus(variant) > 1:
        from .distributed import solve_sharded
        a, b, n, conv, hist = solve_sharded(grid, params, variant, a, b, probes_p2)
    else:
        sweeper = _make_sweeper(grid, params, variant)
        a, b, n, conv, hist = sweeper.solve(a, b, probes_p2)
    P = len(probes_p2)
    history = _records(hist, P)
    return PropagatorSolution(A=a, B=b, iterations=n, converged=conv, history=history, grid=grid,
                              params=params, probes_log10p=tuple(probes_log10p))


def solve_batch(params_list, variant: AlgorithmVariant, grid: MomentumGrid | None = None,
                probes_log10p: tuple[float, ...] = DEFAULT_PROBES_LOG10P, a0s=None, b0s=None) -> list:
    """Independent solves on one grid in one go (parameter scans).

    Equivalent to [solve(p, variant, grid, probes_log10p, a0, b0) for ...]
    (bitwise: each solve runs the same kernel, concurrently on its own
    stream with a share of the GPU).  The grid-defining fields (N, m_rad,
    m_ang, p2_min, p2_max) must agree when grid is None.
    """
    params_list = list(params_list)
    if not params_list:
        return []
    for prm in params_list:
        prm.validate()
    resolve_threads(variant)
    if resolve_gpus(variant) != 1:
        raise ParameterError("solve_batch runs on one GPU; use torchrun + solve for multi-GPU solves")
    p0 = params_list[0]
    if grid is None:
        keys = {(p.N, p.m_rad, p.m_ang, p.p2_min, p.p2_max) for p in params_list}
        if len(keys) != 1:
            raise ParameterError("solve_batch needs one grid: N, m_rad, m_ang, p2_min, p2_max must agree")
        grid = build_grid(p0.N, p0.m_rad, p0.m_ang, p0.p2_min, p0.p2_max)
    S, n = len(params_list), grid.n_ext
    A = np.ones((S, n)) if a0s is None else np.array(a0s, dtype=np.float64).reshape(S, n).copy()
    B = np.ones((S, n)) if b0s is None else np.array(b0s, dtype=np.float64).reshape(S, n).copy()
    probes_p2 = np.array([10.0 ** (2.0 * lp) for lp in probes_log10p], dtype=np.float64)
    P = probes_p2.size
    W = 3 + 2 * P
    cap_max = max(int(p.max_iterations) for p in params_list)
    hist = np.empty((S, cap_max + 1, W))  # rows 0..iterations of each solve are written by the library
    keep = [nat.as_f64(grid.p2_ext), nat.as_f64(grid.q2_int), nat.as_f64(grid.sqrt_q2_int),
            nat.as_f64(grid.radial_measure), nat.as_i64(grid.bracket_idx), nat.as_f64(grid.z_nodes),
            nat.as_f64(grid.z_weights)]
    g = nat.DseGrid(*(p for _, p in keep), grid.n_ext, grid.m_rad, grid.m_ang)
    prms = (nat.DseParams * S)(*[_c_params(p) for p in params_list])
    its = np.zeros(S, np.int64)
    conv = (ctypes.c_int * S)()
    errs = (nat.DseErr * S)()
    strat = nat.INTERP_INDEXED if variant.interp is InterpStrategy.PRECOMPUTED_INDEX else nat.INTERP_SEARCH
    ar = _arith_code(variant.arith)
    rc = nat.load().dse_solve_batch(ctypes.byref(g), prms, S, strat, ar, _device(), probes_p2.ctypes.data_as(nat.f64p),
                                    P, A.ctypes.data_as(nat.f64p), B.ctypes.data_as(nat.f64p),
                                    its.ctypes.data_as(nat.i64p), conv, hist.ctypes.data_as(nat.f64p),
                                    (cap_max + 1) * W, errs)
    if rc:
        for k in range(S):
            if errs[k].code:
                nat.raise_for(errs[k].code, errs[k])
        nat.raise_for(rc, errs[0])
    out = []
    for k, prm in enumerate(params_list):
        nk = int(its[k])
        records = _records(hist[k, : nk + 1], P)
        out.append(PropagatorSolution(A=A[k].copy(), B=B[k].copy(), iterations=nk, converged=bool(conv[k]),
                                      history=records, grid=grid, params=prm, probes_log10p=tuple(probes_log10p)))
    return out


def _row_rhs_gpu(p2, a_p, b_p, a_q, b_q, grid, params, row, arith: Arithmetic = Arithmetic.EXACT):
    """row_rhs (kernels.py:178-226) through dse_row_rhs: one external row with
    the caller's a_q, b_q (exact arithmetic by default, like the reference)."""
    lib = nat.load()
    keep = [nat.as_f64(grid.p2_ext), nat.as_f64(grid.q2_int), nat.as_f64(grid.sqrt_q2_int),
            nat.as_f64(grid.radial_measure), nat.as_i64(grid.bracket_idx), nat.as_f64(grid.z_nodes),
            nat.as_f64(grid.z_weights)]
    g = nat.DseGrid(*(p for _, p in keep), grid.n_ext, grid.m_rad, grid.m_ang)
    aq, paq = nat.as_f64(a_q)
    bq, pbq = nat.as_f64(b_q)
    if aq.shape != (grid.m_rad,) or bq.shape != (grid.m_rad,):
        raise ParameterError("a_q and b_q must match the internal grid size")
    prm = _c_params(params)
    oa, ob = ctypes.c_double(), ctypes.c_double()
    err = nat.DseErr()
    rc = lib.dse_row_rhs(ctypes.byref(g), ctypes.byref(prm), _arith_code(arith), _device(), float(p2), float(a_p), float(b_p), paq, pbq,
                         -1 if row is None else int(row), ctypes.byref(oa), ctypes.byref(ob), ctypes.byref(err))
    if rc == nat.DSE_ENUMERIC and row is None:
        err.row = -1
    nat.raise_for(rc, err)
    return oa.value, ob.value
