"""Multi-GPU solve: external rows sharded across ranks, iterate all-gathered.

SURVEY.md §8e: rows are Jacobi-independent (solver.py:1-13, 159-166), so rank
r of W owns rows r, r+W, ... (cyclic: balances the per-row cost left after
the exact-zero skip).  Each iteration:

  1. every rank sweeps its rows on its GPU (libdse_b200, the same kernel and
     the same per-row reduction order as the single-GPU path);
  2. the compact per-rank results are all-gathered (NCCL over NVLink; one
     2 x ceil(N/W) fp64 message per rank, 16 KiB total at N=1024);
  3. every rank applies the relaxation blend (solver.py:249-251), the
     max-norm deltas (iteration.py:34), the stop rule and the history probes
     to the full arrays -- identical inputs, identical results on all ranks,
     so no all-reduce and no broadcast is needed.

The result is bitwise identical to the single-GPU solve for any W (a row's
reduction never crosses a CTA, let alone a GPU).

The loop body is written once against small callables (sweep_rows, gather,
probe) so the partition/reassembly/convergence logic is exercised on CPU with
gloo in tests/test_distributed.py.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import Callable

import numpy as np

from .errors import ExecutionEnvironmentError, ParameterError

__all__ = ["owned_rows", "ShardedLoop", "solve_sharded", "iterate_once_sharded", "bench_main"]


def owned_rows(n: int, rank: int, world: int) -> np.ndarray:
    return np.arange(rank, n, world)


@dataclass
class ShardedLoop:
    """successive_approximation (iteration.py:18-40) over row-sharded sweeps.

    sweep_rows(a, b) -> (a_rows, b_rows): this rank's raw sweep values for
        owned_rows(n, rank, world), in that order.
    gather(x) -> [W, ceil(n/W)] stacked per-rank padded rows (all-gather).
    probe(a, b) -> (pa[P], pb[P]): search interpolation at the probes.
    xp: array namespace (numpy, or torch for device arrays).
    """

    n: int
    rank: int
    world: int
    sweep_rows: Callable
    gather: Callable
    probe: Callable
    xp: object = np

    def _assemble(self, a_rows, b_rows):
        xp = self.xp
        per = math.ceil(self.n / self.world)
        buf = xp.zeros((2, per), dtype=a_rows.dtype) if xp is np else \
            xp.zeros((2, per), dtype=a_rows.dtype, device=a_rows.device)
        k = a_rows.shape[0]
        buf[0, :k] = a_rows
        buf[1, :k] = b_rows
        g = self.gather(buf)  # [W, 2, per]
        a = xp.empty(self.n, dtype=a_rows.dtype) if xp is np else xp.empty(self.n, dtype=a_rows.dtype,
                                                                             device=a_rows.device)
        b = xp.empty_like(a)
        for r in range(self.world):
            cnt = len(range(r, self.n, self.world))
            a[r::self.world] = g[r, 0, :cnt]
            b[r::self.world] = g[r, 1, :cnt]
        return a, b

    def sweep(self, a, b):
        return self._assemble(*self.sweep_rows(a, b))

    def run(self, a, b, xi: float, cap: int, relaxation: float, check_every: int = 16):
        """successive_approximation with a lazy stop test: the deltas, probes
        and states of the last `check_every` iterations stay on the device and
        the host looks at them once per window (one sync per window instead of
        one per iteration).  The result is that of the eager loop: the solve
        stops at the FIRST iteration whose deltas are both < xi, and that
        iteration's state is returned."""
        xp = self.xp
        hist = [[0.0, math.nan, math.nan, *self._probe_row(a, b)]]
        window = []  # (iteration, a, b, da, db, probes) kept as device values
        for it in range(1, cap + 1):
            an, bn = self.sweep(a, b)
            if relaxation != 1.0:
                an = relaxation * an + (1.0 - relaxation) * a
                bn = relaxation * bn + (1.0 - relaxation) * b
            da = xp.max(xp.abs(an - a))
            db = xp.max(xp.abs(bn - b))
            a, b = an, bn
            window.append((it, a, b, da, db, self.probe(a, b)))
            if len(window) == check_every or it == cap:
                for (n, wa, wb, wda, wdb, (pa, pb)) in window:   # host reads the window once
                    fda, fdb = float(wda), float(wdb)
                    hist.append([float(n), fda, fdb, *[float(x) for x in pa], *[float(x) for x in pb]])
                    if fda < xi and fdb < xi:
                        return wa, wb, n, True, np.array(hist)
                window = []
        return a, b, cap, False, np.array(hist)

    def _probe_row(self, a, b):
        pa, pb = self.probe(a, b)
        return [float(x) for x in pa] + [float(x) for x in pb]


@dataclass
class WindowedStopLoop:
    """successive_approximation (iteration.py:18-40) driven from the host in
    windows, with the stop test on the device -- the loop of the public
    multi-GPU solve (ShardedSolver).

    step(n): enqueue iteration n (sweep of the owned rows, exchange,
        assemble + relaxation, history row n, device stop flag: 1 = both
        deltas < xi, 2 = non-finite sweep; once set, later steps are no-ops
        on the device, so the state stays the stopping iteration's).
    read(lo, hi) -> (rows [hi-lo+1, W], flag): history rows lo..hi and the
        flag, one device->host copy (the only sync of a window).
    locate() -> (row, radial, angular): collective; the lowest failing row
        over all ranks (every rank gets the same answer).

    No collective is needed for the stop decision: every rank holds the
    same full iterate, so the deltas and the flag agree bitwise."""

    step: Callable
    read: Callable
    locate: Callable

    def run(self, xi: float, cap: int, window: int = 16):
        from .errors import NumericalFailureError
        done = 0
        while done < cap:
            w = min(window, cap - done)
            for n in range(done + 1, done + w + 1):
                self.step(n)
            rows, flag = self.read(done + 1, done + w)
            if flag == 2:
                bad = next(int(r[0]) for r in rows if not (np.isfinite(r[1]) and np.isfinite(r[2])))
                row, radial, angular = self.locate()
                raise NumericalFailureError(f"non-finite integrand in sweep at row={row}, radial={radial}, "
                                            f"angular={angular}", row=row, radial=radial, angular=angular,
                                            iteration=bad)
            for r in rows:
                if r[1] < xi and r[2] < xi:  # strict, both (iteration.py:38)
                    return int(r[0]), True
            done += w
        return cap, False


def _torch_env():
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        raise ParameterError("multi-GPU solve needs torch.distributed initialised (one process per GPU)")
    return torch, dist


class FusedShardedStep:
    """One multi-GPU iteration as three device steps around the NCCL
    all-gather (dse_sharded_sweep_pack / dse_sharded_assemble[_step]): the
    sweeper's resident state is the full iterate, the owned rows are packed
    straight into the send buffer, and one kernel reassembles the gathered
    rows with the relaxation blend and the max-norm deltas (and, inside a
    solve, the history row and the device stop flag).  Bitwise the
    single-GPU sweep + blend + deltas at any world size (a row is reduced by
    one CTA/warp set; the blend and deltas are per-element operations)."""

    def __init__(self, sw, n: int, world: int, dev, gather_into, relaxation: float = 1.0):
        import ctypes

        import torch

        from . import _native as nat
        self.sw, self.n, self.world = sw, n, world
        self.per = math.ceil(n / world)
        self.send = torch.zeros((2, self.per), dtype=torch.float64, device=dev)
        self.recv = torch.zeros((world, 2, self.per), dtype=torch.float64, device=dev)
        self.delta = torch.zeros(2, dtype=torch.float64, device=dev)
        self.gather_into = gather_into
        self.relax = relaxation
        self._nat, self._lib = nat, nat.load()
        pa, pb = ctypes.c_void_p(), ctypes.c_void_p()
        nat.raise_for(self._lib.dse_sweeper_state(sw.handle, ctypes.byref(pa), ctypes.byref(pb)), nat.DseErr())
        self.state_ptrs = (pa.value, pb.value)
        self.kind = "nccl"

    def load(self, a, b, stream: int) -> None:
        self.sw.load_device(a.data_ptr(), b.data_ptr(), stream)

    def _assemble(self, recv_ptr: int, stream: int, relax, solve) -> None:
        import ctypes
        err = self._nat.DseErr()
        relax = self.relax if relax is None else relax
        if solve is None:
            rc = self._lib.dse_sharded_assemble(self.sw.handle, recv_ptr, self.world, self.per, relax,
                                                self.delta.data_ptr(), stream, ctypes.byref(err))
        else:  # (xi, iteration, probes tensor, history row address)
            xi, it, probes, row = solve
            rc = self._lib.dse_sharded_assemble_step(self.sw.handle, recv_ptr, self.world, self.per, relax, xi, it,
                                                     probes.data_ptr() if probes.numel() else None, probes.numel(),
                                                     row, self.delta.data_ptr(), stream, ctypes.byref(err))
        self._nat.raise_for(rc, err)

    def step(self, stream: int, relax=None, solve=None):
        import ctypes
        err = self._nat.DseErr()
        self._nat.raise_for(self._lib.dse_sharded_sweep_pack(self.sw.handle, self.send.data_ptr(), self.per, stream,
                                                             ctypes.byref(err)), err)
        self.gather_into(self.recv, self.send)
        self._assemble(self.recv.data_ptr(), stream, relax, solve)
        return self.delta

    def close(self) -> None:
        pass


def device_view(ptr: int, n: int, device):
    """A torch float64 view of n doubles at a raw device address (the
    sweeper's resident state), via __cuda_array_interface__."""
    import torch

    class _Raw:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (int(ptr), False), "version": 3,
                                    "strides": None}
    return torch.as_tensor(_Raw(), device=device)


class P2PShardedStep(FusedShardedStep):
    """The multi-GPU iteration with the all-gather FUSED into the sweep over
    NVLink peer memory (no NCCL on the data path): every rank maps every
    other rank's receive buffer and barrier flag (CUDA IPC handles exchanged
    once through `exchange`, e.g. dist.all_gather_object); the pairs kernel
    stores each finished row into all receive buffers the moment the row is
    done (dse_sharded_sweep_push), a one-thread kernel barriers across the
    GPUs over the flags (bounded spin: a missing peer raises instead of
    hanging), and the assemble kernel rebuilds the full iterate.  3 launches
    per step.

    Construction is collective and failure-safe: every rank makes exactly
    two `exchange` calls whatever fails locally (the IPC handles, then the
    verdict of mapping every peer), so a failure anywhere raises
    ExecutionEnvironmentError on EVERY rank and every rank frees what it
    allocated or mapped."""

    def __init__(self, sw, n: int, world: int, rank: int, device: int, dev, exchange, relaxation: float = 1.0):
        import ctypes

        import torch
        if world > 8:
            raise ParameterError("the peer-memory all-gather maps at most 8 GPUs (one node)")
        super().__init__(sw, n, world, dev, None, relaxation)
        nat, lib = self._nat, self._lib
        self.rank = rank
        self.kind = "p2p"
        # receive buffers double-buffered by step parity: a fast rank's push of
        # step e+1 must not overwrite what a slow rank still assembles of step e
        self._slot = world * 2 * self.per
        self._own, self._mapped = [], []
        err = nat.DseErr()
        local_error, handles = None, []
        try:
            for nbytes in (2 * self._slot * 8, 64):
                ptr = ctypes.c_void_p()
                h = ctypes.create_string_buffer(64)
                nat.raise_for(lib.dse_p2p_alloc(device, nbytes, ctypes.byref(ptr), h, ctypes.byref(err)), err)
                self._own.append(ptr.value)
                handles.append(h.raw)
        except Exception as exc:  # noqa: BLE001 -- reported through the exchange
            local_error = f"{type(exc).__name__}: {exc}"
        everyone = exchange((local_error, tuple(handles)))
        bad = [f"rank {q}: {e}" for q, (e, _) in enumerate(everyone) if e is not None]
        recv, flags = [], []
        if not bad:
            try:
                for q in range(world):
                    if q == rank:
                        recv.append(self._own[0])
                        flags.append(self._own[1])
                        continue
                    got = []
                    for k in range(2):
                        ptr = ctypes.c_void_p()
                        nat.raise_for(lib.dse_p2p_open(device, everyone[q][1][k], ctypes.byref(ptr),
                                                       ctypes.byref(err)), err)
                        got.append(ptr.value)
                        self._mapped.append(ptr.value)
                    recv.append(got[0])
                    flags.append(got[1])
            except Exception as exc:  # noqa: BLE001
                local_error = f"{type(exc).__name__}: {exc}"
            verdict = exchange(local_error)  # second collective: the mapping verdict of every rank
            bad = [f"rank {q}: {e}" for q, e in enumerate(verdict) if e is not None]
        if bad:
            self.close()
            raise ExecutionEnvironmentError("peer-memory setup failed on " + "; ".join(bad))
        self.peer_recv = [(ctypes.c_uint64 * world)(*[r + 8 * self._slot * par for r in recv]) for par in (0, 1)]
        self.peer_flags = (ctypes.c_uint64 * world)(*flags)
        self.recv_local = [self._own[0] + 8 * self._slot * par for par in (0, 1)]
        self.epoch = 0
        self.timed_out = torch.zeros(1, dtype=torch.int32, device=dev)

    def step(self, stream: int, relax=None, solve=None):
        import ctypes
        err = self._nat.DseErr()
        lib = self._lib
        par = self.epoch & 1
        self._nat.raise_for(lib.dse_sharded_sweep_push(self.sw.handle, self.peer_recv[par], self.world, self.rank,
                                                       self.per, stream, ctypes.byref(err)), err)
        self.epoch += 1
        self._nat.raise_for(lib.dse_p2p_barrier(self.peer_flags, self.world, self.rank, self.epoch,
                                                self.timed_out.data_ptr(), stream, ctypes.byref(err)), err)
        self._assemble(self.recv_local[par], stream, relax, solve)
        return self.delta

    def close(self) -> None:
        for q in self._mapped:
            self._lib.dse_p2p_close(q, 0)
        for q in self._own:
            self._lib.dse_p2p_close(q, 1)
        self._mapped, self._own = [], []


def select_stepper(sw, n: int, world: int, rank: int, local: int, dev, dist, probe_state=None):
    """The multi-GPU step a solve (and the torchrun bench) runs: the
    peer-memory step when the sweeper uses the pairs arithmetic, DSE_P2P is
    not 0, every rank maps its peers, and one step from `probe_state` agrees
    BITWISE with the NCCL step on every rank (and no barrier timed out);
    else the NCCL step.  Every rank runs the same collectives on every path.
    Returns (stepper, note)."""
    import torch
    from . import _native as nat

    def gather_into(out, buf):
        dist.all_gather_into_tensor(out, buf)

    fused = FusedShardedStep(sw, n, world, dev, gather_into)
    if os.environ.get("DSE_P2P", "1") == "0":
        return fused, "NCCL all-gather (DSE_P2P=0)"
    if sw.arith_code != nat.ARITH_PAIRS:
        return fused, "NCCL all-gather (the fused peer-memory push needs the pairs arithmetic)"

    def exchange(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out
    try:
        p2p = P2PShardedStep(sw, n, world, rank, local, dev, exchange)
    except ExecutionEnvironmentError as exc:  # raised on every rank together
        return fused, f"NCCL all-gather (peer memory: {str(exc)[:120]})"
    sp = torch.cuda.current_stream(dev).cuda_stream
    a, b = probe_state if probe_state is not None else (
        torch.ones(n, dtype=torch.float64, device=dev), torch.full((n,), 0.3, dtype=torch.float64, device=dev))
    ok_here, why = 0, "peer-memory step disagreed with the NCCL step or timed out on some rank"
    try:
        fused.load(a, b, sp)
        fused.step(sp)
        ref = torch.cat([device_view(fused.state_ptrs[0], n, dev), device_view(fused.state_ptrs[1], n, dev)]).clone()
        p2p.load(a, b, sp)
        p2p.step(sp)
        got = torch.cat([device_view(fused.state_ptrs[0], n, dev), device_view(fused.state_ptrs[1], n, dev)])
        torch.cuda.synchronize()
        ok_here = int(bool(torch.equal(got, ref)) and int(p2p.timed_out.item()) == 0)
    except Exception as exc:  # noqa: BLE001
        ok_here, why = 0, f"{type(exc).__name__}: {str(exc)[:120]}"
    flag = torch.tensor([ok_here], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) == 1:
        return p2p, "peer-memory all-gather fused into the sweep (validated bitwise against the NCCL step)"
    torch.cuda.synchronize()
    dist.barrier()  # no peer may unmap a buffer another rank still writes
    p2p.close()
    return fused, f"NCCL all-gather ({why})"


class ShardedSolver:
    """The public multi-GPU path (solve / iterate_once with gpus = W under
    torchrun): rank r owns rows r, r+W, ... of a row-sharded sweeper; one
    iteration is the selected step (peer-memory push or NCCL all-gather)
    with relaxation, deltas, history row and stop flag on the device;
    WindowedStopLoop reads the history once per window.  Iterations queued
    past the stop inside a window are no-ops on the device (the stop flag),
    so nothing is computed past convergence and the result (state,
    iterations, history) is that of the eager loop and bitwise the
    single-GPU solve's.  A non-finite sweep stops every rank at the same
    iteration and every rank raises the same NumericalFailureError (lowest
    failing row over the ranks)."""

    def __init__(self, grid, params, variant, window: int = 16):
        from .solver import GpuSweeper, resolve_gpus
        torch, dist = _torch_env()
        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        if resolve_gpus(variant) != self.world:
            raise ParameterError(f"variant asks for {resolve_gpus(variant)} GPUs, world size is {self.world}")
        self.local = int(os.environ.get("LOCAL_RANK", torch.cuda.current_device()))
        self.dev = torch.device("cuda", self.local)
        self.grid, self.params, self.window = grid, params, window
        self.n = grid.n_ext
        self.sw = GpuSweeper(grid, params, variant.interp, variant.arith, self.local, rows=(self.rank, self.world))
        self.stepper, self.note = select_stepper(self.sw, self.n, self.world, self.rank, self.local, self.dev, dist)
        self.stop = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._lib = self.sw.lib

    @property
    def stream(self) -> int:
        return self.torch.cuda.current_stream(self.dev).cuda_stream

    def _state(self):
        ptrs = self.stepper.state_ptrs
        return (device_view(ptrs[0], self.n, self.dev).cpu().numpy(),
                device_view(ptrs[1], self.n, self.dev).cpu().numpy())

    def locate(self):
        """Collective: (row, radial, angular) of the lowest failing row."""
        from .errors import NumericalFailureError
        torch = self.torch
        mine = [np.iinfo(np.int64).max, -1, -1]
        try:
            self.sw.check()
        except NumericalFailureError as exc:
            mine = [int(exc.row), int(exc.radial), int(exc.angular)]
        t = torch.tensor(mine, dtype=torch.int64, device=self.dev)
        out = torch.empty((self.world, 3), dtype=torch.int64, device=self.dev)
        self.dist.all_gather_into_tensor(out, t)
        rows = out.cpu().numpy()
        best = rows[np.argmin(rows[:, 0])]
        return int(best[0]), int(best[1]), int(best[2])

    def _load(self, a, b):
        torch = self.torch
        ta = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.dev)
        tb = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).to(self.dev)
        self.stepper.load(ta, tb, self.stream)

    def solve(self, a0, b0, probes_p2, xi: float, cap: int, relaxation: float):
        import ctypes
        torch = self.torch
        P = len(probes_p2)
        W = 3 + 2 * P
        hist = torch.full((cap + 1, W), float("nan"), dtype=torch.float64, device=self.dev)
        probes = torch.tensor(list(probes_p2), dtype=torch.float64, device=self.dev)
        self._load(a0, b0)
        self.stop.zero_()
        nat = self.sw.lib
        nat.dse_sharded_set_stop(self.sw.handle, ctypes.c_void_p(self.stop.data_ptr()))
        row_bytes = W * 8
        base = hist.data_ptr()
        try:
            def step(n):
                self.stepper.step(self.stream, relaxation, (xi, n, probes, base + n * row_bytes))

            def read(lo, hi):
                rows = hist[lo:hi + 1].cpu().numpy()  # stream-ordered after the window's steps
                return rows, int(self.stop.item())
            n, conv = WindowedStopLoop(step, read, self.locate).run(xi, cap, self.window)
        finally:
            nat.dse_sharded_set_stop(self.sw.handle, None)
        a, b = self._state()
        h = hist[: n + 1].cpu().numpy()
        h[0, 0], h[0, 1], h[0, 2] = 0.0, np.nan, np.nan
        if P:
            from .interpolation import interp_search_many
            h[0, 3:3 + P] = interp_search_many(self.grid.p2_ext, a0, list(probes_p2))
            h[0, 3 + P:] = interp_search_many(self.grid.p2_ext, b0, list(probes_p2))
        return a, b, n, conv, h

    def sweep(self, a, b):
        """One sweep (iterate_once): the solve loop capped at one iteration
        with xi = 0 (never met: deltas are >= 0), so a non-finite sweep
        leaves the input state in place for the failure location and every
        rank raises the same NumericalFailureError (without iteration)."""
        from .errors import NumericalFailureError
        try:
            a1, b1, _, _, _ = self.solve(a, b, (), 0.0, 1, 1.0)
        except NumericalFailureError as exc:
            exc.iteration = None
            raise
        return a1, b1

    def close(self) -> None:
        self.torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()  # no peer may unmap a buffer another rank still writes
        self.stepper.close()
        self.sw.close()


_SOLVERS: dict = {}


def sharded_solver(grid, params, variant) -> ShardedSolver:
    """ShardedSolver cached per (grid, params, variant, rank, world, device)
    like the single-GPU sweeper cache (solver._make_sweeper): repeated
    iterate_once / solve calls under torchrun reuse the uploaded grid, the
    plan and the peer mappings."""
    from .solver import _params_key
    torch, dist = _torch_env()
    key = (id(grid), _params_key(params), variant.interp, variant.arith, dist.get_rank(), dist.get_world_size(),
           int(os.environ.get("LOCAL_RANK", torch.cuda.current_device())))
    hit = _SOLVERS.get(key)
    if hit is not None and hit.grid is grid:
        return hit
    close_solvers()
    ctx = ShardedSolver(grid, params, variant)
    _SOLVERS[key] = ctx
    return ctx


def close_solvers() -> None:
    while _SOLVERS:
        _SOLVERS.popitem()[1].close()


def solve_sharded(grid, params, variant, a0, b0, probes_p2):
    ctx = sharded_solver(grid, params, variant)
    return ctx.solve(a0, b0, probes_p2, float(params.xi), int(params.max_iterations), float(params.relaxation))


def iterate_once_sharded(grid, a, b, params, variant):
    return sharded_solver(grid, params, variant).sweep(a, b)


def bench_main(args, metric, unit, cfg, flop_per_point):
    """bench.py under torchrun: config 2's rows split cyclically over the
    ranks (a fixed problem: strong scaling); each step = local sweep of the
    owned rows + NCCL all-gather + relaxation/max-norm deltas on every rank,
    from the same synthetic state.  L2 flushed before every timed step, CUDA
    events on every rank, max over ranks.  e2e: the public iterate_once with
    pinned host buffers through the same sharded path."""
    import json
    import time

    import torch
    import torch.distributed as dist

    from . import VARIANTS, ModelParams, build_grid, iterate_once
    from . import _native as nat
    # the bench contract is ONE JSON line on stdout: the NCCL/c10d version
    # banner (printed on fd 1 at the first communicator) goes to stderr
    import sys
    sys.stdout.flush()
    saved_stdout = os.dup(1)
    os.dup2(2, 1)
    # NCCL's communicator lines (rank count per communicator) on stderr
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ["DSE_DEVICE"] = str(local)
    grid = build_grid(cfg["N"], cfg["M"], cfg["K"], cfg["p2_min"], cfg["p2_max"])
    params = ModelParams(N=cfg["N"], m_rad=cfg["M"], m_ang=cfg["K"], xi=1e-10)
    variant = VARIANTS["indexed-gpu-pairs"].with_gpus(world)
    # the public path's own solver object: the step timed here is the one
    # solve() / iterate_once() run (peer-memory push when it validates)
    ctx = sharded_solver(grid, params, variant)
    sw, dev, stepper, p2p_note = ctx.sw, ctx.dev, ctx.stepper, ctx.note
    a = torch.ones(grid.n_ext, dtype=torch.float64, device=dev)
    b = torch.full((grid.n_ext,), 0.3, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    sp = torch.cuda.current_stream(dev).cuda_stream
    exchanger = stepper if stepper.kind == "p2p" else None
    # the solve's own step: assemble with relaxation, deltas, the history row
    # (probes at the default log10 p) and the device stop flag
    import ctypes
    probes = torch.tensor([10.0 ** (2.0 * lp) for lp in (-2.5, 0.0)], dtype=torch.float64, device=dev)
    hist = torch.zeros((2, 3 + 2 * probes.numel()), dtype=torch.float64, device=dev)
    sw.lib.dse_sharded_set_stop(sw.handle, ctypes.c_void_p(ctx.stop.data_ptr()))

    def step():
        # every step sweeps the same synthetic state (config 2 diverges,
        # SURVEY F3): reload (untimed below), then sweep + exchange + assemble
        return stepper.step(sp, params.relaxation, (params.xi, 1, probes, hist[1].data_ptr()))

    for _ in range(args.warmup):
        stepper.load(a, b, sp)
        ctx.stop.zero_()
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = nat.launch_count()
    clk = None
    if rank == 0:
        from bench import ClockSampler  # the repo's bench.py (rank 0 samples its GPU's clocks)
        clk = ClockSampler(local).__enter__()
    for e0, e1 in ev:
        stepper.load(a, b, sp)
        ctx.stop.zero_()
        flush.fill_(1)
        e0.record()
        step()
        e1.record()
    torch.cuda.synchronize()
    if clk is not None:
        clk.__exit__(None, None, None)
    launches = nat.launch_count() - launches0
    sw.lib.dse_sharded_set_stop(sw.handle, None)
    dist.barrier()
    mine = torch.tensor([sum(e0.elapsed_time(e1) for e0, e1 in ev) / 1e3], device=dev)
    per_rank = torch.empty(world, dtype=mine.dtype, device=dev)
    dist.all_gather_into_tensor(per_rank, mine)
    per_rank_ms = [1e3 * float(x) / args.steps for x in per_rank.cpu()]
    t = max(float(x) for x in per_rank.cpu())  # max over ranks
    st = sw.stats()
    evald = torch.tensor([float(st["evaluated_points"])], device=dev)
    dist.all_reduce(evald, op=dist.ReduceOp.SUM)
    nominal = cfg["N"] * cfg["M"] * cfg["K"]
    # e2e through the public API (pinned host arrays, H2D + D2H every step)
    a_h = torch.ones(grid.n_ext, dtype=torch.float64).pin_memory().numpy()
    b_h = torch.full((grid.n_ext,), 0.3, dtype=torch.float64).pin_memory().numpy()
    iterate_once(grid, a_h, b_h, params, variant)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        iterate_once(grid, a_h, b_h, params, variant)
    te = torch.tensor([time.perf_counter() - t0], device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    peak = None
    try:
        import ctypes
        v = ctypes.c_double(0)
        err = nat.DseErr()
        if nat.load().dse_fp64_peak(local, ctypes.byref(v), ctypes.byref(err)) == 0:
            peak = v.value
    except Exception:  # noqa: BLE001
        peak = None
    achieved = float(evald.item()) * flop_per_point / t * args.steps / 1e12 / world  # per GPU
    # BASELINE config 4 (finite-mu sweep, replicas): rank r solves the mu
    # values r, r + W, ... of the 32 midpoints on [0, 0.4] GeV on its GPU;
    # device-timed per rank (events around the rank's solves), max over ranks
    mu_block = None
    if os.environ.get("DSE_BENCH_MU", "1") != "0":
        from .finite_mu import owned_mus, solve_mu_batch
        from .mu_grid import MuParams, grid_for
        mprm = MuParams()
        mg = grid_for(mprm)
        mus = [0.4 * (k + 0.5) / 32 for k in range(32)]
        mine = owned_mus(mus, rank, world)
        from dataclasses import replace as _replace
        mprm_mo = _replace(mprm, mode="moments")  # one moment table per rank, shared by its mu values
        solve_mu_batch(mine[:1], mprm, mg, local)  # warm-up
        torch.cuda.synchronize()
        dist.barrier()
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record()
        from .finite_mu import solve_mu_batch_sa
        # one moment table per rank; its mu values swept 4 per launch (8 GPUs:
        # one batch each) by plain successive approximation (iteration-equivalent)
        sols = solve_mu_batch_sa(mine, mprm_mo, mg, batch=4, device=local) if mine else []
        m1.record()
        torch.cuda.synchronize()
        tm = torch.tensor([m0.elapsed_time(m1) / 1e3], device=dev)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        its = torch.tensor([float(sum(s.iterations for s in sols))], device=dev)
        dist.all_reduce(its, op=dist.ReduceOp.SUM)
        mu_block = {"config4_solves": len(mus), "seconds": float(tm.item()), "solves_per_s": len(mus) / float(tm.item()),
                    "solves_per_gpu": len(mine), "iterations_total": int(its.item()),
                    "layout": "mu values dealt cyclically over the ranks, no collective (replicas)",
                    "vertex": mprm.vertex,
                    "mode": "moments (table built once per rank inside the timed region), 4 mu values per "
                            "batched launch, successive approximation (iteration counts of the standalone solves)"}
        # config 3 with its 16384 external points sharded over the ranks: one
        # iteration = sweep the owned points + pack | NCCL all-gather | assemble
        import ctypes
        from .finite_mu import MuSweeper, _c_params
        per_mu = math.ceil(mg.n_ext / world)
        send = torch.zeros((3, per_mu, 2), dtype=torch.float64, device=dev)
        recv = torch.zeros((world, 3, per_mu, 2), dtype=torch.float64, device=dev)
        dl = torch.zeros(3, dtype=torch.float64, device=dev)
        init = [torch.full((mg.n_ext,), v, dtype=torch.complex128, device=dev) for v in (1.0, 0.3, 1.0)]
        cpm = _c_params(mprm)
        lib = nat.load()
        err = nat.DseErr()
        ms = []
        with MuSweeper(mg, mprm, local, row_start=rank, row_stride=world) as msw:
            for k in range(args.warmup + 5):
                nat.raise_for(lib.dse_mu_solve_load(msw.handle, *[t.data_ptr() for t in init], sp,
                                                    ctypes.byref(err)), err)
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                nat.raise_for(lib.dse_mu_sharded_sweep_pack(msw.handle, ctypes.byref(cpm), send.data_ptr(), per_mu,
                                                            sp, ctypes.byref(err)), err)
                dist.all_gather_into_tensor(recv, send)
                nat.raise_for(lib.dse_mu_sharded_assemble(msw.handle, recv.data_ptr(), world, per_mu, 1.0,
                                                          dl.data_ptr(), sp, ctypes.byref(err)), err)
                e1.record()
                torch.cuda.synchronize()
                if k >= args.warmup:
                    ms.append(e0.elapsed_time(e1))
            nom = torch.tensor([float(msw.stats()["nominal_points"])], device=dev)
        tmu = torch.tensor([float(np.median(ms)) / 1e3], device=dev)
        dist.all_reduce(tmu, op=dist.ReduceOp.MAX)
        dist.all_reduce(nom, op=dist.ReduceOp.SUM)
        mu_block["config3_sharded"] = {"ms_per_iteration": 1e3 * float(tmu.item()),
                                       "nominal_points_per_s": float(nom.item()) / float(tmu.item()),
                                       "step": "sweep owned points + pack | NCCL all-gather | assemble + deltas",
                                       "l2": "flushed before every timed step"}
    sys.stdout.flush()
    os.dup2(saved_stdout, 1)
    os.close(saved_stdout)
    if rank == 0:
        print(json.dumps({
            "metric": metric, "value": nominal * args.steps / t, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "config2_vacuum_1024x1024x256", "parallelism": f"rows cyclic over {world} GPUs",
                       "collective": "NCCL all_gather of [A'|B'] rows per step",
                       "step": ("sweep owned rows + push each finished row to every GPU (NVLink peer stores) | "
                                "flag barrier | assemble + deltas" if exchanger is not None else
                                "sweep owned rows + pack (libdse) | all_gather (NCCL) | assemble + deltas (libdse)"),
                       "all_gather": p2p_note,
                       "l2": "flushed (256 MiB write) before every timed step",
                       "evaluated_points_per_step": int(evald.item()), "nominal_points_per_step": nominal},
            "e2e": {"value": nominal * args.steps / float(te.item()), "unit": unit,
                    "h2d_bytes_per_step": 2 * grid.n_ext * 8, "d2h_bytes_per_step": 2 * grid.n_ext * 8,
                    "api": "paper_2012_03667_b200.iterate_once(grid, A, B, params, "
                           "VARIANTS['indexed-gpu-pairs'].with_gpus(W)) under torchrun"},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": None,
                         "flop_per_point": flop_per_point, "points": "evaluated, per GPU",
                         "peak_source": "builder-measured: dse_fp64_peak DFMA probe, in process, per GPU (MEASURED_PEAKS.json has no fp64 figure)"},
            "gpu_launches": launches,
            "per_rank_ms_per_step": per_rank_ms,
            "clocks": clk.summary() if clk is not None else None,
            "finite_mu": mu_block,
        }))
    close_solvers()
    dist.destroy_process_group()
    return 0
