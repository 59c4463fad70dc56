"""Finite chemical potential solves on the GPU (BASELINE configs 3-4).

The reference has no finite-mu path:
this module extends the drop-in's vacuum API (solve / iterate_once /
solve_batch, solver.py:201-266) to the complex dressing functions A, B, C of
S^-1(p~) = i gamma.p A + i gamma_4 p~4 C + B on the 2-D external grid
(|p|, p4 + i mu) of mu_grid.py, with the same conventions: a Jacobi sweep,
the optional relaxation blend (solver.py:249-251), the max-norm stop rule
all(d < xi) over |dA|, |dB|, |dC| (iteration.py:34-38), cap -> converged=False
(iteration.py:40), the error classes of errors.py.

Everything numeric runs in libdse_b200.so (dse_mu_* in include/dse_b200.h):
the whole loop is one cooperative kernel launch per solve.  There is no CPU
fallback.  The equations are in DESIGN.md "Finite chemical potential"; the CPU
oracle (test infrastructure only) is oracle/mu_oracle.py.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native as nat
from .errors import NumericalFailureError, ParameterError
from .mu_grid import MODES, VERTICES, MuGrid, MuParams, build_mu_grid, grid_for

__all__ = ["MuIterationRecord", "MuSolution", "MuSweeper", "solve_mu", "iterate_mu_once", "solve_mu_batch",
           "solve_mu_batch_sharded", "solve_mu_sharded", "solve_mu_anderson", "solve_mu_batch_anderson", "solve_mu_newton", "NewtonReport", "owned_mus", "interp_mu", "MuParams", "MuGrid", "build_mu_grid"]


@dataclass(frozen=True)
class MuIterationRecord:
    n: int
    delta_a: float
    delta_b: float
    delta_c: float


@dataclass
class MuSolution:
    A: np.ndarray            # complex (n_s, n_4)
    B: np.ndarray
    C: np.ndarray
    iterations: int
    converged: bool
    history: list = field(repr=False)
    grid: MuGrid = field(repr=False)
    params: MuParams = field(repr=False)

    @property
    def mass(self) -> np.ndarray:
        """M = B / A (complex), the mass function on the external grid."""
        return self.B / self.A


def _check_c_projection(grid: MuGrid, p: MuParams) -> None:
    """C = z1 + P_C / p~4 needs p~4 = p4 + i mu != 0 at every external point."""
    if p.mu == 0.0 and np.any(np.asarray(grid.p4_ext) == 0.0):
        raise ParameterError("mu = 0 with an external p4 node at 0: the C projection divides by p4 + i mu")


def _c_params(p: MuParams) -> nat.DseMuParams:
    return nat.DseMuParams(coeff=p.interaction_coeff, omega=p.omega, m0=p.m0, z1=p.z1, mu=p.mu, xi=p.xi,
                           relaxation=p.relaxation, max_iterations=int(p.max_iterations),
                           vertex=VERTICES.index(p.vertex), mode=MODES.index(p.mode))


def _state(x, shape, default) -> np.ndarray:
    if x is None:
        return np.full(shape, default, dtype=np.complex128)
    a = np.array(x, dtype=np.complex128).reshape(shape)
    return np.ascontiguousarray(a)


def _ptr(a: np.ndarray):
    return a.view(np.float64).ctypes.data_as(nat.f64p)


class MuSweeper:
    """Device-resident finite-mu grid + state buffers (dse_mu_sweeper_*).
    rows row_start + r*row_stride are owned (multi-GPU sharding)."""

    def __init__(self, grid: MuGrid, params: MuParams, device: int = 0, row_start: int = 0, row_stride: int = 1):
        params.validate()
        _check_c_projection(grid, params)
        self.grid, self.params, self.device = grid, params, device
        lib = nat.load()
        self._keep = [np.ascontiguousarray(getattr(grid, n), dtype=np.float64) for n in
                      ("p_ext", "ps2_ext", "p4_ext", "q_int", "qs2_int", "q4_int", "meas_s", "meas_4", "z_nodes",
                       "z_weights")]
        bs = np.ascontiguousarray(grid.brk_s, dtype=np.int64)
        b4 = np.ascontiguousarray(grid.brk_4, dtype=np.int64)
        self._keep += [bs, b4]
        g = nat.DseMuGrid(*[a.ctypes.data_as(nat.f64p) for a in self._keep[:10]], bs.ctypes.data_as(nat.i64p),
                          b4.ctypes.data_as(nat.i64p), grid.n_s, grid.n_4, grid.m_s, grid.m_4, grid.m_ang)
        cp = _c_params(params)
        h = ctypes.c_void_p()
        err = nat.DseErr()
        nat.raise_for(lib.dse_mu_sweeper_create(ctypes.byref(g), ctypes.byref(cp), device, row_start, row_stride,
                                                ctypes.byref(h), ctypes.byref(err)), err)
        self._h = h
        self._lib = lib

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.dse_mu_sweeper_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def solve(self, params: MuParams | None = None, a0=None, b0=None, c0=None, history: bool = True) -> MuSolution:
        p = self.params if params is None else params
        p.validate()
        _check_c_projection(self.grid, p)
        shape = (self.grid.n_s, self.grid.n_4)
        A, B, C = _state(a0, shape, 1.0), _state(b0, shape, 0.3), _state(c0, shape, 1.0)
        hist = np.full((p.max_iterations + 1, 4), np.nan) if history else None
        it = ctypes.c_int64()
        conv = ctypes.c_int()
        err = nat.DseErr()
        cp = _c_params(p)
        rc = self._lib.dse_mu_solve(self._h, ctypes.byref(cp), _ptr(A), _ptr(B), _ptr(C), ctypes.byref(it),
                                    ctypes.byref(conv), hist.ctypes.data_as(nat.f64p) if hist is not None else None,
                                    ctypes.byref(err))
        nat.raise_for(rc, err)
        n = int(it.value)
        records = []
        if hist is not None:
            records = [MuIterationRecord(0, float("nan"), float("nan"), float("nan"))]
            records += [MuIterationRecord(int(r[0]), float(r[1]), float(r[2]), float(r[3])) for r in hist[1:n + 1]]
        return MuSolution(A=A, B=B, C=C, iterations=n, converged=bool(conv.value), history=records, grid=self.grid,
                          params=p)

    def sweep(self, A, B, C, params: MuParams | None = None):
        p = self.params if params is None else params
        shape = (self.grid.n_s, self.grid.n_4)
        A, B, C = _state(A, shape, 0), _state(B, shape, 0), _state(C, shape, 0)
        outs = [np.empty(shape, np.complex128) for _ in range(3)]
        err = nat.DseErr()
        cp = _c_params(p)
        rc = self._lib.dse_mu_sweep(self._h, ctypes.byref(cp), _ptr(A), _ptr(B), _ptr(C), *[_ptr(o) for o in outs],
                                    ctypes.byref(err))
        nat.raise_for(rc, err)
        return tuple(outs)

    def interp(self, F) -> np.ndarray:
        shape = (self.grid.n_s, self.grid.n_4)
        F = _state(F, shape, 0)
        out = np.empty((self.grid.m_s, self.grid.m_4), np.complex128)
        err = nat.DseErr()
        nat.raise_for(self._lib.dse_mu_interp(self._h, _ptr(F), _ptr(out), ctypes.byref(err)), err)
        return out

    def load_device(self, dA: int, dB: int, dC: int, stream: int = 0) -> None:
        """Device-resident state (complex, n_ext each, raw device addresses) as iteration 0."""
        err = nat.DseErr()
        nat.raise_for(self._lib.dse_mu_solve_load(self._h, dA, dB, dC, stream, ctypes.byref(err)), err)

    def resume(self, n_iterations: int, stream: int = 0) -> None:
        """Enqueue the next n_iterations of the on-device loop (no stop test, no sync)."""
        err = nat.DseErr()
        nat.raise_for(self._lib.dse_mu_solve_resume(self._h, n_iterations, stream, ctypes.byref(err)), err)

    def batch_sweep(self, x_in, x_out, params_list, stream: int = 0):
        """One sweep of S = 2 or 4 independent states (dse_mu_batch_sweep,
        moments mode): x_in, x_out device complex128 tensors [S, 3, n_ext];
        returns the per-solve lowest failing row (-1 = fine)."""
        S = len(params_list)
        cps = (nat.DseMuParams * S)(*[_c_params(p) for p in params_list])
        failed = (ctypes.c_int64 * S)()
        err = nat.DseErr()
        nat.raise_for(self._lib.dse_mu_batch_sweep(self._h, cps, S, x_in.data_ptr(), x_out.data_ptr(), stream,
                                                   failed, ctypes.byref(err)), err)
        return list(failed)

    def stats(self) -> dict:
        nom, ev, sm = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        blocks = ctypes.c_int32()
        self._lib.dse_mu_sweeper_stats(self._h, ctypes.byref(nom), ctypes.byref(ev), ctypes.byref(blocks),
                                       ctypes.byref(sm))
        return dict(nominal_points=nom.value, evaluated_points=ev.value, blocks=blocks.value, smem_bytes=sm.value)


def solve_mu(params: MuParams | None = None, grid: MuGrid | None = None, a0=None, b0=None, c0=None,
             device: int = 0) -> MuSolution:
    """Finite-mu analogue of solve (solver.py:221-266): A = C = 1, B = 0.3
    GeV by default (BASELINE config 3's initial guess)."""
    params = MuParams() if params is None else params
    params.validate()
    grid = grid_for(params) if grid is None else grid
    with MuSweeper(grid, params, device) as sw:
        return sw.solve(params, a0, b0, c0)


def iterate_mu_once(grid: MuGrid, A, B, C, params: MuParams, device: int = 0):
    """One Jacobi sweep (iterate_once, solver.py:201-212) -> (A', B', C')."""
    with MuSweeper(grid, params, device) as sw:
        return sw.sweep(A, B, C, params)


def solve_mu_batch(mus, params: MuParams | None = None, grid: MuGrid | None = None, device: int = 0,
                   history: bool = False) -> list:
    """Independent solves at each chemical potential in `mus` on one grid
    (BASELINE config 4: replicas, no exchange): the grid is uploaded once
    and every solve is one on-device loop."""
    params = MuParams() if params is None else params
    grid = grid_for(params) if grid is None else grid
    out = []
    with MuSweeper(grid, params, device) as sw:
        for m in mus:
            out.append(sw.solve(replace(params, mu=float(m)), history=history))
    return out


def _collective_failure(rc: int, err, world: int, dev) -> None:
    """Raise a numerical failure on EVERY rank together: the owning rank's
    location, the others a failure naming no point.  One MAX all-reduce of
    the verdict per iteration (skipped at world 1 or without an initialised
    process group), so no rank leaves the loop while the others block in
    the next all-gather."""
    import torch
    import torch.distributed as dist
    local = None
    try:
        nat.raise_for(rc, err)
    except NumericalFailureError as exc:
        local = exc
    if world > 1 and dist.is_available() and dist.is_initialized():
        flag = torch.tensor([0 if local is None else 1], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        if local is None and int(flag.item()):
            raise NumericalFailureError("non-finite integrand in the sharded sweep of another rank")
    if local is not None:
        raise local


def solve_mu_sharded(params: MuParams | None = None, grid: MuGrid | None = None, a0=None, b0=None, c0=None,
                     rank: int | None = None, world: int | None = None, device: int | None = None,
                     gather=None) -> MuSolution:
    """Config 3 with the external points sharded over the ranks of a
    torch.distributed job (rank r owns points r, r + W, ...): per iteration
    each GPU sweeps its points, the compact [3][ceil(N/W)] complex results
    are all-gathered (NCCL), and every rank rebuilds the full iterate with
    the relaxation blend and the max-norm deltas on the device; the stop
    rule and history are the single-GPU solve's, and the result is bitwise
    the single-GPU solve's (a point's reduction never depends on the owner).
    `gather(out[W,3,per,2], buf[3,per,2])` defaults to all_gather_into_tensor."""
    import ctypes
    import math

    import torch
    import torch.distributed as dist
    params = MuParams() if params is None else params
    params.validate()
    grid = grid_for(params) if grid is None else grid
    if rank is None or world is None:
        rank, world = dist.get_rank(), dist.get_world_size()
    if device is None:
        device = torch.cuda.current_device()
    if gather is None:
        def gather(out, buf):
            dist.all_gather_into_tensor(out, buf)
    dev = torch.device("cuda", device)
    shape = (grid.n_s, grid.n_4)
    n = grid.n_ext
    per = math.ceil(n / world)
    state = [torch.from_numpy(_state(x, shape, d).reshape(-1)).to(dev) for x, d in ((a0, 1.0), (b0, 0.3), (c0, 1.0))]
    send = torch.zeros((3, per, 2), dtype=torch.float64, device=dev)
    recv = torch.zeros((world, 3, per, 2), dtype=torch.float64, device=dev)
    delta = torch.zeros(3, dtype=torch.float64, device=dev)
    lib = nat.load()
    cp = _c_params(params)
    hist = [MuIterationRecord(0, float("nan"), float("nan"), float("nan"))]
    with MuSweeper(grid, params, device, row_start=rank, row_stride=world) as sw:
        err = nat.DseErr()
        st = torch.cuda.current_stream(dev).cuda_stream
        nat.raise_for(lib.dse_mu_solve_load(sw.handle, state[0].data_ptr(), state[1].data_ptr(),
                                            state[2].data_ptr(), st, ctypes.byref(err)), err)
        converged, n_it = False, params.max_iterations
        for it in range(1, params.max_iterations + 1):
            nat.raise_for(lib.dse_mu_sharded_sweep_pack(sw.handle, ctypes.byref(cp), send.data_ptr(), per, st,
                                                        ctypes.byref(err)), err)
            gather(recv, send)
            nat.raise_for(lib.dse_mu_sharded_assemble(sw.handle, recv.data_ptr(), world, per, params.relaxation,
                                                      delta.data_ptr(), st, ctypes.byref(err)), err)
            d = delta.cpu().numpy()
            _collective_failure(lib.dse_mu_sharded_failure(sw.handle, st, ctypes.byref(err)), err, world, dev)
            hist.append(MuIterationRecord(it, float(d[0]), float(d[1]), float(d[2])))
            if d[0] < params.xi and d[1] < params.xi and d[2] < params.xi:
                converged, n_it = True, it
                break
        px = ctypes.c_void_p()
        nat.raise_for(lib.dse_mu_sweeper_state(sw.handle, ctypes.byref(px)), nat.DseErr())
        from .distributed import device_view
        full = device_view(px.value, 3 * 2 * n, dev).cpu().numpy().view(np.complex128).reshape(3, *shape)
    return MuSolution(A=full[0].copy(), B=full[1].copy(), C=full[2].copy(), iterations=n_it, converged=converged,
                      history=hist, grid=grid, params=params)


def _aa_solve(gram: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """The L x L regularised solve on the host (LAPACK, one small matrix per
    solve: identical alone or stacked), gram [..., L, L], rhs [..., L]."""
    L = gram.shape[-1]
    tr = np.real(np.trace(gram, axis1=-2, axis2=-1))
    reg = gram + (1e-14 * tr + 1e-300)[..., None, None] * np.eye(L)
    return np.linalg.solve(reg, rhs[..., None])[..., 0]


class _DeviceAnderson:
    """Anderson acceleration state of S solves on the device (dse_mu_aa_*):
    the last `depth` residual and iterate differences in ring slots, the
    residual, deltas, new Gram column and right-hand side formed by two
    kernels and copied to the host in one transfer per sweep; the Gram matrix
    is kept on the host (one new column per sweep) and the depth x depth
    system solved there (_aa_solve); the update is one kernel.  Every solve is
    processed by the same per-solve code: a solve batched with others is
    bitwise its standalone run."""

    def __init__(self, S: int, n_ext: int, depth: int, beta: float, dev, stream: int):
        import torch
        if not 1 <= depth <= 16:
            raise ParameterError("Anderson depth must be in 1..16")
        self.S, self.n, self.depth, self.beta, self.stream = S, n_ext, depth, float(beta), stream
        N = 3 * n_ext

        def z(*shape):
            return torch.zeros(shape, dtype=torch.complex128, device=dev)
        self.f, self.fprev, self.xprev = z(S, N), z(S, N), z(S, N)
        self.dF, self.dX = z(S, depth, N), z(S, depth, N)
        self.scratch = torch.zeros(3 * S + 4 * S * depth, dtype=torch.float64, device=dev)
        self.host = np.zeros(3 * S + 4 * S * depth)
        self.G = np.zeros((S, depth, depth), dtype=np.complex128)
        self.count = 0          # differences formed so far
        self.started = False
        self.cols = np.zeros(0, dtype=np.int32)
        self.rhs = None
        self.lib = nat.load()

    def residual(self, x, gx) -> np.ndarray:
        """f = gx - x and the new difference; returns max |f| [S, 3] (A, B, C)."""
        S, depth = self.S, self.depth
        slot = -1
        if self.started:
            slot = self.count % depth
            self.count += 1
        L = min(self.count, depth)
        self.cols = np.array([(self.count - L + k) % depth for k in range(L)], dtype=np.int32)
        err = nat.DseErr()
        nat.raise_for(self.lib.dse_mu_aa_residual(
            S, self.n, x.data_ptr(), gx.data_ptr(), self.f.data_ptr(), self.fprev.data_ptr(), self.xprev.data_ptr(),
            self.dF.data_ptr(), self.dX.data_ptr(), depth, slot, self.cols.ctypes.data_as(nat.i32p), L,
            self.scratch.data_ptr(), self.host.ctypes.data_as(nat.f64p), self.stream, ctypes.byref(err)), err)
        self.started = True
        if L:
            c = self.host[:4 * S * L].view(np.complex128).reshape(S, 2, L)
            for k, col in enumerate(self.cols):
                self.G[:, slot, col] = np.conj(c[:, 0, k])
                self.G[:, col, slot] = c[:, 0, k]
            self.rhs = c[:, 1, :].copy()
        return self.host[4 * S * L:4 * S * L + 3 * S].reshape(S, 3).copy()

    def update(self, x) -> None:
        """x <- x + beta f - (dX + beta dF) gamma, in place."""
        L = len(self.cols)
        gamma = np.zeros((self.S, 0), dtype=np.complex128)
        if L:
            gamma = np.ascontiguousarray(_aa_solve(self.G[:, self.cols][:, :, self.cols], self.rhs))
        err = nat.DseErr()
        nat.raise_for(self.lib.dse_mu_aa_update(
            self.S, self.n, x.data_ptr(), self.f.data_ptr(), self.dF.data_ptr(), self.dX.data_ptr(), self.depth,
            self.cols.ctypes.data_as(nat.i32p), L, gamma.view(np.float64).ctypes.data_as(nat.f64p), self.beta,
            self.stream, ctypes.byref(err)), err)


def solve_mu_anderson(params: MuParams | None = None, grid: MuGrid | None = None, a0=None, b0=None, c0=None,
                      depth: int = 8, beta: float = 1.0, device: int = 0, sweeper: "MuSweeper | None" = None
                      ) -> MuSolution:
    """Finite-mu solve with Anderson acceleration (type II, depth m) of the
    same fixed-point map g = one Jacobi sweep: x <- x + beta f - (dX + beta dF) gamma,
    gamma = argmin |f - dF gamma| over the last m residual differences
    (normal equations, m x m, on the device).  Stops when max|g(x) - x| of
    A, B and C are all < xi (the successive-approximation rule applied to
    the sweep's update).  The reference has no finite-mu solver; this is an
    option next to solve_mu's plain successive approximation (it converges
    to the same fixed point in fewer sweeps: config 3 25 vs 63; it does NOT
    rescue the divergent full 'bc' vertex).  params.relaxation is ignored
    (beta plays its role); history rows hold max|g(x) - x| per function."""
    import ctypes

    import torch
    params = MuParams() if params is None else params
    params.validate()
    grid = grid_for(params) if grid is None else grid
    _check_c_projection(grid, params)
    dev = torch.device("cuda", device)
    n = grid.n_ext
    shape = (grid.n_s, grid.n_4)
    x = torch.cat([torch.from_numpy(_state(v, shape, d).reshape(-1)) for v, d in ((a0, 1.0), (b0, 0.3), (c0, 1.0))])
    x = x.to(dev)
    send = torch.zeros(3 * n, dtype=torch.complex128, device=dev)
    lib = nat.load()
    cp = _c_params(params)
    own = sweeper is None
    sw = MuSweeper(grid, params, device) if own else sweeper
    hist = [MuIterationRecord(0, float("nan"), float("nan"), float("nan"))]
    converged, n_it = False, params.max_iterations
    try:
        st = torch.cuda.current_stream(dev).cuda_stream
        err = nat.DseErr()
        aa = _DeviceAnderson(1, n, depth, beta, dev, st)
        for it in range(1, params.max_iterations + 1):
            nat.raise_for(lib.dse_mu_solve_load(sw.handle, x[:n].data_ptr(), x[n:2 * n].data_ptr(),
                                                x[2 * n:].data_ptr(), st, ctypes.byref(err)), err)
            nat.raise_for(lib.dse_mu_sharded_sweep_pack(sw.handle, ctypes.byref(cp), send.data_ptr(), n, st,
                                                        ctypes.byref(err)), err)
            nat.raise_for(lib.dse_mu_sharded_failure(sw.handle, st, ctypes.byref(err)), err)
            d = aa.residual(x, send)[0]
            hist.append(MuIterationRecord(it, float(d[0]), float(d[1]), float(d[2])))
            if d[0] < params.xi and d[1] < params.xi and d[2] < params.xi:
                x = send.clone()
                converged, n_it = True, it
                break
            aa.update(x)
    finally:
        if own:
            sw.close()
    xs = x.cpu().numpy()
    A, B, C = (xs[k * n:(k + 1) * n].reshape(shape).copy() for k in range(3))
    return MuSolution(A=A, B=B, C=C, iterations=n_it, converged=converged, history=hist, grid=grid, params=params)


def solve_mu_batch_anderson(mus, params: MuParams | None = None, grid: MuGrid | None = None, depth: int = 8,
                            beta: float = 1.0, batch: int = 4, device: int = 0) -> list:
    """BASELINE config 4 on one GPU: the mu values in groups of `batch`
    (2 or 4) swept together by dse_mu_batch_sweep (one moment table for all,
    read once per pair per group sweep), each solve Anderson-accelerated like
    solve_mu_anderson (same update, same stop rule, its own history)."""
    import torch
    params = MuParams() if params is None else params
    params = replace(params, mode="moments")
    params.validate()
    grid = grid_for(params) if grid is None else grid
    if batch not in (2, 4):
        raise ParameterError("batch must be 2 or 4")
    dev = torch.device("cuda", device)
    n = grid.n_ext
    shape = (grid.n_s, grid.n_4)
    init = torch.cat([torch.full((n,), v, dtype=torch.complex128) for v in (1.0, 0.3, 1.0)]).to(dev)
    out_all = []
    with MuSweeper(grid, params, device) as sw:
        mus = list(mus)
        for g0 in range(0, len(mus), batch):
            group = mus[g0:g0 + batch]
            S = 4 if len(group) > 2 else 2
            plist = [replace(params, mu=float(m)) for m in group]
            plist += [plist[-1]] * (S - len(plist))  # pad with a repeat (its result is dropped)
            for p_ in plist:
                _check_c_projection(grid, p_)
            x = init.repeat(S, 1).contiguous()
            gx = torch.empty_like(x)
            aa = _DeviceAnderson(S, n, depth, beta, dev, torch.cuda.current_stream(dev).cuda_stream)
            hist = [[MuIterationRecord(0, float("nan"), float("nan"), float("nan"))] for _ in range(S)]
            res = [None] * S
            its = [params.max_iterations] * S
            for it in range(1, params.max_iterations + 1):
                failed = sw.batch_sweep(x, gx, plist, torch.cuda.current_stream(dev).cuda_stream)
                for s in range(S):
                    if res[s] is None and failed[s] >= 0:
                        from .errors import NumericalFailureError
                        raise NumericalFailureError(f"non-finite integrand in batched finite-mu sweep, mu="
                                                    f"{plist[s].mu}, row={failed[s]}", row=failed[s], iteration=it)
                d = aa.residual(x, gx)
                for s in range(S):
                    if res[s] is not None:
                        continue
                    hist[s].append(MuIterationRecord(it, float(d[s, 0]), float(d[s, 1]), float(d[s, 2])))
                    if d[s, 0] < params.xi and d[s, 1] < params.xi and d[s, 2] < params.xi:
                        res[s] = gx[s].clone()
                        its[s] = it
                if all(r is not None for r in res):
                    break
                aa.update(x)
            for s in range(len(group)):
                xs = (res[s] if res[s] is not None else x[s]).cpu().numpy()
                A, B, C = (xs[k * n:(k + 1) * n].reshape(shape).copy() for k in range(3))
                out_all.append(MuSolution(A=A, B=B, C=C, iterations=its[s], converged=res[s] is not None,
                                          history=hist[s], grid=grid, params=plist[s]))
    return out_all


def solve_mu_batch_sa(mus, params: MuParams | None = None, grid: MuGrid | None = None, batch: int = 4,
                      device: int = 0) -> list:
    """BASELINE config 4 on one GPU by plain successive approximation -- the
    parity-equivalent path: every solve is solve_mu's loop (same sweep, same
    max-norm deltas, same strict stop rule, iteration.py:18-40), so its
    iterations, state and history are bitwise those of the standalone solve.
    The mu values run `batch` (2 or 4) at a time, each group as ONE
    cooperative launch (dse_mu_batch_solve: the device-resident loop of the
    single solve, run per solve) that reads each pair's five moments once per
    group sweep (moments mode: one table for all mu values, built once) and
    stops sweeping a solve once it has stopped; no host round trip per
    iteration.  relaxation != 1 runs the solves one by one (solve_mu_batch)."""
    import torch
    params = MuParams() if params is None else params
    params = replace(params, mode="moments")
    params.validate()
    grid = grid_for(params) if grid is None else grid
    if batch not in (2, 4):
        raise ParameterError("batch must be 2 or 4")
    if params.relaxation != 1.0:
        return solve_mu_batch(mus, params, grid, device, history=True)
    dev = torch.device("cuda", device)
    n = grid.n_ext
    shape = (grid.n_s, grid.n_4)
    init = torch.cat([torch.full((n,), v, dtype=torch.complex128) for v in (1.0, 0.3, 1.0)]).to(dev)
    lib = nat.load()
    out_all = []
    cap = params.max_iterations
    with MuSweeper(grid, params, device) as sw:
        mus = list(mus)
        st = torch.cuda.current_stream(dev).cuda_stream
        hist = torch.full((batch, cap + 1, 4), float("nan"), dtype=torch.float64, device=dev)
        for g0 in range(0, len(mus), batch):
            group = mus[g0:g0 + batch]
            S = 4 if len(group) > 2 else 2
            plist = [replace(params, mu=float(m)) for m in group]
            plist += [plist[-1]] * (S - len(plist))  # pad with a repeat (its result is dropped)
            for p_ in plist:
                _check_c_projection(grid, p_)
            x0 = init.repeat(S, 1).contiguous()
            x1 = torch.empty_like(x0)
            cps = (nat.DseMuParams * S)(*[_c_params(p_) for p_ in plist])
            its = (ctypes.c_int64 * S)()
            conv = (ctypes.c_int32 * S)()
            fit = (ctypes.c_int64 * S)()
            frow = (ctypes.c_int64 * S)()
            err = nat.DseErr()
            nat.raise_for(lib.dse_mu_batch_solve(sw.handle, cps, S, x0.data_ptr(), x1.data_ptr(), hist.data_ptr(),
                                                 cap + 1, its, conv, fit, frow, st, ctypes.byref(err)), err)
            for s_ in range(len(group)):
                if fit[s_] > 0:
                    raise NumericalFailureError(f"non-finite integrand in batched finite-mu sweep, mu="
                                                f"{plist[s_].mu}, row={frow[s_]}", row=frow[s_], iteration=fit[s_])
            h = hist[:S].cpu().numpy()
            for s_ in range(len(group)):
                n_it = int(its[s_])
                xs = (x0 if n_it % 2 == 0 else x1)[s_].cpu().numpy()
                A, B, C = (xs[k * n:(k + 1) * n].reshape(shape).copy() for k in range(3))
                rec = [MuIterationRecord(0, float("nan"), float("nan"), float("nan"))]
                rec += [MuIterationRecord(int(r[0]), float(r[1]), float(r[2]), float(r[3])) for r in h[s_, 1:n_it + 1]]
                out_all.append(MuSolution(A=A, B=B, C=C, iterations=n_it, converged=bool(conv[s_]),
                                          history=rec, grid=grid, params=plist[s_]))
    return out_all


def owned_mus(mus, rank: int, world: int) -> list:
    """The chemical potentials rank `rank` of `world` solves (config 4 is
    replicas: mu values are dealt cyclically, no data-path collective)."""
    return list(mus)[rank::world]


def solve_mu_batch_sharded(mus, params: MuParams | None = None, grid: MuGrid | None = None, device: int = 0,
                           rank: int | None = None, world: int | None = None) -> list:
    """BASELINE config 4 across the ranks of a torch.distributed job (one
    process per GPU): rank r solves owned_mus(mus, r, W) on its GPU -- by
    solve_mu_batch_sa (4 mu values per cooperative launch, one moment table
    per rank; bitwise the standalone solves) when the relaxation is 1, else
    one by one -- then the (mu, iterations, converged, A, B, C) records are
    all-gathered so every rank returns the full list in the order of `mus`."""
    import torch.distributed as dist
    if rank is None or world is None:
        rank, world = dist.get_rank(), dist.get_world_size()
    mine = owned_mus(mus, rank, world)
    prm = MuParams() if params is None else params
    if not mine:
        sols = []
    elif prm.relaxation == 1.0:
        sols = solve_mu_batch_sa(mine, prm, grid, batch=4 if len(mine) > 2 else 2, device=device)
    else:
        sols = solve_mu_batch(mine, prm, grid, device)
    recs = [(float(m), s.iterations, s.converged, s.A, s.B, s.C) for m, s in zip(mine, sols)]
    if world == 1:
        gathered = [recs]
    else:
        gathered = [None] * world
        dist.all_gather_object(gathered, recs)
    by_mu = {}
    for part in gathered:
        for r in part:
            by_mu[r[0]] = r
    return [by_mu[float(m)] for m in mus]


@dataclass
class NewtonReport:
    """Per-solve record of solve_mu_newton: sweeps used by the start solve
    and by the Newton steps, and per Newton step (residual max per function,
    GMRES iterations)."""
    start_iterations: int
    sweeps: int
    steps: list = field(default_factory=list)   # (step, max|F_A|, max|F_B|, max|F_C|, gmres_iterations)


def _gmres_real(matvec, b, rtol: float, restart: int, max_restarts: int, dot):
    """Restarted GMRES for J dx = b in the REAL inner product Re<u, v> of the
    complex state (the sweep is not holomorphic in (A, B, C) in general, so
    J is a real-linear map of the 2n real components).  Classical Gram-
    Schmidt applied twice (one stacked product per pass); the small
    Hessenberg least-squares problem is solved on the host."""
    import torch
    x = torch.zeros_like(b)
    bnorm = float(dot(b, b)) ** 0.5
    if bnorm == 0.0:
        return x, 0
    total = 0
    r = b.clone()
    for _ in range(max_restarts):
        beta = float(dot(r, r)) ** 0.5
        if beta <= rtol * bnorm:
            break
        V = torch.zeros((restart + 1, b.numel()), dtype=b.dtype, device=b.device)
        H = np.zeros((restart + 1, restart))
        V[0] = r / beta
        k_used = 0
        y = np.zeros(0)
        for k in range(restart):
            w = matvec(V[k])
            total += 1
            for _pass in range(2):
                h = torch.real(torch.conj(V[:k + 1]) @ w)
                w = w - (h.to(V.dtype)[:, None] * V[:k + 1]).sum(0)
                H[:k + 1, k] += h.cpu().numpy()
            H[k + 1, k] = float(dot(w, w)) ** 0.5
            k_used = k + 1
            e1 = np.zeros(k + 2)
            e1[0] = beta
            y, *_ = np.linalg.lstsq(H[:k + 2, :k + 1], e1, rcond=None)
            res = np.linalg.norm(H[:k + 2, :k + 1] @ y - e1)
            if H[k + 1, k] == 0.0 or res <= rtol * bnorm:
                break
            V[k + 1] = w / H[k + 1, k]
        x = x + (torch.from_numpy(y).to(V.device).to(V.dtype)[:, None] * V[:k_used]).sum(0)
        r = b - matvec(x)
        total += 1
        if float(dot(r, r)) ** 0.5 <= rtol * bnorm:
            break
    return x, total


def solve_mu_newton(params: MuParams | None = None, grid: MuGrid | None = None, a0=None, b0=None, c0=None,
                    start: str | None = "bcb", max_newton: int = 40, restart: int = 60, max_restarts: int = 4,
                    fd_eps: float = 1e-7, line_search: int = 0, device: int = 0,
                    sweeper: "MuSweeper | None" = None):
    """Finite-mu solve by Newton-Krylov on the fixed-point residual
    F(x) = g(x) - x, g = one Jacobi sweep (the device sweep of solve_mu),
    x = (A, B, C) complex: each Newton step solves J dx = -F with restarted
    GMRES in the real inner product, every Jacobian-vector product one
    forward difference of the sweep, (g(x + h v) - g(x)) / h - v with
    h = fd_eps (1 + |x|) / |v|; inexact-Newton forcing term
    min(0.1, max(1e-4, max|F|)); line_search > 0 backtracks (halving, at
    most that many extra sweeps) while |F|_2 grows.  Stops when max|F| of A, B and C are all
    < xi (the successive-approximation rule applied to the sweep's update,
    as solve_mu_anderson).

    This is the solver for the FULL in-medium Ball-Chiu vertex ('bc'):
    successive approximation, relaxation and Anderson acceleration all
    diverge on it (the sweep's Jacobian has eigenvalues far outside the unit
    circle), Newton's method does not need a contraction.  By
    default (start='bcb') the initial guess is the converged solve of the
    same parameters with the 'bcb' vertex (plain successive approximation
    on the device); start=None starts from (a0, b0, c0).  Not
    iteration-equivalent to anything in the reference (which has no finite-mu
    path).  Returns (MuSolution, NewtonReport); the solution's `iterations`
    counts Newton steps and its history rows hold max|F| per function after
    each step."""
    import torch
    params = MuParams() if params is None else params
    params.validate()
    grid = grid_for(params) if grid is None else grid
    _check_c_projection(grid, params)
    dev = torch.device("cuda", device)
    n = grid.n_ext
    shape = (grid.n_s, grid.n_4)
    lib = nat.load()
    own = sweeper is None
    sw = MuSweeper(grid, params, device) if own else sweeper
    start_its = 0
    try:
        if start is not None:
            s0 = sw.solve(replace(params, vertex=start), a0, b0, c0, history=False)
            if not s0.converged:
                raise NumericalFailureError(f"start solve ({start}) did not converge in {params.max_iterations}")
            start_its = s0.iterations
            a0, b0, c0 = s0.A, s0.B, s0.C
        x = torch.cat([torch.from_numpy(_state(v, shape, d).reshape(-1)) for v, d in ((a0, 1.0), (b0, 0.3),
                                                                                         (c0, 1.0))]).to(dev)
        gx = torch.zeros_like(x)
        cp = _c_params(params)
        st = torch.cuda.current_stream(dev).cuda_stream
        err = nat.DseErr()
        sweeps = [0]

        def g(v, out):
            nat.raise_for(lib.dse_mu_solve_load(sw.handle, v[:n].data_ptr(), v[n:2 * n].data_ptr(),
                                                v[2 * n:].data_ptr(), st, ctypes.byref(err)), err)
            nat.raise_for(lib.dse_mu_sharded_sweep_pack(sw.handle, ctypes.byref(cp), out.data_ptr(), n, st,
                                                        ctypes.byref(err)), err)
            nat.raise_for(lib.dse_mu_sharded_failure(sw.handle, st, ctypes.byref(err)), err)
            sweeps[0] += 1
            return out

        def dot(u, v):
            return torch.real(torch.vdot(u, v)).item()

        report = NewtonReport(start_iterations=start_its, sweeps=0)
        hist = [MuIterationRecord(0, float("nan"), float("nan"), float("nan"))]
        converged, step = False, 0
        gp = torch.zeros_like(x)
        for step in range(1, max_newton + 2):
            g(x, gx)
            F = gx - x
            d = torch.stack([F[k * n:(k + 1) * n].abs().max() for k in range(3)]).cpu().numpy()
            if step > 1:
                hist.append(MuIterationRecord(step - 1, float(d[0]), float(d[1]), float(d[2])))
            if not np.all(np.isfinite(d)):
                raise NumericalFailureError("non-finite Newton residual in the finite-mu solve")
            if d[0] < params.xi and d[1] < params.xi and d[2] < params.xi:
                x = gx.clone()
                converged = True
                break
            if step > max_newton:
                break
            xnorm = dot(x, x) ** 0.5

            def jv(v):
                nv = dot(v, v) ** 0.5
                if nv == 0.0:
                    return torch.zeros_like(v)
                h = fd_eps * (1.0 + xnorm) / nv
                return (g(x + h * v, gp) - gx) / h - v

            rtol = min(0.1, max(1e-4, float(d.max())))
            dx, its = _gmres_real(jv, -F, rtol, restart, max_restarts, dot)
            report.steps.append((step, float(d[0]), float(d[1]), float(d[2]), its))
            # backtracking on |F|_2: halve the step while the residual grows
            fn = dot(F, F)
            lam = 1.0
            for _ls in range(line_search):
                g(x + lam * dx, gp)
                Ft = gp - (x + lam * dx)
                if dot(Ft, Ft) < fn:
                    break
                lam *= 0.5
            x = x + lam * dx
        report.sweeps = sweeps[0]
    finally:
        if own:
            sw.close()
    xs = x.cpu().numpy()
    A, B, C = (xs[k * n:(k + 1) * n].reshape(shape).copy() for k in range(3))
    sol = MuSolution(A=A, B=B, C=C, iterations=len(hist) - 1, converged=converged, history=hist, grid=grid,
                     params=params)
    return sol, report


def interp_mu(grid: MuGrid, F, params: MuParams | None = None, device: int = 0) -> np.ndarray:
    """The sweep's complex 2-D interpolation of F at every internal node."""
    params = MuParams() if params is None else params
    with MuSweeper(grid, params, device) as sw:
        return sw.interp(F)

