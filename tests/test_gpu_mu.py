"""GPU: the finite-mu path (BASELINE configs 3-4) through the C ABI against
the CPU oracle oracle/mu_oracle.py.  Parity is to the self-derived oracle:
there is no reference implementation ("parity unpinned").

Tolerances: interpolation bitwise (same op order); one sweep 1e-11 hybrid
(SURVEY §8c measure; the kernel contracts angular moments per pair, a
different summation order); a converged solve 1e-9 hybrid with the same
iteration count (north_star)."""
import os

import numpy as np
import pytest

import mu_oracle
from conftest import hybrid_rel
from paper_2012_03667_b200 import NumericalFailureError
from paper_2012_03667_b200.finite_mu import MuSweeper, iterate_mu_once, solve_mu, solve_mu_batch
from paper_2012_03667_b200.mu_grid import MuParams, grid_for

pytestmark = pytest.mark.gpu

SMALL = dict(n_s=10, n_4=12, m_s=14, m_4=16, m_ang=6)


def _state(g, seed):
    rng = np.random.default_rng(seed)
    shape = (g.n_s, g.n_4)
    A = 1.0 + 0.8 * rng.random(shape) + 0.1j * rng.standard_normal(shape)
    B = 0.1 + 0.5 * rng.random(shape) + 0.05j * rng.standard_normal(shape)
    C = 1.0 + 0.8 * rng.random(shape) + 0.1j * rng.standard_normal(shape)
    return A, B, C


def _cmp(x, ref):
    return max(hybrid_rel(np.real(x), np.real(ref)), hybrid_rel(np.imag(x), np.imag(ref)))


def test_interp_bitwise():
    p = MuParams(**SMALL)
    g = grid_for(p)
    A, _, _ = _state(g, 1)
    with MuSweeper(g, p) as sw:
        out = sw.interp(A)
    ref = mu_oracle.interp2d(g, A)
    assert np.array_equal(out.view(np.float64), ref.view(np.float64))


@pytest.mark.parametrize("vertex", ["bc", "bc1", "bcb"])
@pytest.mark.parametrize("mu", [0.0, 0.2])
def test_sweep_matches_oracle(vertex, mu):
    p = MuParams(mu=mu, vertex=vertex, **SMALL)
    g = grid_for(p)
    A, B, C = _state(g, 2)
    got = iterate_mu_once(g, A, B, C, p)
    ref = mu_oracle.sweep(g, p, A, B, C)
    for x, r in zip(got, ref):
        assert _cmp(x, r) < 1e-11


def test_sweep_row_sharding_and_grid_size_bitwise():
    p = MuParams(**SMALL)
    g = grid_for(p)
    A, B, C = _state(g, 3)
    with MuSweeper(g, p) as sw:
        full = sw.sweep(A, B, C)
    W = 3
    stitched = [np.zeros_like(full[0]) for _ in range(3)]
    for r in range(W):
        with MuSweeper(g, p, row_start=r, row_stride=W) as sw:
            part = sw.sweep(A, B, C)
        for f in range(3):
            stitched[f].reshape(-1)[r::W] = part[f].reshape(-1)[r::W]
    for f in range(3):
        assert np.array_equal(stitched[f].view(np.float64), full[f].view(np.float64))
    os.environ["DSE_MU_BLOCKS"] = "5"
    try:
        with MuSweeper(g, p) as sw:
            few = sw.sweep(A, B, C)
            few_mo = sw.sweep(A, B, C, MuParams(**{**p.__dict__, "mode": "moments"}))
    finally:
        del os.environ["DSE_MU_BLOCKS"]
    for f in range(3):
        assert np.array_equal(few[f].view(np.float64), full[f].view(np.float64))
        assert np.array_equal(few_mo[f].view(np.float64), full[f].view(np.float64))


@pytest.mark.parametrize("vertex", ["bcb", "bc1"])
def test_solve_matches_oracle_iterations_and_values(vertex):
    p = MuParams(mu=0.2, vertex=vertex, max_iterations=200, **SMALL)
    g = grid_for(p)
    A, B, C, n, conv, hist = mu_oracle.solve(g, p)
    sol = solve_mu(p, g)
    assert conv and sol.converged
    assert sol.iterations == n
    assert _cmp(sol.A, A) < 1e-9 and _cmp(sol.B, B) < 1e-9 and _cmp(sol.C, C) < 1e-9
    assert len(sol.history) == len(hist)
    for rec, h in zip(sol.history[1:], hist[1:]):
        assert rec.n == h[0]
        for got, ref in ((rec.delta_a, h[1]), (rec.delta_b, h[2]), (rec.delta_c, h[3])):
            assert abs(got - ref) <= 1e-6 * ref + 1e-14


def test_cap_is_not_an_error_and_relaxation():
    p = MuParams(mu=0.1, vertex="bc1", max_iterations=3, relaxation=0.7, **SMALL)
    g = grid_for(p)
    A, B, C, n, conv, _ = mu_oracle.solve(g, p)
    sol = solve_mu(p, g)
    assert (sol.iterations, sol.converged) == (n, conv) == (3, False)
    # three sweeps compound the per-sweep 1e-11 bound
    assert _cmp(sol.A, A) < 1e-10 and _cmp(sol.B, B) < 1e-10 and _cmp(sol.C, C) < 1e-10


def test_batch_equals_standalone():
    p = MuParams(vertex="bc1", max_iterations=100, **SMALL)
    g = grid_for(p)
    mus = [0.05, 0.3]
    batch = solve_mu_batch(mus, p, g)
    for m, sol in zip(mus, batch):
        one = solve_mu(MuParams(**{**p.__dict__, "mu": m}), g)
        assert sol.iterations == one.iterations
        assert np.array_equal(sol.A.view(np.float64), one.A.view(np.float64))


def test_failure_location_matches_oracle():
    p = MuParams(**SMALL)
    g = grid_for(p)
    A, B, C = _state(g, 4)
    A[3, 5] = np.nan
    with pytest.raises(mu_oracle.MuNumericalFailure) as ref:
        mu_oracle.sweep(g, p, A, B, C)
    with pytest.raises(NumericalFailureError) as got:
        iterate_mu_once(g, A, B, C, p)
    assert (got.value.row, got.value.radial, got.value.angular) == (ref.value.row, ref.value.radial,
                                                                      ref.value.angular)


def test_stats_count_points():
    p = MuParams(vertex="bc1", max_iterations=2, **SMALL)
    g = grid_for(p)
    with MuSweeper(g, p) as sw:
        sw.solve(p)
        st = sw.stats()
    assert st["nominal_points"] == g.nominal_points
    assert 0 < st["evaluated_points"] <= st["nominal_points"]


def test_sharded_solve_world1_equals_solve():
    """solve_mu_sharded (sweep+pack | gather | assemble+blend+deltas per
    iteration) at world 1 is bitwise the on-device single-GPU solve."""
    import torch

    from paper_2012_03667_b200.finite_mu import solve_mu_sharded
    p = MuParams(mu=0.2, vertex="bcb", max_iterations=200, relaxation=0.8, **SMALL)
    g = grid_for(p)
    ref = solve_mu(p, g)

    def copy_gather(out, buf):
        out[0].copy_(buf)

    got = solve_mu_sharded(p, g, rank=0, world=1, device=0, gather=copy_gather)
    assert got.iterations == ref.iterations and got.converged == ref.converged
    for x, y in ((got.A, ref.A), (got.B, ref.B), (got.C, ref.C)):
        assert np.array_equal(x.view(np.float64), y.view(np.float64))
    assert [(r.n, r.delta_a, r.delta_b, r.delta_c) for r in got.history[1:]] == \
        [(r.n, r.delta_a, r.delta_b, r.delta_c) for r in ref.history[1:]]
    torch.cuda.synchronize()


def test_sharded_iteration_world3_emulated():
    """Three row-sharded sweepers (ranks run one after another on one GPU,
    nothing waits on anything) + the stacked send buffers reproduce one
    single-GPU sweep bitwise on every rank."""
    import ctypes
    import math

    import torch

    from paper_2012_03667_b200 import _native as nat
    from paper_2012_03667_b200.distributed import device_view
    from paper_2012_03667_b200.finite_mu import _c_params
    p = MuParams(**SMALL)
    g = grid_for(p)
    A, B, C = _state(g, 6)
    ref = iterate_mu_once(g, A, B, C, p)
    W = 3
    per = math.ceil(g.n_ext / W)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev).cuda_stream
    lib = nat.load()
    cp = _c_params(p)
    tens = [torch.from_numpy(np.ascontiguousarray(x.reshape(-1))).to(dev) for x in (A, B, C)]
    sws = [MuSweeper(g, p, row_start=r, row_stride=W) for r in range(W)]
    sends = [torch.zeros((3, per, 2), dtype=torch.float64, device=dev) for _ in range(W)]
    err = nat.DseErr()
    for sw, send in zip(sws, sends):
        nat.raise_for(lib.dse_mu_solve_load(sw.handle, *[t.data_ptr() for t in tens], st, ctypes.byref(err)), err)
        nat.raise_for(lib.dse_mu_sharded_sweep_pack(sw.handle, ctypes.byref(cp), send.data_ptr(), per, st,
                                                    ctypes.byref(err)), err)
    recv = torch.stack(sends)
    delta = torch.zeros(3, dtype=torch.float64, device=dev)
    for sw in sws:
        nat.raise_for(lib.dse_mu_sharded_assemble(sw.handle, recv.data_ptr(), W, per, 1.0, delta.data_ptr(), st,
                                                  ctypes.byref(err)), err)
        px = ctypes.c_void_p()
        nat.raise_for(lib.dse_mu_sweeper_state(sw.handle, ctypes.byref(px)), nat.DseErr())
        full = device_view(px.value, 6 * g.n_ext, dev).cpu().numpy().view(np.complex128).reshape(3, g.n_s, g.n_4)
        for f in range(3):
            assert np.array_equal(full[f].view(np.float64), ref[f].view(np.float64))
        d = delta.cpu().numpy()
        # |new - old| is CUDA's hypot on the device, numpy's here: the two
        # libraries may differ by an ulp (the state itself is compared bitwise)
        np.testing.assert_allclose(d, [np.max(np.abs(r - x)) for r, x in zip(ref, (A, B, C))], rtol=4.5e-16, atol=0)
    for sw in sws:
        sw.close()


@pytest.mark.parametrize("vertex", ["bcb", "bc1", "bc"])
def test_moments_mode_bitwise_equals_direct(vertex):
    """Moments mode (angular moments built once per grid, contracted every
    iteration) is the direct sweep's own arithmetic: bitwise equal, for one
    sweep and for a whole solve (iterations, state, history)."""
    A, B, C = None, None, None
    p = MuParams(mu=0.2, vertex=vertex, max_iterations=60, **SMALL)
    pm = MuParams(**{**p.__dict__, "mode": "moments"})
    g = grid_for(p)
    A, B, C = _state(g, 7)
    d = iterate_mu_once(g, A, B, C, p)
    m = iterate_mu_once(g, A, B, C, pm)
    for x, y in zip(d, m):
        assert np.array_equal(x.view(np.float64), y.view(np.float64))
    if vertex == "bc":
        return  # diverges under successive approximation
    sd, sm = solve_mu(p, g), solve_mu(pm, g)
    assert (sd.iterations, sd.converged) == (sm.iterations, sm.converged)
    for x, y in ((sd.A, sm.A), (sd.B, sm.B), (sd.C, sm.C)):
        assert np.array_equal(x.view(np.float64), y.view(np.float64))


def test_moments_mode_reuse_across_mu_and_failure():
    """One sweeper serves several mu values from one moment table (config 4),
    each bitwise equal to its direct solve; a non-finite state fails with the
    reference's location."""
    p = MuParams(vertex="bcb", max_iterations=80, mode="moments", **SMALL)
    g = grid_for(p)
    with MuSweeper(g, p) as sw:
        for mu in (0.05, 0.3):
            pm = MuParams(**{**p.__dict__, "mu": mu})
            got = sw.solve(pm)
            ref = solve_mu(MuParams(**{**pm.__dict__, "mode": "direct"}), g)
            assert got.iterations == ref.iterations
            assert np.array_equal(got.A.view(np.float64), ref.A.view(np.float64))
        A, B, C = _state(g, 4)
        A[3, 5] = np.nan
        with pytest.raises(mu_oracle.MuNumericalFailure) as ref_exc:
            mu_oracle.sweep(g, p, A, B, C)
        with pytest.raises(NumericalFailureError) as got_exc:
            sw.sweep(A, B, C)
        assert (got_exc.value.row, got_exc.value.radial, got_exc.value.angular) == \
            (ref_exc.value.row, ref_exc.value.radial, ref_exc.value.angular)


@pytest.mark.parametrize("dims", [dict(n_s=2, n_4=2, m_s=2, m_4=2, m_ang=1), dict(n_s=3, n_4=5, m_s=7, m_4=4, m_ang=3)])
def test_minimum_and_ragged_grids(dims):
    p = MuParams(mu=0.15, **dims)
    g = grid_for(p)
    A, B, C = _state(g, 8)
    got = iterate_mu_once(g, A, B, C, p)
    ref = mu_oracle.sweep(g, p, A, B, C)
    for x, r in zip(got, ref):
        assert _cmp(x, r) < 1e-11


@pytest.mark.parametrize("mode", ["direct", "moments"])
def test_anderson_reaches_the_same_fixed_point_faster(mode):
    from paper_2012_03667_b200.finite_mu import solve_mu_anderson
    p = MuParams(mu=0.2, vertex="bcb", max_iterations=300, xi=1e-11, mode=mode, **SMALL)
    g = grid_for(p)
    sa = solve_mu(p, g)
    aa = solve_mu_anderson(p, g, depth=8)
    assert sa.converged and aa.converged and aa.iterations < sa.iterations
    for x, y in ((aa.A, sa.A), (aa.B, sa.B), (aa.C, sa.C)):
        assert np.max(np.abs(x - y)) <= 1e-9 * np.max(np.abs(y))


@pytest.mark.parametrize("S", [2, 4])
def test_batched_sweep_bitwise_equals_single(S):
    """dse_mu_batch_sweep: each solve's sweep is bitwise its standalone
    moments-mode sweep (own mu, D and state; shared moment table)."""
    import torch
    p = MuParams(vertex="bcb", mode="moments", **SMALL)
    g = grid_for(p)
    plist = [MuParams(**{**p.__dict__, "mu": 0.05 + 0.1 * s, "D": 0.5 + 0.02 * s}) for s in range(S)]
    states = [_state(g, 20 + s) for s in range(S)]
    dev = torch.device("cuda", 0)
    x = torch.stack([torch.from_numpy(np.concatenate([v.reshape(-1) for v in st])) for st in states]).to(dev)
    y = torch.empty_like(x)
    with MuSweeper(g, p) as sw:
        failed = sw.batch_sweep(x, y, plist)
        assert failed == [-1] * S
        for s in range(S):
            ref = sw.sweep(*states[s], plist[s])
            got = y[s].cpu().numpy()
            for f in range(3):
                part = got[f * g.n_ext:(f + 1) * g.n_ext].reshape(g.n_s, g.n_4)
                assert np.array_equal(part.view(np.float64), ref[f].view(np.float64))


def test_batched_anderson_matches_single_anderson():
    from paper_2012_03667_b200.finite_mu import solve_mu_anderson, solve_mu_batch_anderson
    p = MuParams(vertex="bcb", mode="moments", max_iterations=200, **SMALL)
    g = grid_for(p)
    mus = [0.05, 0.15, 0.25]
    batch = solve_mu_batch_anderson(mus, p, g, batch=4)
    for m, sol in zip(mus, batch):
        one = solve_mu_anderson(MuParams(**{**p.__dict__, "mu": m}), g)
        assert sol.converged == one.converged and sol.iterations == one.iterations
        assert np.max(np.abs(sol.A - one.A)) <= 1e-12 * np.max(np.abs(one.A))


@pytest.mark.parametrize("vertex", ["bcb", "bc1"])
def test_narrow_interaction_skip_windows(vertex):
    """A narrow interaction (omega = 0.05) leaves most pairs exactly zero:
    rows whose skip windows are short or empty, and pair counts that do not
    fill a CTA's 256 threads.  Direct mode matches the oracle, and moments mode
    (cp.async-staged contraction) is bitwise the direct sweep."""
    p = MuParams(mu=0.2, omega=0.05, vertex=vertex, **SMALL)
    pm = MuParams(**{**p.__dict__, "mode": "moments"})
    g = grid_for(p)
    A, B, C = _state(g, 11)
    d = iterate_mu_once(g, A, B, C, p)
    m = iterate_mu_once(g, A, B, C, pm)
    ref = mu_oracle.sweep(g, p, A, B, C)
    for x, y, r in zip(d, m, ref):
        assert np.array_equal(x.view(np.float64), y.view(np.float64))
        assert _cmp(x, r) < 1e-11
    with MuSweeper(g, pm) as sw:
        sw.solve(MuParams(**{**pm.__dict__, "max_iterations": 1}))
        st = sw.stats()
    assert 0 < st["evaluated_points"] < st["nominal_points"] // 4, st


def test_device_anderson_kernels_match_numpy():
    """dse_mu_aa_residual / dse_mu_aa_update (the device Anderson state) against
    a numpy restatement of the same step on random data: residual maxima
    bitwise, Gram columns and right-hand sides to rounding, the ring order of
    the columns, and the update x + beta f - (dX + beta dF) gamma."""
    import torch
    from paper_2012_03667_b200.finite_mu import _DeviceAnderson, _aa_solve
    rng = np.random.default_rng(5)
    S, n, depth, beta = 2, 50, 3, 0.7
    dev = torch.device("cuda", 0)
    aa = _DeviceAnderson(S, n, depth, beta, dev, 0)
    x = torch.from_numpy(rng.standard_normal((S, 3 * n)) + 1j * rng.standard_normal((S, 3 * n))).to(dev)
    X, F = [], []
    for step in range(6):
        gx_h = x.cpu().numpy() + 0.5 ** step * (rng.standard_normal((S, 3 * n)) + 1j * rng.standard_normal((S, 3 * n)))
        gx = torch.from_numpy(gx_h).to(dev)
        xh = x.cpu().numpy()
        f = gx_h - xh
        d = aa.residual(x, gx)
        ref_d = np.abs(f).reshape(S, 3, n).max(axis=2)
        assert np.allclose(d, ref_d, rtol=1e-15, atol=0)
        X.append(xh)
        F.append(f)
        X, F = X[-(depth + 1):], F[-(depth + 1):]
        L = len(F) - 1
        assert len(aa.cols) == L
        if L:
            dF = np.stack([F[k + 1] - F[k] for k in range(L)], axis=2)   # oldest first
            dX = np.stack([X[k + 1] - X[k] for k in range(L)], axis=2)
            G = np.einsum("sik,sil->skl", dF.conj(), dF)
            rhs = np.einsum("sik,si->sk", dF.conj(), f)
            got_G = aa.G[:, aa.cols][:, :, aa.cols]
            assert np.max(np.abs(got_G - G)) <= 1e-12 * np.max(np.abs(G))
            assert np.max(np.abs(aa.rhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))
            gamma = _aa_solve(got_G, aa.rhs)
            ref_x = xh + beta * f - np.einsum("sik,sk->si", dX + beta * dF, gamma)
        else:
            ref_x = xh + beta * f
        aa.update(x)
        torch.cuda.synchronize()
        got = x.cpu().numpy()
        assert np.max(np.abs(got - ref_x)) <= 1e-12 * np.max(np.abs(ref_x))


@pytest.mark.parametrize("count,batch,cap", [(3, 4, 120), (5, 4, 120), (2, 2, 120), (5, 4, 7), (3, 2, 9)])
def test_batched_successive_approximation_equals_standalone(count, batch, cap):
    """solve_mu_batch_sa (config 4's parity-equivalent path, one cooperative
    launch per group): each mu value's iterations, history and state are
    bitwise its standalone solve_mu; groups of 4 and 2, a padded remainder,
    and a cap below the convergence point (converged False, the capped
    state)."""
    from paper_2012_03667_b200.finite_mu import solve_mu_batch_sa
    p = MuParams(vertex="bcb", max_iterations=cap, **SMALL)
    g = grid_for(p)
    mus = [0.02 + 0.37 * k / count for k in range(count)]
    batch = solve_mu_batch_sa(mus, p, g, batch=batch)
    assert len(batch) == count
    for m, sol in zip(mus, batch):
        one = solve_mu(MuParams(**{**p.__dict__, "mu": m}), g)
        assert sol.converged == one.converged and sol.iterations == one.iterations
        for x, y in ((sol.A, one.A), (sol.B, one.B), (sol.C, one.C)):
            assert np.array_equal(x.view(np.float64), y.view(np.float64))
        h1 = [(r.n, r.delta_a, r.delta_b, r.delta_c) for r in one.history]
        h2 = [(r.n, r.delta_a, r.delta_b, r.delta_c) for r in sol.history]
        assert np.array_equal(np.array(h1[1:]), np.array(h2[1:]))


def test_batch_sharded_world1_equals_standalone():
    """solve_mu_batch_sharded (config 4's public multi-GPU API) at world 1:
    the batched successive approximation path, every record bitwise the
    standalone solve_mu."""
    from paper_2012_03667_b200.finite_mu import solve_mu_batch_sharded
    p = MuParams(vertex="bcb", max_iterations=120, **SMALL)
    g = grid_for(p)
    mus = [0.05, 0.15, 0.25, 0.35, 0.3]
    recs = solve_mu_batch_sharded(mus, p, g, rank=0, world=1)
    for m, (mu_r, its, conv, A, B, C) in zip(mus, recs):
        one = solve_mu(MuParams(**{**p.__dict__, "mu": m}), g)
        assert mu_r == m and its == one.iterations and conv == one.converged
        for x, y in ((A, one.A), (B, one.B), (C, one.C)):
            assert np.array_equal(x.view(np.float64), y.view(np.float64))


@pytest.mark.parametrize("mu", [0.0, 0.2])
def test_newton_solves_full_bc_vertex_on_small_grids(mu):
    """The full in-medium Ball-Chiu vertex diverges under successive
    approximation; solve_mu_newton (Newton-Krylov on g(x) - x, device
    sweeps) converges it on small grids, and the result is a fixed point of
    the ORACLE's map: max|g_oracle(x) - x| within the stop tolerance
    (conditioning-independent check of the GPU solution)."""
    from paper_2012_03667_b200.finite_mu import solve_mu_newton
    p = MuParams(vertex="bc", mu=mu, xi=1e-10, n_s=12, n_4=12, m_s=16, m_4=16, m_ang=8)
    g = grid_for(p)
    sol, rep = solve_mu_newton(p, g)
    assert sol.converged and sol.iterations <= 10 and rep.start_iterations > 0
    out = mu_oracle.sweep_rows_c(g, p, sol.A, sol.B, sol.C, np.arange(g.n_ext))
    for c, F in enumerate((sol.A, sol.B, sol.C)):
        assert np.max(np.abs(out[:, c] - F.reshape(-1))) < 1e-9
    # successive approximation does not converge on the same problem (it
    # runs to the cap or overflows into a numerical failure)
    try:
        sa = solve_mu(MuParams(**{**p.__dict__, "max_iterations": 300}), g)
        assert not sa.converged
    except NumericalFailureError:
        pass


def test_newton_reaches_the_successive_approximation_fixed_point():
    """On the convergent 'bcb' vertex, Newton-Krylov started (start=None)
    from the 10th successive-approximation iterate lands on solve_mu's fixed
    point.  (From the raw initial guess A = C = 1, B = 0.3 it can land on a
    different solution of the same equations: the gap equation has several.)"""
    from paper_2012_03667_b200.finite_mu import solve_mu_newton
    p = MuParams(vertex="bcb", mu=0.2, xi=1e-11, max_iterations=300, **SMALL)
    g = grid_for(p)
    sa = solve_mu(p, g)
    s10 = solve_mu(MuParams(**{**p.__dict__, "max_iterations": 10}), g)
    nk, rep = solve_mu_newton(p, g, s10.A, s10.B, s10.C, start=None)
    assert sa.converged and nk.converged and rep.start_iterations == 0 and rep.sweeps > 0
    for x, y in ((nk.A, sa.A), (nk.B, sa.B), (nk.C, sa.C)):
        assert np.max(np.abs(x - y)) <= 1e-9 * np.max(np.abs(y))
