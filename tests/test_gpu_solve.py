"""GPU parity of the on-device successive-approximation loop (solve).

North-star bar: converged A, B within 1e-9 relative (hybrid measure, SURVEY
§8c) of the reference's own CPU solve, and EXACTLY the same iteration count.
"""
import numpy as np
import pytest

import paper_2012_03667_b200 as p
from conftest import golden, golden_grid, hybrid_rel, params_ns

pytestmark = pytest.mark.gpu


def _run(fname, tag, variant):
    z = golden(fname)
    D, om, m0, z1, xi, relax, cap, c = z["params"]
    prm = params_ns(D=D, omega=om, m0=m0, z1=z1, xi=xi, relaxation=relax, max_iterations=int(cap), coeff=c)
    g = golden_grid(tag)
    b0 = z["b0"] if z["b0"].shape == (g.n_ext,) else None
    sol = p.solve(prm, variant, grid=g, probes_log10p=tuple(z["probes_log10p"]), b0=b0)
    return z, sol


def _hist(sol):
    return np.array([[r.iteration, r.max_delta_a, r.max_delta_b, *r.probe_a, *r.probe_b] for r in sol.history])


@pytest.mark.parametrize("vname", ["indexed-gpu-exact", "search-gpu-exact", "indexed-gpu", "indexed-gpu-moments",
                                   "indexed-gpu-pairs"])
def test_solve_default_config(vname):
    z, sol = _run("solve_default.npz", "default", p.VARIANTS[vname])
    assert sol.iterations == int(z["iterations"]) and sol.converged == bool(z["converged"])
    assert hybrid_rel(sol.A, z["A"]) <= 1e-11 and hybrid_rel(sol.B, z["B"]) <= 1e-11
    h = _hist(sol)
    assert h.shape == z["history"].shape
    assert np.isnan(h[0, 1]) and np.isnan(h[0, 2])
    np.testing.assert_allclose(h[1:, 1:3], z["history"][1:, 1:3], rtol=1e-6)
    np.testing.assert_allclose(h[:, 3:], z["history"][:, 3:], rtol=1e-11)


@pytest.mark.parametrize("vname", ["indexed-gpu-exact", "indexed-gpu", "indexed-gpu-moments",
                                   "search-gpu-moments", "indexed-gpu-pairs", "search-gpu-pairs"])
def test_solve_config0_exact_iteration_count(vname):
    """Config 0 (128/128/64, xi=1e-10, b0=0.3): the reference converges in 2923 sweeps."""
    z, sol = _run("solve_c0.npz", "c0", p.VARIANTS[vname])
    assert sol.converged and sol.iterations == int(z["iterations"]) == 2923
    assert hybrid_rel(sol.A, z["A"]) <= 1e-9 and hybrid_rel(sol.B, z["B"]) <= 1e-9
    h = _hist(sol)
    assert h.shape == z["history"].shape


@pytest.mark.parametrize("vname", ["indexed-gpu-exact", "indexed-gpu", "indexed-gpu-moments", "indexed-gpu-pairs"])
def test_solve_config2_first_10_sweeps(vname):
    """Config 2 (1024/1024/256) does not converge in the reference:
    parity = first 10 sweeps + converged=False at the same cap."""
    z, sol = _run("solve_c2k10.npz", "c2", p.VARIANTS[vname])
    assert sol.iterations == 10 and not sol.converged and not bool(z["converged"])
    assert hybrid_rel(sol.A, z["A"]) <= 1e-11 and hybrid_rel(sol.B, z["B"]) <= 1e-11
    np.testing.assert_allclose(_hist(sol)[1:, 1:3], z["history"][1:, 1:3], rtol=1e-6)


@pytest.mark.parametrize("vname", ["indexed-gpu-exact", "indexed-gpu", "indexed-gpu-moments", "indexed-gpu-pairs"])
def test_solve_large_substitute_relaxation(vname):
    """N=M=K=256 at relaxation 0.5: the reference converges in 421 iterations."""
    z, sol = _run("solve_sub256.npz", "sub256", p.VARIANTS[vname])
    assert sol.converged and sol.iterations == int(z["iterations"])
    assert hybrid_rel(sol.A, z["A"]) <= 1e-9 and hybrid_rel(sol.B, z["B"]) <= 1e-9


def test_solve_cap_and_warm_start():
    g = golden_grid("default")
    prm = params_ns(xi=1e-14, max_iterations=3)
    sol = p.solve(prm, p.VARIANTS["indexed-gpu-exact"], grid=g)
    assert sol.iterations == 3 and not sol.converged and len(sol.history) == 4
    # warm start from the 3-iteration state continues the same trajectory
    a, b = np.ones(g.n_ext), np.ones(g.n_ext)
    for _ in range(3):
        a, b = p.iterate_once(g, a, b, prm, p.VARIANTS["indexed-gpu-exact"])
    assert np.array_equal(a, sol.A) and np.array_equal(b, sol.B)


def test_solve_numerical_failure_raises():
    g = golden_grid("small")
    a0 = np.ones(g.n_ext)
    a0[5] = np.inf
    with pytest.raises(p.NumericalFailureError) as ei:
        p.solve(params_ns(xi=1e-3, max_iterations=5), p.VARIANTS["indexed-gpu-exact"], grid=g, a0=a0)
    assert ei.value.iteration == 1 and ei.value.row is not None


@pytest.mark.parametrize("vname", ["indexed-gpu-moments", "indexed-gpu-pairs"])
def test_moments_batch_equals_standalone(vname):
    """Batched solves with the moments / pairs arithmetic (concurrent
    per-solve sweepers) equal the standalone solves bitwise."""
    g = golden_grid("c0")
    v = p.VARIANTS[vname]
    prms = [p.ModelParams(N=128, m_rad=128, m_ang=64, xi=1e-10, max_iterations=5000, D=D) for D in (0.5, 0.6)]
    batch = p.solve_batch(prms, v, grid=g, b0s=[np.full(g.n_ext, 0.3)] * 2)
    for prm, sb in zip(prms, batch):
        s1 = p.solve(prm, v, grid=g, b0=np.full(g.n_ext, 0.3))
        assert sb.iterations == s1.iterations and sb.converged == s1.converged
        assert np.array_equal(sb.A, s1.A) and np.array_equal(sb.B, s1.B)


@pytest.mark.parametrize("arith", [p.Arithmetic.EXACT, p.Arithmetic.FAST, p.Arithmetic.MOMENTS,
                                   p.Arithmetic.PAIRS])
def test_load_resume_status_protocol(arith):
    """dse_solve_load + dse_solve_resume on a fresh sweeper (no sweep/solve
    first): a clean run checks clean, a non-finite state reports the reference
    location, and a following clean load/resume is clean again."""
    import torch

    E = golden("errors.npz")
    g = golden_grid("small")
    name = str(E["names"][0])
    for _ in range(3):  # fresh sweepers, possibly on recycled device memory
        sw = p.GpuSweeper(g, params_ns(), p.InterpStrategy.PRECOMPUTED_INDEX, arith)
        good = (torch.ones(g.n_ext, dtype=torch.float64, device="cuda"),
                torch.full((g.n_ext,), 0.3, dtype=torch.float64, device="cuda"))
        bad = (torch.as_tensor(E[f"{name}__a"], device="cuda"), torch.as_tensor(E[f"{name}__b"], device="cuda"))
        sw.load_device(good[0].data_ptr(), good[1].data_ptr())
        sw.resume(3)
        sw.check()
        sw.load_device(bad[0].data_ptr(), bad[1].data_ptr())
        sw.resume(1)
        with pytest.raises(p.NumericalFailureError) as ei:
            sw.check()
        assert (ei.value.row, ei.value.radial, ei.value.angular) == tuple(int(v) for v in E[f"{name}__loc"])
        sw.load_device(good[0].data_ptr(), good[1].data_ptr())
        sw.resume(2)
        sw.check()
        sw.close()


@pytest.mark.parametrize("tag", ["d050", "d056", "r070"])
@pytest.mark.parametrize("vname", ["indexed-seq", "indexed-gpu", "indexed-gpu-moments", "indexed-gpu-pairs"])
def test_solve_slow_converging_iteration_counts(tag, vname):
    """Config-0 grid at D = 0.50, D = 0.56 and relaxation 0.7 (xi = 1e-10,
    b0 = 0.3): the reference's own iteration counts, exactly, for the
    reference-order arithmetic and for every fast form (the count
    is the most rounding-sensitive observable)."""
    import os
    from conftest import GOLDEN
    fname = f"solve_slow_{tag}.npz"
    if not os.path.exists(os.path.join(GOLDEN, fname)):
        pytest.skip(f"{fname} not generated")
    z, sol = _run(fname, "c0", p.VARIANTS[vname])
    assert sol.converged == bool(z["converged"]) and sol.iterations == int(z["iterations"])
    assert hybrid_rel(sol.A, z["A"]) <= 1e-9 and hybrid_rel(sol.B, z["B"]) <= 1e-9
    assert _hist(sol).shape == z["history"].shape
