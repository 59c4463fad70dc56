"""The reference's own hot-path test expectations, run against the drop-in.

Each test restates (in this repo's words, not copied) one check of the
reference's suite -- /root/reference/pkg/tests/test_solver.py:24-143,
test_interpolation.py:19-109 and test_acceptance.py:60-111, 130-155, 209-232
(the CPU-performance ordering of criterion 5 excluded) -- with caller code
written exactly as a `dsegap` user writes it: the reference's variant names
(`indexed-seq`, `indexed-par`, ...), `with_threads(C)`, `SOLVER_THREADS`,
`_eval_rows`.  Nothing here reads /root/reference: the brute-force
comparison of test_solver.py:83-91 goes to the C restatement in oracle/
(the checker), and the grids are built by the drop-in itself.
"""
import math
import os

import numpy as np
import pytest

import paper_2012_03667_b200 as p
from paper_2012_03667_b200.solver import _eval_rows

pytestmark = pytest.mark.gpu

SMALL = p.ModelParams(N=24, m_rad=20, m_ang=8, p2_min=1e-5, p2_max=1e3)
CORES = os.cpu_count() or 1


def _with(params, **kw):
    return p.ModelParams(**{**vars(params), **kw})


@pytest.fixture(scope="module")
def small_grid():
    return p.build_grid(SMALL.N, SMALL.m_rad, SMALL.m_ang, SMALL.p2_min, SMALL.p2_max)


# ---- test_solver.py ---------------------------------------------------------

def test_free_theory_fixed_point(small_grid):  # test_solver.py:24-29
    sol = p.solve(_with(SMALL, D=0.0, m0=0.005), p.VARIANTS["indexed-seq"], grid=small_grid)
    assert sol.converged and sol.iterations <= 2
    assert np.all(sol.A == 1.0) and np.all(sol.B == 0.005)


def test_chiral_b_stays_exactly_zero(small_grid):  # test_solver.py:32-37
    prm = _with(SMALL, m0=0.0, max_iterations=10, xi=1e-30)
    sol = p.solve(prm, p.VARIANTS["indexed-seq"], grid=small_grid, b0=np.zeros(small_grid.n_ext))
    assert not sol.converged and sol.iterations == 10
    assert np.all(sol.B == 0.0)


def test_reference_variants_bitwise_equal(small_grid):  # test_solver.py:40-48
    sols = {name: p.solve(SMALL, p.VARIANTS[name].with_threads(2), grid=small_grid)
            for name in ("search-seq", "indexed-seq", "search-par", "indexed-par")}
    first = sols["search-seq"]
    assert first.converged
    for name, sol in sols.items():
        assert sol.iterations == first.iterations, name
        assert np.array_equal(sol.A, first.A) and np.array_equal(sol.B, first.B), name


def test_rows_in_any_order(small_grid):  # test_solver.py:51-64
    rng = np.random.default_rng(2)
    a = 1.0 + 0.1 * rng.random(small_grid.n_ext)
    b = 0.5 + 0.1 * rng.random(small_grid.n_ext)
    fa, fb = p.iterate_once(small_grid, a, b, SMALL, p.VARIANTS["indexed-seq"])
    strat = p.VARIANTS["indexed-seq"].interp
    ga, gb = np.empty_like(fa), np.empty_like(fb)
    for i in rng.permutation(small_grid.n_ext):
        ra, rb = _eval_rows(small_grid, SMALL, strat, a, b, int(i), int(i) + 1)
        ga[i], gb[i] = ra[0], rb[0]
    assert np.array_equal(ga, fa) and np.array_equal(gb, fb)
    # a chunk, as a reference worker evaluates it (solver.py:141-145)
    ca, cb = _eval_rows(small_grid, SMALL, strat, a, b, 5, 17)
    assert np.array_equal(ca, fa[5:17]) and np.array_equal(cb, fb[5:17])


def test_worker_count_changes_no_bit(small_grid):  # test_solver.py:67-71
    one = p.solve(SMALL, p.VARIANTS["indexed-par"].with_threads(1), grid=small_grid)
    for threads in (2, 3, CORES):
        sol = p.solve(SMALL, p.VARIANTS["indexed-par"].with_threads(threads), grid=small_grid)
        assert np.array_equal(sol.A, one.A) and np.array_equal(sol.B, one.B)


def test_solver_threads_env(small_grid, monkeypatch):  # test_solver.py:74-80
    monkeypatch.setenv("SOLVER_THREADS", "4")
    assert p.resolve_threads(p.VARIANTS["indexed-par"]) == 4
    assert p.resolve_threads(p.VARIANTS["indexed-par"].with_threads(2)) == 2
    # the env var names host workers: a solve under it stays a one-GPU solve
    sol = p.solve(SMALL, p.VARIANTS["indexed-par"], grid=small_grid)
    monkeypatch.delenv("SOLVER_THREADS")
    assert p.resolve_threads(p.VARIANTS["indexed-par"]) >= 1
    ref = p.solve(SMALL, p.VARIANTS["indexed-par"], grid=small_grid)
    assert np.array_equal(sol.A, ref.A) and np.array_equal(sol.B, ref.B)


def test_iterate_once_vs_brute_force(small_grid):  # test_solver.py:83-91
    import oracle
    rng = np.random.default_rng(4)
    a = 1.0 + 0.2 * rng.random(small_grid.n_ext)
    b = 0.8 + 0.2 * rng.random(small_grid.n_ext)
    ga, gb = p.iterate_once(small_grid, a, b, SMALL, p.VARIANTS["search-seq"])
    wa, wb = oracle.sweep(small_grid, a, b, SMALL, strategy=0)
    np.testing.assert_allclose(ga, wa, rtol=1e-11)
    np.testing.assert_allclose(gb, wb, rtol=1e-11)


def test_history_rows(small_grid):  # test_solver.py:94-104
    sol = p.solve(SMALL, p.VARIANTS["indexed-seq"], grid=small_grid)
    assert sol.converged and len(sol.history) == sol.iterations + 1
    h0, last = sol.history[0], sol.history[-1]
    assert h0.iteration == 0 and math.isnan(h0.max_delta_a)
    assert last.max_delta_a < SMALL.xi and last.max_delta_b < SMALL.xi
    assert h0.probe_a == pytest.approx((1.0, 1.0)) and h0.probe_b == pytest.approx((1.0, 1.0))


def test_uv_end_is_free(small_grid):  # test_solver.py:107-111
    sol = p.solve(SMALL, p.VARIANTS["indexed-seq"], grid=small_grid)
    assert abs(sol.A[-1] - 1.0) < 1e-3 and abs(sol.B[-1] - SMALL.m0) < 1e-3


def test_current_mass_in_the_uv(small_grid):  # test_solver.py:114-118
    sol = p.solve(_with(SMALL, m0=0.12), p.VARIANTS["indexed-seq"], grid=small_grid)
    assert sol.converged and sol.B[-1] == pytest.approx(0.12, abs=1e-3) and sol.B[0] > 0.12


def test_cap_is_not_an_error(small_grid):  # test_solver.py:121-125
    sol = p.solve(_with(SMALL, max_iterations=2), p.VARIANTS["indexed-seq"], grid=small_grid)
    assert not sol.converged and sol.iterations == 2
    assert np.all(np.isfinite(sol.A)) and np.all(np.isfinite(sol.B))


def test_under_relaxation_same_fixed_point(small_grid):  # test_solver.py:128-134
    plain = p.solve(SMALL, p.VARIANTS["indexed-seq"], grid=small_grid)
    damped = p.solve(_with(SMALL, relaxation=0.7, xi=1e-6), p.VARIANTS["indexed-seq"], grid=small_grid)
    assert damped.converged
    assert np.max(np.abs(damped.A - plain.A)) < 20 * SMALL.xi
    assert np.max(np.abs(damped.B - plain.B)) < 20 * SMALL.xi


def test_failure_location(small_grid):  # test_solver.py:137-143
    with pytest.raises(p.NumericalFailureError) as exc:
        p.iterate_once(small_grid, np.ones(small_grid.n_ext), np.ones(small_grid.n_ext),
                       _with(SMALL, D=1e308), p.VARIANTS["indexed-seq"])
    assert exc.value.row is not None


def test_eval_rows_failure_only_for_own_rows(small_grid):
    """_eval_rows raises only for a failing row inside its range, like a
    reference worker that evaluates just its chunk.  At D = 1e305 the sums of
    rows 0 and 1 overflow (1/p2 is largest there) and rows 2.. stay finite
    (checked with the oracle)."""
    import oracle
    n = small_grid.n_ext
    prm = _with(SMALL, D=1e305)
    one = np.ones(n)
    strat = p.VARIANTS["indexed-seq"].interp
    with pytest.raises(p.NumericalFailureError) as exc:
        p.iterate_once(small_grid, one, one, prm, p.VARIANTS["indexed-seq"])
    assert exc.value.row == 0
    ra, rb = _eval_rows(small_grid, prm, strat, one, one, 2, n)
    wa, wb = oracle.sweep(small_grid, one, one, prm, strategy=1, rows=(2, n))
    np.testing.assert_allclose(ra, wa, rtol=1e-13)
    np.testing.assert_allclose(rb, wb, rtol=1e-13)
    with pytest.raises(p.NumericalFailureError) as exc2:
        _eval_rows(small_grid, prm, strat, one, one, 1, 5)
    assert exc2.value.row == 1


def test_successive_approximation_zero_step():  # test_solver.py:146-150
    state, n, ok = p.successive_approximation(lambda s: s, (np.ones(3), np.zeros(2)), tol=1e-12, cap=5)
    assert ok and n == 1 and np.all(state[0] == 1.0)


# ---- test_interpolation.py --------------------------------------------------

KN, KV = [1.0, 2.0, 3.0], [10.0, 20.0, 30.0]


def test_interp_known_answers():  # test_interpolation.py:19-35
    assert p.interp_search(KN, KV, 2.5) == 25.0
    assert p.interp_search(KN, KV, 3.7) == 30.0
    assert p.interp_search(KN, KV, 0.2) == 10.0
    for x, v in zip(KN, KV):
        assert p.interp_search(KN, KV, x) == v


def test_interp_rejects_bad_tables():  # test_interpolation.py:38-45
    for x, v, q in (([1.0, 2.0], [1.0], 1.5), ([2.0, 1.0], [1.0, 2.0], 1.5), ([1.0], [1.0], 1.0)):
        with pytest.raises(p.ParameterError):
            p.interp_search(x, v, q)


def test_indexed_equals_search_on_random_grids():  # test_interpolation.py:48-63
    rng = np.random.default_rng(17)
    for _ in range(300):
        n, m = int(rng.integers(2, 40)), int(rng.integers(2, 40))
        g = p.build_grid(n, m, 1, 10.0 ** rng.uniform(-6, -2), 10.0 ** rng.uniform(1, 4))
        vals = rng.normal(size=n)
        many = p.interp_indexed_many(g, vals)
        srch = p.interp_search_many(g.p2_ext, vals, g.q2_int)
        assert np.array_equal(many, srch)
        for j in (0, g.m_rad // 2, g.m_rad - 1):
            assert p.interp_indexed(g, vals, j) == p.interp_search(g.p2_ext, vals, g.q2_int[j]) == many[j]


def test_indexed_does_no_comparisons():  # test_interpolation.py:66-78
    g = p.build_grid(20, 15, 1, 1e-4, 1e3)
    vals = np.linspace(0.0, 1.0, 20)
    ctr = p.ComparisonCounter()
    for j in range(g.m_rad):
        p.interp_search(g.p2_ext, vals, g.q2_int[j], counter=ctr)
    assert ctr.count >= 2 * g.m_rad
    before = ctr.count
    for j in range(g.m_rad):
        p.interp_indexed(g, vals, j)
    assert ctr.count == before


def test_no_overshoot():  # test_interpolation.py:81-92
    rng = np.random.default_rng(23)
    x = np.sort(rng.uniform(0.0, 10.0, size=12)) + np.arange(12) * 1e-6
    v = rng.normal(size=12)
    q = rng.uniform(x[0], x[-1], size=300)
    out = p.interp_search_many(x, v, q)
    i = np.minimum(np.searchsorted(x, q, side="right") - 1, 10)
    lo, hi = np.minimum(v[i], v[i + 1]), np.maximum(v[i], v[i + 1])
    assert np.all(lo - 1e-12 <= out) and np.all(out <= hi + 1e-12)


def test_constants_and_lines():  # test_interpolation.py:95-104
    g = p.build_grid(25, 18, 1, 1e-3, 1e3)
    assert np.all(p.interp_indexed_many(g, np.full(25, 4.25)) == 4.25)
    got = p.interp_indexed_many(g, 0.75 * g.p2_ext - 2.0)
    inside = g.bracket_idx < g.n_ext - 1
    np.testing.assert_allclose(got[inside], (0.75 * g.q2_int - 2.0)[inside], rtol=1e-12)


def test_indexed_rejects_bad_arguments():  # test_interpolation.py:107-114
    g = p.build_grid(10, 6, 1, 1e-2, 1e2)
    for vals, j in ((np.ones(9), 0), (np.ones(10), 6), (np.ones(10), -1)):
        with pytest.raises(p.ParameterError):
            p.interp_indexed(g, vals, j)


# ---- test_acceptance.py -----------------------------------------------------

@pytest.fixture(scope="module")
def default_runs():
    prm = p.ModelParams()
    g = p.build_grid(prm.N, prm.m_rad, prm.m_ang, prm.p2_min, prm.p2_max)
    runs = {name: p.solve(prm, p.VARIANTS[name].with_threads(CORES if name.endswith("par") else None), grid=g)
            for name in ("search-seq", "indexed-seq", "search-par", "indexed-par")}
    return prm, g, runs


def test_acceptance_variant_equivalence(default_runs):  # test_acceptance.py:60-74
    _, _, runs = default_runs
    first = runs["search-seq"]
    assert first.converged
    for sol in runs.values():
        assert sol.iterations == first.iterations
        assert np.array_equal(sol.A, first.A) and np.array_equal(sol.B, first.B)


def test_acceptance_interpolation_equivalence():  # test_acceptance.py:77-92
    rng = np.random.default_rng(101)
    for _ in range(200):
        n, m = int(rng.integers(2, 32)), int(rng.integers(2, 32))
        g = p.build_grid(n, m, 1, 10.0 ** rng.uniform(-6, -1), 10.0 ** rng.uniform(0.5, 4))
        vals = rng.normal(size=n)
        assert np.array_equal(p.interp_indexed_many(g, vals), p.interp_search_many(g.p2_ext, vals, g.q2_int))


def test_acceptance_parallel_determinism(default_runs, tmp_path):  # test_acceptance.py:95-105
    from paper_2012_03667_b200.cli import write_solution_csv
    prm, g, _ = default_runs
    blobs = []
    for threads in sorted({1, 2, CORES}):
        sol = p.solve(prm, p.VARIANTS["indexed-par"].with_threads(threads), grid=g)
        path = tmp_path / f"sol_{threads}.csv"
        write_solution_csv(str(path), sol)
        blobs.append(path.read_bytes())
    assert all(x == blobs[0] for x in blobs)


def test_acceptance_convergence_iterations(default_runs):  # test_acceptance.py:108-111
    sol = default_runs[2]["search-seq"]
    assert sol.converged and 5 <= sol.iterations <= 30


def test_acceptance_free_and_chiral():  # test_acceptance.py:130-146
    sol = p.solve(p.ModelParams(D=0.0, m0=0.005, N=64, m_rad=48, m_ang=8), p.VARIANTS["indexed-seq"])
    assert sol.converged and sol.iterations <= 2
    assert np.max(np.abs(sol.A - 1.0)) <= 1e-14 and np.max(np.abs(sol.B - 0.005)) <= 1e-14
    prm = p.ModelParams(N=64, m_rad=48, m_ang=8, m0=0.0, xi=1e-30, max_iterations=10)
    g = p.build_grid(prm.N, prm.m_rad, prm.m_ang, prm.p2_min, prm.p2_max)
    sol = p.solve(prm, p.VARIANTS["indexed-seq"], grid=g, b0=np.zeros(g.n_ext))
    assert sol.iterations == 10 and np.all(sol.B == 0.0)


def test_acceptance_uv_and_mass_generation(default_runs):  # test_acceptance.py:149-173
    import oracle
    prm, _, runs = default_runs
    sol = runs["search-seq"]
    assert sol.converged and abs(sol.A[-1] - 1.0) < 1e-3 and abs(sol.B[-1] - prm.m0) < 1e-3
    assert sol.B[0] > 10.0 * prm.xi
    coarse = p.ModelParams(N=32, m_rad=32, m_ang=8, xi=1e-6)
    cg = p.build_grid(coarse.N, coarse.m_rad, coarse.m_ang, coarse.p2_min, coarse.p2_max)
    cs = p.solve(coarse, p.VARIANTS["indexed-seq"], grid=cg)
    ra, rb = oracle.sweep(cg, cs.A, cs.B, coarse, strategy=1)
    assert cs.converged and max(np.max(np.abs(cs.A - ra)), np.max(np.abs(cs.B - rb))) < 1e-3


def test_acceptance_history_csv(default_runs, tmp_path):  # test_acceptance.py:209-232
    from paper_2012_03667_b200.cli import write_history_csv
    prm, _, runs = default_runs
    sol = runs["search-seq"]
    path = tmp_path / "hist.csv"
    write_history_csv(str(path), sol)
    lines = path.read_text().strip().splitlines()
    head = lines[0].split(",")
    assert head[:3] == ["iteration", "max_dA", "max_dB"]
    for col in ("A(logp=-2.5)", "B(logp=-2.5)", "A(logp=0)", "B(logp=0)"):
        assert col in head
    assert len(lines) - 1 == sol.iterations + 1
    last, prev = lines[-1].split(","), lines[-2].split(",")
    assert float(last[1]) < prm.xi and float(last[2]) < prm.xi
    for col, lp in ((3, -2.5), (5, 0.0)):
        p2 = 10.0 ** (2.0 * lp)
        assert float(last[col]) == p.interp_search(sol.grid.p2_ext, sol.A, p2)
        assert float(last[col + 1]) == p.interp_search(sol.grid.p2_ext, sol.B, p2)
    for col in (3, 4, 5, 6):
        assert abs(float(last[col]) - float(prev[col])) < prm.xi
