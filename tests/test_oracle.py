"""CPU: pin the oracle (oracle/dse_oracle.c) against golden vectors generated
by RUNNING THE REFERENCE (tests/golden/make_golden.py)."""
import numpy as np
import pytest

import oracle
from conftest import golden, golden_grid, hybrid_rel, params_ns


def _case_params(S, name, **kw):
    D, om, m0, z1, c = S[f"{name}__params"]
    return params_ns(D=D, omega=om, m0=m0, z1=z1, coeff=c, **kw)


def test_pairwise_sum_matches_numpy_sum():
    rng = np.random.default_rng(3)
    for shape in [(128, 64), (100, 32), (37, 5), (20, 8), (1024, 256), (3, 2), (7, 1), (1, 1), (129, 1)]:
        x = rng.standard_normal(shape) * np.exp(rng.uniform(-30, 30, shape))
        assert oracle.pairwise_sum(x) == float(np.sum(x)), shape


def test_oracle_sweep_bitwise_vs_reference_with_glibc_exp():
    """With numpy.exp routed through glibc exp, the reference's sweep equals the
    oracle BITWISE: the oracle restates row_rhs's op order and np.sum's tree."""
    S = golden("sweeps.npz")
    L = golden("sweeps_libm.npz")
    for name in S["names"]:
        g = golden_grid(str(S[f"{name}__grid"]))
        p = _case_params(S, name)
        a, b = oracle.sweep(g, S[f"{name}__a"], S[f"{name}__b"], p, strategy=1, threads=2)
        assert np.array_equal(a, L[f"{name}__a_out"]), name
        assert np.array_equal(b, L[f"{name}__b_out"]), name


@pytest.mark.parametrize("strategy", [0, 1])
def test_oracle_sweep_vs_reference(strategy):
    S = golden("sweeps.npz")
    for name in S["names"]:
        g = golden_grid(str(S[f"{name}__grid"]))
        p = _case_params(S, name)
        a, b = oracle.sweep(g, S[f"{name}__a"], S[f"{name}__b"], p, strategy=strategy, threads=2)
        assert hybrid_rel(a, S[f"{name}__a_out"]) <= 1e-13, name
        assert hybrid_rel(b, S[f"{name}__b_out"]) <= 1e-13, name


def test_oracle_interp_vs_reference():
    z = golden("interp_c1.npz")
    vals, idx, cmp = oracle.interp_search_many(z["x"], z["v"], z["q"], threads=2, with_index=True)
    assert np.array_equal(vals, z["values"], equal_nan=True)
    assert np.array_equal(idx, z["idx"])
    assert cmp == int(z["comparisons"])
    vals2, idx2, _ = oracle.interp_search_many(z["x2"], z["v2"], z["q2"], with_index=True)
    assert np.array_equal(vals2, z["values2"]) and np.array_equal(idx2, z["idx2"])


def test_oracle_merge_bracket_indices():
    for tag in ("c0", "default", "ragged", "coincide", "c2"):
        g = golden_grid(tag)
        assert np.array_equal(oracle.merge_bracket_indices(g.p2_ext, g.q2_int), g.bracket_idx)


def test_oracle_error_locations():
    E = golden("errors.npz")
    g = golden_grid("small")
    p = params_ns()
    for name in E["names"]:
        with pytest.raises(oracle.OracleError) as ei:
            oracle.sweep(g, E[f"{name}__a"], E[f"{name}__b"], p)
        assert ei.value.loc == tuple(int(v) for v in E[f"{name}__loc"]), name


def _solve_golden(fname, tag, threads=4):
    z = golden(fname)
    D, om, m0, z1, xi, relax, cap, c = z["params"]
    p = params_ns(D=D, omega=om, m0=m0, z1=z1, xi=xi, relaxation=relax, max_iterations=int(cap), coeff=c)
    g = golden_grid(tag)
    probes = [10.0 ** (2.0 * lp) for lp in z["probes_log10p"]]
    b0 = z["b0"] if z["b0"].shape == (g.n_ext,) else np.ones(g.n_ext)
    return z, oracle.solve(g, p, np.ones(g.n_ext), b0, probes, strategy=1, threads=threads)


def test_oracle_solve_default_config():
    z, (a, b, n, conv, hist) = _solve_golden("solve_default.npz", "default")
    assert n == int(z["iterations"]) and conv == bool(z["converged"])
    assert hybrid_rel(a, z["A"]) <= 1e-12 and hybrid_rel(b, z["B"]) <= 1e-12
    assert hist.shape == z["history"].shape
    np.testing.assert_allclose(hist[1:, 1:3], z["history"][1:, 1:3], rtol=1e-6)
    np.testing.assert_allclose(hist[:, 3:], z["history"][:, 3:], rtol=1e-12)


@pytest.mark.slow
def test_oracle_solve_config0_2923_iterations():
    z, (a, b, n, conv, hist) = _solve_golden("solve_c0.npz", "c0", threads=8)
    assert n == int(z["iterations"]) == 2923 and conv
    assert hybrid_rel(a, z["A"]) <= 1e-9 and hybrid_rel(b, z["B"]) <= 1e-9
