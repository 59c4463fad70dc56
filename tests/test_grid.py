"""CPU: the host grid builder reproduces the reference's grids bitwise."""
import numpy as np
import pytest

from conftest import golden
from paper_2012_03667_b200 import (GridConstructionError, ParameterError, build_grid, gauss_chebyshev2,
                                   gauss_legendre, merge_bracket_indices)

FIELDS = ["p2_ext", "s_nodes", "s_weights", "q2_int", "bracket_idx", "z_nodes", "z_weights", "sqrt_q2_int",
          "radial_measure"]


@pytest.mark.parametrize("tag", ["c0", "default", "small", "ragged", "tiny", "coincide", "sub256", "c2"])
def test_build_grid_bitwise_vs_reference(tag):
    z = golden(f"grid_{tag}.npz")
    n, m, k = (int(v) for v in z["args"])
    lo, hi = (float(v) for v in z["p2_range"])
    g = build_grid(n, m, k, lo, hi)
    for f in FIELDS:
        assert np.array_equal(getattr(g, f), z[f]), (tag, f)
    assert np.array_equal(g.weight_jk, np.outer(z["radial_measure"], z["z_weights"]))
    assert np.array_equal(g.sz, np.outer(z["sqrt_q2_int"], z["z_nodes"]))


def test_coincidence_shift_applied():
    g = build_grid(3, 3, 2, 1.0, 9.0)
    assert g.p2_ext[1] != 3.0 and np.all(np.diff(g.p2_ext) > 0)
    assert np.min(np.abs(g.q2_int[:, None] - g.p2_ext[None, :])) > 1e-6


def test_merge_indices_equal_searchsorted_and_invariant():
    rng = np.random.default_rng(0)
    for _ in range(200):
        n, m = rng.integers(2, 60, 2)
        g = build_grid(int(n), int(m), 3, 10 ** rng.uniform(-6, -1), 10 ** rng.uniform(1, 4))
        idx = g.bracket_idx
        for j, q in enumerate(g.q2_int):
            i = idx[j]
            if i < 0:
                assert q < g.p2_ext[0]
            elif i >= g.n_ext - 1:
                assert q >= g.p2_ext[-1]
            else:
                assert g.p2_ext[i] <= q < g.p2_ext[i + 1]


def test_quadrature_known_answers():
    r = gauss_legendre(2, -1.0, 1.0)
    np.testing.assert_allclose(r.nodes, [-1 / np.sqrt(3), 1 / np.sqrt(3)], rtol=1e-15)
    np.testing.assert_allclose(r.weights, [1.0, 1.0], rtol=1e-15)
    r = gauss_legendre(64, 0.0, 2.0)
    assert abs(r.integrate(r.nodes ** 9) - 2.0 ** 10 / 10) < 1e-10
    c = gauss_chebyshev2(16)
    assert abs(c.integrate(np.ones(16)) - np.pi / 2) < 1e-14
    assert abs(c.integrate(c.nodes ** 2) - np.pi / 8) < 1e-14


def test_grid_validation():
    with pytest.raises(ParameterError):
        build_grid(1, 4, 4, 1e-6, 1e4)
    with pytest.raises(ParameterError):
        build_grid(4, 4, 4, 1.0, 1.0)
    with pytest.raises(ParameterError):
        gauss_legendre(0, 0.0, 1.0)
    assert issubclass(GridConstructionError, RuntimeError)
    assert np.array_equal(merge_bracket_indices(np.array([1.0, 2.0, 3.0]), np.array([0.5, 1.0, 2.5, 3.0, 4.0])),
                          [-1, 0, 1, 2, 2])
