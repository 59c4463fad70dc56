"""GPU, BASELINE config 3 at full size (128 x 128 external, 128 x 128 x 32
internal, mu = 0.2 GeV): parity on sampled rows against the numpy oracle
(each row is a full 524,288-point block; the oracle takes ~0.5 s per row),
and size-independent properties of the converged solution -- the p4 -> -p4
conjugation symmetry F(|p|, -p4) = conj F(|p|, p4) of the equations on the
symmetric grids, and bitwise row-sharding invariance."""
import numpy as np
import pytest

import mu_oracle
from paper_2012_03667_b200.finite_mu import MuSweeper
from paper_2012_03667_b200.mu_grid import MuParams, grid_for

pytestmark = pytest.mark.gpu

ROWS = [0, 77, 5000, 8191, 8192, 12345, 16383]


@pytest.fixture(scope="module")
def config3():
    p = MuParams(max_iterations=3)
    g = grid_for(p)
    with MuSweeper(g, p) as sw:
        st = sw.solve(p)  # 3 iterations from A = C = 1, B = 0.3: a non-trivial complex state
        out = sw.sweep(st.A, st.B, st.C)
    return p, g, st, out


def test_config3_sweep_rows_match_oracle(config3):
    p, g, st, out = config3
    Aq, Bq, Cq = (mu_oracle.interp2d(g, X) for X in (st.A, st.B, st.C))
    for i in ROWS:
        ra, rb, rc, _ = mu_oracle.sweep_row(g, p, i, st.A, st.B, st.C, Aq, Bq, Cq)
        for got, ref in ((out[0].reshape(-1)[i], ra), (out[1].reshape(-1)[i], rb), (out[2].reshape(-1)[i], rc)):
            assert abs(got - ref) <= 1e-11 * max(abs(ref), 1e-3), (i, got, ref)


def test_config3_conjugation_symmetry_and_convergence():
    p = MuParams()
    g = grid_for(p)
    assert np.allclose(g.p4_ext, -g.p4_ext[::-1], rtol=0, atol=1e-12) and np.allclose(g.q4_int, -g.q4_int[::-1])
    with MuSweeper(g, p) as sw:
        sol = sw.solve(p)
    assert sol.converged and sol.iterations < 100
    for F in (sol.A, sol.B, sol.C):
        assert np.max(np.abs(F[:, ::-1] - np.conj(F))) <= 1e-10 * np.max(np.abs(F))
    # a finite density makes the functions complex; the imaginary parts are odd in p4
    assert np.max(np.abs(sol.A.imag)) > 1e-6


def test_config3_row_sharding_bitwise(config3):
    p, g, st, full = config3
    W = 2
    parts = [np.zeros_like(full[f]) for f in range(3)]
    for r in range(W):
        with MuSweeper(g, p, row_start=r, row_stride=W) as sw:
            x = sw.sweep(st.A, st.B, st.C)
        for f in range(3):
            parts[f].reshape(-1)[r::W] = x[f].reshape(-1)[r::W]
    for f in range(3):
        assert np.array_equal(parts[f].view(np.float64), full[f].view(np.float64))


def test_config3_moments_mode_equals_direct():
    p = MuParams()
    g = grid_for(p)
    with MuSweeper(g, p) as sw:
        ref = sw.solve(p)
        got = sw.solve(MuParams(**{**p.__dict__, "mode": "moments"}))
    assert got.iterations == ref.iterations and got.converged
    for x, y in ((got.A, ref.A), (got.B, ref.B), (got.C, ref.C)):
        assert np.array_equal(x.view(np.float64), y.view(np.float64))
