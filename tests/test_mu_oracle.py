"""CPU: the finite-mu oracle (BASELINE configs 3-4; no reference path exists,
SURVEY.md §8c) pinned three ways -- explicit Dirac traces, the reference's
own vacuum integrand at mu = 0 (tests/golden/mu_vacuum_points.npz, made by
tests/golden/make_mu_golden.py), and the grid's known-answer integrals."""
import numpy as np
import pytest

import mu_dirac
import mu_oracle
from conftest import golden
from paper_2012_03667_b200.mu_grid import MuParams, build_mu_grid, grid_for


def _random_point(rng):
    P, Qs = rng.uniform(0.05, 3, 2)
    z = rng.uniform(-1, 1)
    p4r, q4r = rng.uniform(-2, 2, 2)
    mu = rng.uniform(0, 0.5)
    vals = [complex(rng.uniform(0.5, 2), rng.uniform(-0.3, 0.3)) for _ in range(6)]
    return (P, p4r + 1j * mu, Qs, z, q4r + 1j * mu, q4r, p4r, *vals)


@pytest.mark.parametrize("vertex", ["bc", "bc1", "bcb"])
def test_projections_match_dirac_traces(vertex):
    rng = np.random.default_rng(7)
    for _ in range(25):
        args = _random_point(rng)
        k2d, pa, pc, pb, wti = mu_dirac.projections(*args, vertex=vertex)
        P, p4t, Qs, z, q4t, q4r, p4r = args[:7]
        k2, PA, PC, PB = mu_oracle.point_projections(np.float64(P), p4t, np.float64(Qs), np.float64(z), q4t, q4r,
                                                     p4r, *args[7:], vertex=vertex)
        assert wti < 1e-12  # Ward-Takahashi identity of the in-medium Ball-Chiu vertex
        assert abs(k2 - k2d) <= 1e-14 * k2d
        for x, y in ((pa, PA), (pc, PC), (pb, PB)):
            assert abs(x - y) <= 1e-13 * max(abs(x), 1e-300), (vertex, x, y)


def test_mu0_reduces_to_reference_vacuum_integrand():
    """mu = 0, C = A: P_A + p4 P_C == IA2 + IA3 and P_B == IB1 + IB2 + IB3 of
    the reference (kernels.py:152-175), pointwise."""
    g = golden("mu_vacuum_points.npz")
    c = lambda x: x + 0j  # noqa: E731
    k2, PA, PC, PB = mu_oracle.point_projections(g["P"], c(g["p4"]), g["Qs"], g["z"], c(g["q4"]), g["q4"], g["p4"],
                                                 c(g["ap"]), c(g["bp"]), c(g["ap"]), c(g["aq"]), c(g["bq"]),
                                                 c(g["aq"]))
    ia = PA + g["p4"] * PC
    assert np.max(np.abs(ia.imag)) == 0.0 and np.max(np.abs(PB.imag)) == 0.0
    assert np.max(np.abs(ia.real - g["ia"]) / np.abs(g["ia"])) < 1e-12
    assert np.max(np.abs(PB.real - g["ib"]) / np.abs(g["ib"])) < 1e-12
    kin_k2 = g["p2"] + g["q2"] - 2 * np.sqrt(g["p2"] * g["q2"]) * g["z4"]
    assert np.max(np.abs(k2 - kin_k2) / kin_k2) < 1e-10


def test_grid_brackets_and_measure():
    g = build_mu_grid(24, 20, 32, 28, 8)
    assert np.array_equal(g.brk_s, np.searchsorted(g.ps2_ext, g.qs2_int, side="right") - 1)
    assert np.array_equal(g.brk_4, np.searchsorted(g.p4_ext, g.q4_int, side="right") - 1)
    assert np.all(np.diff(g.p_ext) > 0) and np.all(np.diff(g.p4_ext) > 0)
    assert g.node_measure.shape == (32, 28)
    # int d^4q/(2 pi)^4 exp(-q^2) = 1/(16 pi^2)  (vacuum KAT, test_kernels.py:197-201)
    gg = grid_for(MuParams())
    val = np.sum(gg.node_measure * np.exp(-(gg.qs2_int[:, None] + gg.q4_int[None, :] ** 2))) * np.sum(gg.z_weights)
    assert abs(val - 1.0 / (16 * np.pi**2)) < 1e-8 / (16 * np.pi**2)


def test_interp2d_exact_on_bilinear_and_clamped():
    g = build_mu_grid(12, 10, 16, 14, 4)
    S, T = np.meshgrid(g.ps2_ext, g.p4_ext, indexing="ij")
    F = (1.5 + 0.25 * S - 0.5 * T + 0.125 * S * T) + 1j * (0.5 - S + 2 * T)
    out = mu_oracle.interp2d(g, F)
    qs, q4 = np.meshgrid(g.qs2_int, g.q4_int, indexing="ij")
    qs_c = np.clip(qs, g.ps2_ext[0], g.ps2_ext[-1])
    q4_c = np.clip(q4, g.p4_ext[0], g.p4_ext[-1])
    ref = (1.5 + 0.25 * qs_c - 0.5 * q4_c + 0.125 * qs_c * q4_c) + 1j * (0.5 - qs_c + 2 * q4_c)
    assert np.max(np.abs(out - ref) / np.abs(ref)) < 1e-12


@pytest.mark.slow
def test_mu0_bc1_restores_o4_symmetry():
    """mu = 0: the converged A and C agree (O(4) symmetry) up to discretisation."""
    p = MuParams(mu=0.0, n_s=10, n_4=10, m_s=16, m_4=16, m_ang=6, vertex="bc1", max_iterations=200, xi=1e-8)
    A, B, C, n, conv, hist = mu_oracle.solve(grid_for(p), p)
    assert conv
    assert np.max(np.abs(A.imag)) == 0.0
    ir = slice(0, 6)
    assert np.max(np.abs(A[ir] - C[ir]) / np.abs(A[ir])) < 0.25


def test_mu0_p4_zero_node_rejected_before_any_device_call():
    from paper_2012_03667_b200.errors import ParameterError
    from paper_2012_03667_b200.finite_mu import MuSweeper
    p = MuParams(mu=0.0, n_s=4, n_4=5, m_s=6, m_4=6, m_ang=2)  # odd n_4: the middle midpoint is p4 = 0
    g = grid_for(p)
    assert np.any(g.p4_ext == 0.0)
    with pytest.raises(ParameterError):
        MuSweeper(g, p)


def test_grid_rejects_bad_sizes():
    from paper_2012_03667_b200.errors import ParameterError
    for kw in (dict(n_s=1), dict(m_4=1), dict(m_ang=0)):
        args = dict(n_s=4, n_4=4, m_s=4, m_4=4, m_ang=2)
        args.update(kw)
        with pytest.raises(ParameterError):
            build_mu_grid(**args)
    with pytest.raises(ParameterError):
        MuParams(vertex="rainbow").validate()
    with pytest.raises(ParameterError):
        MuParams(mode="fast").validate()


@pytest.mark.parametrize("vertex", ["bc", "bc1", "bcb"])
def test_c_restatement_matches_numpy_oracle(vertex):
    p = MuParams(mu=0.2, vertex=vertex, n_s=8, n_4=10, m_s=12, m_4=14, m_ang=6)
    g = grid_for(p)
    rng = np.random.default_rng(3)
    shape = (g.n_s, g.n_4)
    A = 1 + rng.random(shape) + 0.1j * rng.standard_normal(shape)
    B = 0.2 + 0.3 * rng.random(shape) + 0.05j * rng.standard_normal(shape)
    C = 1 + rng.random(shape) + 0.1j * rng.standard_normal(shape)
    rows = np.arange(g.n_ext)
    got = mu_oracle.sweep_rows_c(g, p, A, B, C, rows, threads=2)
    ref = mu_oracle.sweep(g, p, A, B, C)
    for f in range(3):
        r = ref[f].reshape(-1)
        assert np.max(np.abs(got[:, f] - r)) <= 1e-12 * np.max(np.abs(r))


@pytest.mark.parametrize("vertex", ["bc", "bcb"])
def test_c_restatement_node_skip_is_bitwise(vertex):
    """The exact-zero node skip of the C oracle (the GPU kernels' window skip)
    changes no bit: every skipped summand is an exact zero.  A narrow
    interaction (omega = 0.15) makes most nodes skippable on this grid."""
    p = MuParams(mu=0.2, vertex=vertex, omega=0.15, n_s=10, n_4=12, m_s=16, m_4=18, m_ang=6)
    g = grid_for(p)
    rng = np.random.default_rng(5)
    shape = (g.n_s, g.n_4)
    A = 1 + rng.random(shape) + 0.1j * rng.standard_normal(shape)
    B = 0.2 + 0.3 * rng.random(shape) + 0.05j * rng.standard_normal(shape)
    C = 1 + rng.random(shape) + 0.1j * rng.standard_normal(shape)
    rows = np.arange(g.n_ext)
    a = mu_oracle.sweep_rows_c(g, p, A, B, C, rows, threads=2, skip=True)
    b = mu_oracle.sweep_rows_c(g, p, A, B, C, rows, threads=2, skip=False)
    assert np.array_equal(a.view(np.float64), b.view(np.float64))
