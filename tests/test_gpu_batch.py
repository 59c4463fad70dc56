"""GPU: batched independent solves (solve_batch) equal the individual solves
bitwise -- iterations, converged flags, A, B and the full history."""
import numpy as np
import pytest

import paper_2012_03667_b200 as p
from conftest import golden, golden_grid, params_ns

pytestmark = pytest.mark.gpu


def _same(x, y):
    assert x.iterations == y.iterations and x.converged == y.converged
    assert np.array_equal(x.A, y.A) and np.array_equal(x.B, y.B)
    hx = np.array([[r.iteration, r.max_delta_a, r.max_delta_b, *r.probe_a, *r.probe_b] for r in x.history])
    hy = np.array([[r.iteration, r.max_delta_a, r.max_delta_b, *r.probe_a, *r.probe_b] for r in y.history])
    assert np.array_equal(hx, hy, equal_nan=True)


@pytest.fixture(params=["kernel", "streams"])
def batch_mode(request, monkeypatch):
    """dse_solve_batch has two implementations: one batched cooperative kernel
    (default) and concurrent per-solve kernels on streams (fallback)."""
    if request.param == "streams":
        monkeypatch.setenv("DSE_BATCH_STREAMS", "1")
    else:
        monkeypatch.delenv("DSE_BATCH_STREAMS", raising=False)
    return request.param


@pytest.mark.parametrize("vname", ["indexed-gpu", "search-gpu-exact", "indexed-gpu-moments", "search-gpu-moments"])
def test_batch_equals_individual_solves(vname, batch_mode):
    g = golden_grid("default")
    plist = [params_ns(D=d, m0=m0, relaxation=r, xi=1e-6, max_iterations=cap)
             for d, m0, r, cap in ((0.55, 0.0, 1.0, 200), (0.45, 0.005, 1.0, 200), (0.65, 0.0, 0.7, 300),
                                   (0.0, 0.01, 1.0, 50), (0.55, 0.0, 1.0, 3), (0.6, 0.002, 0.9, 250))]
    b0s = np.stack([np.full(g.n_ext, b) for b in (0.3, 1.0, 0.5, 1.0, 0.3, 0.8)])
    batch = p.solve_batch(plist, p.VARIANTS[vname], grid=g, b0s=b0s)
    for prm, b0, got in zip(plist, b0s, batch):
        _same(got, p.solve(prm, p.VARIANTS[vname], grid=g, b0=b0))
    assert batch[3].iterations <= 2 and np.all(batch[3].A == 1.0)   # free theory
    assert batch[4].iterations == 3 and not batch[4].converged       # cap


@pytest.mark.parametrize("vname", ["indexed-gpu", "indexed-gpu-moments"])
def test_batch_config0_scan(batch_mode, vname):
    z = golden("solve_c0.npz")
    g = golden_grid("c0")
    plist = [params_ns(D=d, xi=1e-10, max_iterations=4000) for d in (0.55, 0.5, 0.6)]
    sols = p.solve_batch(plist, p.VARIANTS[vname], grid=g, b0s=np.full((3, g.n_ext), 0.3))
    assert sols[0].iterations == int(z["iterations"]) == 2923 and sols[0].converged
    for prm, got in zip(plist[1:], sols[1:]):
        _same(got, p.solve(prm, p.VARIANTS[vname], grid=g, b0=np.full(g.n_ext, 0.3)))


def test_batch_validation():
    with pytest.raises(p.ParameterError):
        p.solve_batch([p.ModelParams(N=20), p.ModelParams(N=30)], p.VARIANTS["indexed-gpu"])
    assert p.solve_batch([], p.VARIANTS["indexed-gpu"]) == []


@pytest.mark.parametrize("vname", ["indexed-gpu", "indexed-gpu-moments"])
def test_batch_failure_is_per_solve_and_located(batch_mode, vname):
    g = golden_grid("small")
    b0s = np.full((2, g.n_ext), 0.3)
    a0s = np.ones((2, g.n_ext))
    a0s[1, 5] = np.inf
    with pytest.raises(p.NumericalFailureError) as ei:
        p.solve_batch([params_ns(xi=1e-3, max_iterations=5)] * 2, p.VARIANTS[vname], grid=g, a0s=a0s, b0s=b0s)
    single = None
    try:
        p.solve(params_ns(xi=1e-3, max_iterations=5), p.VARIANTS[vname], grid=g, a0=a0s[1], b0=b0s[1])
    except p.NumericalFailureError as exc:
        single = exc
    assert single is not None
    assert (ei.value.row, ei.value.radial, ei.value.angular) == (single.row, single.radial, single.angular)


def test_batch_moments_mixed_omega_falls_back_bitwise():
    """Moments solves with different omegas cannot share one moment table:
    solve_batch runs them on the per-solve path, still bitwise the standalone
    solves."""
    g = golden_grid("default")
    plist = [params_ns(D=0.55, omega=0.678, xi=1e-6, max_iterations=200),
             params_ns(D=0.55, omega=0.6, xi=1e-6, max_iterations=200),
             params_ns(D=0.5, omega=0.678, xi=1e-6, max_iterations=200)]
    v = p.VARIANTS["indexed-gpu-moments"]
    b0s = np.full((3, g.n_ext), 0.3)
    batch = p.solve_batch(plist, v, grid=g, b0s=b0s)
    for prm, b0, got in zip(plist, b0s, batch):
        _same(got, p.solve(prm, v, grid=g, b0=b0))
