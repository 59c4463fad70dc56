"""GPU parity of the batched interpolation (config 1) and the internal-node
interpolation: bitwise values and bracket indices vs the reference."""
import numpy as np
import pytest

import oracle
import paper_2012_03667_b200 as p
from conftest import golden, golden_grid

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["search", "direct"])
def test_interp_golden_sample_bitwise(mode):
    z = golden("interp_c1.npz")
    vals, idx = p.interp_linear_batch(z["x"], z["v"], z["q"], mode=mode, with_index=True)
    assert np.array_equal(vals, z["values"], equal_nan=True)
    assert np.array_equal(idx.astype(np.int64), z["idx"])
    vals2, idx2 = p.interp_linear_batch(z["x2"], z["v2"], z["q2"], mode=mode, with_index=True)
    assert np.array_equal(vals2, z["values2"]) and np.array_equal(idx2.astype(np.int64), z["idx2"])


def test_comparison_counter_matches_reference():
    z = golden("interp_c1.npz")
    c = p.ComparisonCounter()
    p.interp_search_many(z["x"], z["v"], z["q"], counter=c)
    assert c.count == int(z["comparisons"])


def test_internal_node_interp_bitwise():
    g = golden_grid("c0")
    rng = np.random.default_rng(4)
    v = rng.uniform(-2, 2, g.n_ext)
    r1 = p.interp_indexed_many(g, v)
    r2 = p.interp_search_many(g.p2_ext, v, g.q2_int)
    ref = oracle.interp_search_many(g.p2_ext, v, g.q2_int)
    assert np.array_equal(r1, ref) and np.array_equal(r2, ref)
    assert p.interp_indexed(g, v, 5) == ref[5]
    assert p.interp_search(g.p2_ext, v, 0.37) == oracle.interp_search_many(g.p2_ext, v, [0.37])[0]


@pytest.mark.parametrize("mode", ["search", "direct"])
def test_interp_config1_full_size(mode):
    """BASELINE config 1 at full size (2**26 seeded queries): indices equal the
    reference's index oracle clip(searchsorted(x, q, 'right') - 1, -1, n-1)
    (test_grid.py:30 pattern) and values equal the C oracle bitwise."""
    x = np.logspace(-4, 4, 512)
    v = 1.0 / (1.0 + x) + 0.1 * np.log1p(x)
    q = np.exp(np.random.default_rng(0).uniform(np.log(1e-4), np.log(1e4), 2 ** 26))
    vals, idx = p.interp_linear_batch(x, v, q, mode=mode, with_index=True)
    ref_idx = np.clip(np.searchsorted(x, q, "right") - 1, -1, x.size - 1)
    assert np.array_equal(idx, ref_idx)
    ref = oracle.interp_search_many(x, v, q, threads=oracle.max_threads())
    assert np.array_equal(vals, ref)


def test_interp_validation():
    with pytest.raises(p.ParameterError):
        p.interp_search_many(np.array([1.0]), np.array([1.0]), np.array([1.0]))
    with pytest.raises(p.ParameterError):
        p.interp_search_many(np.array([1.0, 1.0]), np.array([1.0, 2.0]), np.array([1.0]))
    assert p.interp_search_many(np.array([1.0, 2.0]), np.array([1.0, 2.0]), np.array([])).size == 0


@pytest.mark.parametrize("table", ["logspace", "nonuniform", "flat_pieces"])
@pytest.mark.parametrize("mode", ["search", "direct"])
def test_streaming_kernel_edge_cases_bitwise(table, mode, monkeypatch):
    """The TMA-streamed kernel (tables replicated per bank group, precomputed
    reciprocals, one-branch fast path) against the C oracle and against the
    plain kernel (DSE_INTERP_NOSTREAM): knots, their neighbours, clamps,
    NaN/inf, constant pieces (zero dv: the reciprocal path falls back to
    IEEE division) -- 40k queries, so full tiles, a tail and the slow path
    all run."""
    rng = np.random.default_rng(31)
    if table == "logspace":
        x = np.logspace(-4, 4, 512)
        v = 1.0 / (1.0 + x) + 0.1 * np.log1p(x)
    elif table == "nonuniform":
        x = np.cumsum(rng.exponential(1.0, 300)) + 1e-3
        v = rng.normal(size=300)
    else:
        x = np.logspace(-2, 2, 64)
        v = np.repeat(rng.normal(size=16), 4)  # constant on 3 of every 4 intervals
    edge = np.concatenate([x, np.nextafter(x, 0), np.nextafter(x, np.inf), [0.0, -1.0, np.inf, -np.inf, np.nan],
                           [x[0] * 0.5, x[-1] * 2.0]])
    q = np.concatenate([np.exp(rng.uniform(np.log(x[0]) - 0.1, np.log(x[-1]) + 0.1, 40000 - edge.size)), edge])
    rng.shuffle(q)
    ref = oracle.interp_search_many(x, v, q)
    ref_idx = np.clip(np.searchsorted(x, q, "right") - 1, -1, x.size - 1)
    ref_idx[np.isnan(q)] = 0
    got, idx = p.interp_linear_batch(x, v, q, mode=mode, with_index=True)
    monkeypatch.setenv("DSE_INTERP_NOSTREAM", "1")
    plain, pidx = p.interp_linear_batch(x, v, q, mode=mode, with_index=True)
    assert np.array_equal(got, ref, equal_nan=True) and np.array_equal(plain, ref, equal_nan=True)
    assert np.array_equal(idx, ref_idx) and np.array_equal(pidx, ref_idx)
