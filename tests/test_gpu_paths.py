"""GPU: the fast sweep's execution layouts give bit-identical results.

The many-rows regime can run 8 threads per leaf (one numpy lane sum each) or
4 threads per leaf (two lane sums each), and rows may be split into subtree
chunks.  All of these evaluate every lane sum with the same operation
sequence and combine in numpy's tree order, so the outputs must agree bit for
bit (the layout is chosen from the environment at launch: DSE_GL8,
DSE_SPLIT_ROWS/DSE_CHUNK_LEAVES).
"""
import os

import numpy as np
import pytest

import paper_2012_03667_b200 as p

pytestmark = pytest.mark.gpu

# (N, M, K): power-of-two trees (32 leaves of 128, 64 of 72 elements), an
# unequal-leaf tree (3000 elements: leaves of 88-96) and an irregularly shaped
# one (132 x 32: subtrees of 264 split 128 | 64 + 72)
GRIDS = [(400, 64, 64), (320, 96, 48), (350, 100, 30), (330, 132, 32)]


def _sweep(g, prm, env, arith=p.Arithmetic.FAST):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, arith, 0)
        try:
            rng = np.random.default_rng(7)
            a = 1.0 + 0.3 * rng.random(g.n_ext)
            b = 0.2 + 0.2 * rng.random(g.n_ext)
            ao, bo = sw.sweep(a, b)
            return ao, bo, sw.layout()
        finally:
            sw.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("n,m,k", GRIDS)
def test_layouts_bitwise_equal(n, m, k):
    g = p.build_grid(n, m, k, 1e-4, 1e4)
    prm = p.ModelParams(N=n, m_rad=m, m_ang=k, xi=1e-10)
    a0, b0, lay = _sweep(g, prm, {})
    assert lay["lanes_per_leaf"] == 4 and lay["static_items"] == 0 and lay["node_chunk"] > 0
    variants = [{"DSE_GL8": "1"},
                {"DSE_SPLIT_ROWS": "-1", "DSE_CHUNK_LEAVES": "8"},
                {"DSE_SPLIT_ROWS": "-1", "DSE_CHUNK_LEAVES": "16", "DSE_GL8": "1"}]
    for env in variants:
        a1, b1, lay1 = _sweep(g, prm, env)
        assert np.array_equal(a0, a1) and np.array_equal(b0, b1), (env, lay1)
    assert _sweep(g, prm, variants[0])[2]["lanes_per_leaf"] == 8
    assert _sweep(g, prm, variants[1])[2]["split_rows"] == n
    # and the layouts agree with exact arithmetic to the fast-mode tolerance
    ae, be, _ = _sweep(g, prm, {}, p.Arithmetic.EXACT)
    assert np.max(np.abs(a0 - ae) / np.abs(ae)) < 1e-12
    assert np.max(np.abs(b0 - be)) / np.max(np.abs(be)) < 1e-12


@pytest.mark.parametrize("n,m,k", [(128, 128, 64), (300, 1000, 16)])
def test_moments_warps_per_row_bitwise_equal(n, m, k):
    """The moments kernel's warps per row (DSE_MOM_WPR) changes which warp
    sums which group of radial nodes, never the order: bit-identical."""
    g = p.build_grid(n, m, k, 1e-4, 1e4)
    prm = p.ModelParams(N=n, m_rad=m, m_ang=k, xi=1e-10)
    ref = _sweep(g, prm, {}, p.Arithmetic.MOMENTS)
    for wpr in ("1", "2", "4", "8", "3"):
        x = _sweep(g, prm, {"DSE_MOM_WPR": wpr}, p.Arithmetic.MOMENTS)
        assert np.array_equal(ref[0], x[0]) and np.array_equal(ref[1], x[1]), wpr


@pytest.mark.parametrize("n,m,k", [(128, 128, 64), (300, 1000, 16), (1024, 1024, 256)])
def test_pairs_grid_size_bitwise_equal(n, m, k):
    """The pairs kernel deals (row, 32-node group) items to warps by ticket;
    the grid size changes who computes a group, never the order of any sum."""
    g = p.build_grid(n, m, k, 1e-6, 1e4)
    prm = p.ModelParams(N=n, m_rad=m, m_ang=k, xi=1e-10)
    ref = _sweep(g, prm, {}, p.Arithmetic.PAIRS)
    for blocks in ("1", "7", "150"):
        x = _sweep(g, prm, {"DSE_PAIRS_BLOCKS": blocks}, p.Arithmetic.PAIRS)
        assert np.array_equal(ref[0], x[0]) and np.array_equal(ref[1], x[1]), blocks
    for threads in ("640", "320", "96"):  # the launch shape (one CTA of 640 / two of 320 by problem size)
        x = _sweep(g, prm, {"DSE_PAIRS_LAUNCH_THREADS": threads}, p.Arithmetic.PAIRS)
        assert np.array_equal(ref[0], x[0]) and np.array_equal(ref[1], x[1]), threads
    for chunks in ("2", "4"):  # angle chunks change the partition, not the result beyond rounding
        x = _sweep(g, prm, {"DSE_PAIRS_CHUNKS": chunks}, p.Arithmetic.PAIRS)
        assert np.max(np.abs(ref[0] - x[0]) / np.abs(ref[0])) < 1e-13
    fast = _sweep(g, prm, {}, p.Arithmetic.FAST)
    assert np.max(np.abs(ref[0] - fast[0]) / np.abs(fast[0])) < 1e-12
    assert np.max(np.abs(ref[1] - fast[1])) / np.max(np.abs(fast[1])) < 1e-12


@pytest.mark.parametrize("arith", [p.Arithmetic.EXACT, p.Arithmetic.FAST])
def test_cluster_layout_bitwise(arith, monkeypatch):
    """The few-rows layouts (2-CTA clusters for the exact arithmetic, one
    512-thread CTA per row otherwise; DSE_NO_CLUSTER forces the latter) give
    bit-identical sweeps and solves."""
    g = p.build_grid(128, 128, 64, 1e-6, 1e4)
    prm = p.ModelParams(N=128, m_rad=128, m_ang=64, xi=1e-10, max_iterations=300)
    rng = np.random.default_rng(12)
    a, b = rng.uniform(1, 2, 128), rng.uniform(0, 1, 128)
    outs = []
    for env in (None, "1"):
        if env is None:
            monkeypatch.delenv("DSE_NO_CLUSTER", raising=False)
        else:
            monkeypatch.setenv("DSE_NO_CLUSTER", env)
        sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, arith)
        lay = sw.layout()
        x = sw.sweep(a, b)
        y = sw.solve(np.ones(128), np.full(128, 0.3), (1e-5, 1.0))
        outs.append((lay, x, y))
        sw.close()
    if arith is p.Arithmetic.EXACT:
        assert outs[0][0]["cluster2"] == 1 and outs[1][0]["cluster2"] == 0
    (_, x0, y0), (_, x1, y1) = outs
    assert np.array_equal(x0[0], x1[0]) and np.array_equal(x0[1], x1[1])
    assert y0[2] == y1[2] and np.array_equal(y0[0], y1[0]) and np.array_equal(y0[1], y1[1])
    assert np.array_equal(y0[4], y1[4], equal_nan=True)
