"""CPU, world_size 2 over gloo: the row-sharded loop (partition, all-gather,
reassembly, relaxation, max-norm deltas, history) equals the unsharded loop
bitwise.  The per-row map is a synthetic Jacobi contraction (a test double
for the GPU sweep): this tests the host logic of distributed.py, the GPU
sweep's own row-sharding invariance is tests/test_gpu_sweep.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2012_03667_b200.distributed import ShardedLoop, owned_rows

N = 37


def jacobi_map(a, b):
    """a'_i, b'_i depend on the whole previous iterate (like the qDSE sweep)."""
    a_next = 1.0 + 0.4 * np.sin(np.roll(a, 1)) + 0.1 * b + 0.01 * np.mean(a)
    b_next = 0.3 + 0.2 * np.cos(np.roll(b, 3)) + 0.1 * a
    return a_next, b_next


def probe(a, b):
    x = np.linspace(1.0, 2.0, N)
    return np.interp([1.25, 1.7], x, a), np.interp([1.25, 1.7], x, b)


def _run(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = owned_rows(N, rank, world)

    def sweep_rows(a, b):
        an, bn = jacobi_map(a, b)
        return an[rows], bn[rows]

    def gather(buf):
        parts = [torch.empty(buf.shape, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(buf)))
        return np.stack([t.numpy() for t in parts])

    loop = ShardedLoop(N, rank, world, sweep_rows, gather, probe)
    res = loop.run(np.ones(N), np.full(N, 0.3), 1e-12, 200, 0.5, check_every=7)
    q.put((rank, res))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _single(check_every=1):
    loop = ShardedLoop(N, 0, 1, lambda a, b: jacobi_map(a, b), lambda buf: buf[None], probe)
    return loop.run(np.ones(N), np.full(N, 0.3), 1e-12, 200, 0.5, check_every=check_every)


@pytest.mark.parametrize("window", [1, 3, 16, 1000])
def test_lazy_stop_test_equals_eager(window):
    """The windowed stop test returns the eager loop's iteration, state and history."""
    a1, b1, n1, c1, h1 = _single(1)
    a2, b2, n2, c2, h2 = _single(window)
    assert (n1, c1) == (n2, c2) and np.array_equal(a1, a2) and np.array_equal(b1, b2)
    assert np.array_equal(h1, h2, equal_nan=True)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_loop_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a1, b1, n1, c1, h1 = _single()
    assert c1 and n1 < 200
    for r in range(world):
        a, b, n, c, h = out[r]
        assert n == n1 and c == c1
        assert np.array_equal(a, a1) and np.array_equal(b, b1)
        assert np.array_equal(h, h1, equal_nan=True)


def test_owned_rows_partition():
    for world in (1, 2, 3, 8):
        allrows = np.sort(np.concatenate([owned_rows(1024, r, world) for r in range(world)]))
        assert np.array_equal(allrows, np.arange(1024))


def test_owned_mus_partition():
    from paper_2012_03667_b200.finite_mu import owned_mus
    mus = [0.4 * (k + 0.5) / 32 for k in range(32)]
    for world in (1, 2, 3, 8):
        parts = [owned_mus(mus, r, world) for r in range(world)]
        assert sorted(m for p_ in parts for m in p_) == sorted(mus)
        assert max(map(len, parts)) - min(map(len, parts)) <= 1
    assert len(owned_mus(mus, 0, 8)) == 4  # BASELINE config 4: 4 mu values per GPU at 8 GPUs


def _run_mu(rank, world, port, q):
    """solve_mu_batch_sharded's partition and all_gather_object over gloo,
    with the GPU solve replaced by a test double (a deterministic fake)."""
    import types

    from paper_2012_03667_b200 import finite_mu
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def fake_batch(mus, params=None, grid=None, device=0, history=False):
        return [types.SimpleNamespace(iterations=int(100 * m) + rank * 0, converged=True,
                                      A=np.full(2, m), B=np.full(2, 2 * m), C=np.full(2, 3 * m)) for m in mus]

    finite_mu.solve_mu_batch = fake_batch
    mus = [0.4 * (k + 0.5) / 32 for k in range(32)]
    recs = finite_mu.solve_mu_batch_sharded(mus, grid=object())
    q.put((rank, [(r[0], r[1], float(r[3][0])) for r in recs]))
    dist.destroy_process_group()


def test_mu_batch_sharded_gathers_in_order():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_mu, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mus = [0.4 * (k + 0.5) / 32 for k in range(32)]
    for r in range(world):
        assert [x[0] for x in out[r]] == mus
        assert all(x[2] == x[0] and x[1] == int(100 * x[0]) for x in out[r])
