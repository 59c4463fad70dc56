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

    def fake_batch_sa(mus, params=None, grid=None, batch=4, device=0):
        return fake_batch(mus, params, grid, device)
    finite_mu.solve_mu_batch_sa = fake_batch_sa
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


# ---- WindowedStopLoop: the public multi-GPU solve's host loop ---------------
# The device semantics it relies on (dse_sharded_assemble_step + the stop
# flag: history row n written, flag 1 when both deltas < xi, 2 on a non-finite
# sweep with the state left at that sweep's input, every later step a no-op)
# are emulated in numpy here; the kernels themselves are tested on the GPU
# (tests/test_gpu_distributed.py).

class _EmulatedRank:
    def __init__(self, rank, world, gather, xi, relax, nan_at=None, locate=None):
        self.rank, self.world, self.gather, self.xi, self.relax = rank, world, gather, xi, relax
        self.a, self.b = np.ones(N), np.full(N, 0.3)
        self.rows = owned_rows(N, rank, world)
        self.stop, self.hist, self.nan_at, self.bad_row = 0, {}, nan_at, None
        self._locate = locate

    def step(self, n):
        an, bn = jacobi_map(self.a, self.b)
        mine = np.stack([an[self.rows], bn[self.rows]])
        if self.nan_at is not None and n == self.nan_at[0] and self.nan_at[1] in self.rows:
            k = list(self.rows).index(self.nan_at[1])
            mine[0, k] = np.nan
            self.bad_row = self.nan_at[1]
        full = self.gather(mine)  # every rank takes part in every exchange, stopped or not
        if self.stop:
            return
        an, bn = np.empty(N), np.empty(N)
        for r in range(self.world):
            idx = owned_rows(N, r, self.world)
            an[idx], bn[idx] = full[r][0][:idx.size], full[r][1][:idx.size]
        if self.relax != 1.0:
            an = self.relax * an + (1.0 - self.relax) * self.a
            bn = self.relax * bn + (1.0 - self.relax) * self.b
        da, db = np.max(np.abs(an - self.a)), np.max(np.abs(bn - self.b))
        if not (np.isfinite(da) and np.isfinite(db)):
            self.hist[n] = np.array([n, da, db, np.nan, np.nan, np.nan, np.nan])
            self.stop = 2
            return
        self.a, self.b = an, bn
        pa, pb = probe(an, bn)
        self.hist[n] = np.array([n, da, db, *pa, *pb])
        if da < self.xi and db < self.xi:
            self.stop = 1

    def read(self, lo, hi):
        nan = np.full(7, np.nan)
        return np.stack([self.hist.get(k, nan) for k in range(lo, hi + 1)]), self.stop

    def locate(self):
        return self._locate(self.bad_row)


def _run_windowed(rank, world, port, q, window, nan_at):
    from paper_2012_03667_b200.distributed import WindowedStopLoop
    from paper_2012_03667_b200.errors import NumericalFailureError
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    per = -(-N // world)

    def gather(mine):
        buf = np.zeros((2, per))
        buf[:, :mine.shape[1]] = mine
        parts = [torch.empty((2, per), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(buf))
        return [t.numpy() for t in parts]

    def locate(bad_row):
        t = torch.tensor([bad_row if bad_row is not None else 1 << 60, 3, 1], dtype=torch.int64)
        parts = [torch.empty(3, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(parts, t)
        best = min(parts, key=lambda x: int(x[0]))
        return tuple(int(v) for v in best)

    dev = _EmulatedRank(rank, world, gather, 1e-12, 0.5, nan_at, locate)
    loop = WindowedStopLoop(dev.step, dev.read, dev.locate)
    try:
        n, conv = loop.run(1e-12, 200, window)
        h = np.stack([dev.hist[k] for k in range(1, n + 1)])
        q.put((rank, ("ok", n, conv, dev.a, dev.b, h)))
    except NumericalFailureError as exc:
        q.put((rank, ("fail", exc.row, exc.radial, exc.angular, exc.iteration)))
    dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q, *args)) for r in range(world)]
    for p_ in procs:
        p_.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    return out


@pytest.mark.parametrize("window", [1, 5, 16])
def test_windowed_stop_loop_world2_equals_eager_loop(window):
    a1, b1, n1, c1, h1 = _single()
    out = _spawn(_run_windowed, 2, window, None)
    for r in range(2):
        kind, n, conv, a, b, h = out[r]
        assert kind == "ok" and (n, conv) == (n1, c1)
        assert np.array_equal(a, a1) and np.array_equal(b, b1)
        assert np.array_equal(h, h1[1:], equal_nan=True)


def test_windowed_stop_loop_failure_raises_everywhere():
    """A non-finite row on rank 1 at iteration 9: both ranks raise the same
    NumericalFailureError (lowest failing row, iteration 9), whatever the window."""
    out = _spawn(_run_windowed, 2, 4, (9, 5))  # row 5 is owned by rank 1 at world 2
    assert out[0] == out[1] == ("fail", 5, 3, 1, 9)
