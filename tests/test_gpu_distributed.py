"""GPU: the NCCL row-sharded solve (distributed.py) on one rank equals the
single-GPU solve bitwise (real NCCL all-gather, real sharded sweeper).  The
multi-rank host logic is covered by tests/test_distributed.py (gloo)."""
import os
import socket

import numpy as np
import pytest

import paper_2012_03667_b200 as p
from conftest import golden, golden_grid, params_ns

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_world1():
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0", WORLD_SIZE="1",
                      LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


def test_sharded_solve_world1_bitwise(nccl_world1):
    z = golden("solve_default.npz")
    g = golden_grid("default")
    prm = params_ns(xi=0.005, max_iterations=500)
    ref = p.solve(prm, p.VARIANTS["indexed-gpu"], grid=g)
    sol = p.solve(prm, p.VARIANTS["indexed-gpu"].with_gpus(1), grid=g)  # gpus=1 -> single GPU
    from paper_2012_03667_b200.distributed import solve_sharded
    a, b, n, conv, hist = solve_sharded(g, prm, p.VARIANTS["indexed-gpu"].with_gpus(1), np.ones(g.n_ext),
                                        np.ones(g.n_ext), tuple(10.0 ** (2.0 * lp) for lp in (-2.5, 0.0)))
    assert n == ref.iterations == sol.iterations == int(z["iterations"]) and conv
    assert np.array_equal(a, ref.A) and np.array_equal(b, ref.B)
    h_ref = np.array([[r.iteration, r.max_delta_a, r.max_delta_b, *r.probe_a, *r.probe_b] for r in ref.history])
    assert np.array_equal(hist, h_ref, equal_nan=True)


def test_sharded_sweep_world1_bitwise(nccl_world1):
    g = golden_grid("c0")
    rng = np.random.default_rng(5)
    a, b = rng.uniform(1, 2, g.n_ext), rng.uniform(0, 1, g.n_ext)
    from paper_2012_03667_b200.distributed import iterate_once_sharded
    x = iterate_once_sharded(g, a, b, params_ns(), p.VARIANTS["indexed-gpu"].with_gpus(1))
    y = p.iterate_once(g, a, b, params_ns(), p.VARIANTS["indexed-gpu"])
    assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])



def _device_to_host(ptr, n):
    from cuda.bindings import runtime as cudart  # cuda-python: a raw device pointer -> host
    out = np.empty(n)
    err, = cudart.cudaMemcpy(out.ctypes.data, ptr, n * 8, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    assert int(err) == 0, err
    return out


@pytest.mark.parametrize("world,relax", [(1, 1.0), (3, 1.0), (4, 0.5)])
def test_fused_sharded_step_equals_sweep(world, relax):
    """FusedShardedStep's device steps (sweep+pack | all-gather | assemble)
    reproduce the single-GPU sweep + blend + deltas bitwise.  The W ranks run
    one after another on one GPU (no kernel waits on another); the
    all-gather is the stack of their send buffers."""
    import ctypes

    import torch

    from paper_2012_03667_b200 import _native as nat
    from paper_2012_03667_b200.distributed import FusedShardedStep
    g = golden_grid("default")
    prm = params_ns()
    rng = np.random.default_rng(5)
    a, b = rng.uniform(1, 2, g.n_ext), rng.uniform(0.1, 1, g.n_ext)
    ref_a, ref_b = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic.PAIRS).sweep(a, b)
    if relax != 1.0:
        ref_a = relax * ref_a + (1.0 - relax) * a
        ref_b = relax * ref_b + (1.0 - relax) * b
    dev = torch.device("cuda", 0)
    ta, tb = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    sws = [p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic.PAIRS, 0, rows=(r, world))
           for r in range(world)]
    steps = [FusedShardedStep(sw, g.n_ext, world, dev, None, relax) for sw in sws]
    sp = torch.cuda.current_stream(dev).cuda_stream
    lib = nat.load()
    for st in steps:
        st.load(ta, tb, sp)
    for st in steps:  # every rank sweeps and packs its rows
        err = nat.DseErr()
        nat.raise_for(lib.dse_sharded_sweep_pack(st.sw.handle, st.send.data_ptr(), st.per, sp,
                                                 ctypes.byref(err)), err)
    recv = torch.stack([st.send for st in steps])
    for st in steps:  # every rank assembles the same full state
        err = nat.DseErr()
        nat.raise_for(lib.dse_sharded_assemble(st.sw.handle, recv.data_ptr(), world, st.per, relax,
                                               st.delta.data_ptr(), sp, ctypes.byref(err)), err)
    torch.cuda.synchronize()
    for st in steps:
        out_a = _device_to_host(st.state_ptrs[0], g.n_ext)
        out_b = _device_to_host(st.state_ptrs[1], g.n_ext)
        assert np.array_equal(out_a, ref_a) and np.array_equal(out_b, ref_b)
        d = st.delta.cpu().numpy()
        assert d[0] == np.max(np.abs(ref_a - a)) and d[1] == np.max(np.abs(ref_b - b))
    for sw in sws:
        sw.close()


@pytest.mark.parametrize("relax", [1.0, 0.5])
def test_p2p_step_world1_equals_sweep(relax):
    """P2PShardedStep at world 1 (the peer is this GPU: the push, the flag
    barrier and the assemble all run; multi-GPU is correct by construction,
    one GPU per test box) equals the sweep + blend + deltas bitwise, twice
    in a row (the barrier epochs advance)."""
    import torch

    from paper_2012_03667_b200.distributed import P2PShardedStep, device_view
    g = golden_grid("default")
    prm = params_ns()
    rng = np.random.default_rng(9)
    a, b = rng.uniform(1, 2, g.n_ext), rng.uniform(0.1, 1, g.n_ext)
    dev = torch.device("cuda", 0)
    sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic.PAIRS, 0)
    step = P2PShardedStep(sw, g.n_ext, 1, 0, 0, dev, lambda obj: [obj], relax)
    sp = torch.cuda.current_stream(dev).cuda_stream
    from paper_2012_03667_b200.distributed import FusedShardedStep
    ptrs = FusedShardedStep(sw, g.n_ext, 1, dev, None).state_ptrs
    state_a, state_b = a, b
    step.load(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), sp)
    for _ in range(2):
        ra, rb = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic.PAIRS).sweep(state_a, state_b)
        if relax != 1.0:
            ra = relax * ra + (1.0 - relax) * state_a
            rb = relax * rb + (1.0 - relax) * state_b
        d = step.step(sp).cpu().numpy()
        torch.cuda.synchronize()
        ga = device_view(ptrs[0], g.n_ext, dev).cpu().numpy()
        gb = device_view(ptrs[1], g.n_ext, dev).cpu().numpy()
        assert int(step.timed_out.item()) == 0
        assert np.array_equal(ga, ra) and np.array_equal(gb, rb)
        assert d[0] == np.max(np.abs(ra - state_a)) and d[1] == np.max(np.abs(rb - state_b))
        state_a, state_b = ra, rb
    step.close()
    sw.close()


@pytest.mark.parametrize("vname", ["indexed-gpu-pairs", "indexed-seq"])
def test_public_sharded_solve_world1_stops_exactly(nccl_world1, vname):
    """The public multi-GPU solve (ShardedSolver: the selected step with
    history row and stop flag on the device, a 16-iteration host window)
    equals the single-GPU solve bitwise -- state, iteration count, history --
    so the iterations queued past convergence inside the window changed
    nothing (they are device no-ops).  Relaxation 0.5 on the 256^3 grid."""
    z = golden("solve_sub256.npz")
    g = golden_grid("sub256")
    prm = params_ns(xi=1e-10, relaxation=0.5, max_iterations=2000)
    b0 = np.full(g.n_ext, 0.3)
    ref = p.solve(prm, p.VARIANTS[vname], grid=g, b0=b0)
    from paper_2012_03667_b200.distributed import close_solvers, solve_sharded
    a, b, n, conv, hist = solve_sharded(g, prm, p.VARIANTS[vname].with_gpus(1), np.ones(g.n_ext), b0,
                                        tuple(10.0 ** (2.0 * lp) for lp in (-2.5, 0.0)))
    assert conv and n == ref.iterations == int(z["iterations"])
    assert np.array_equal(a, ref.A) and np.array_equal(b, ref.B)
    h_ref = np.array([[r.iteration, r.max_delta_a, r.max_delta_b, *r.probe_a, *r.probe_b] for r in ref.history])
    assert np.array_equal(hist, h_ref, equal_nan=True)
    close_solvers()


def test_public_sharded_failure_matches_single_gpu(nccl_world1):
    """A non-finite sweep inside the sharded solve raises the reference's
    NumericalFailureError with the single-GPU solve's (iteration, row,
    radial, angular)."""
    g = golden_grid("small")
    prm = params_ns(xi=1e-3, max_iterations=50)
    a0 = np.ones(g.n_ext)
    a0[5] = np.inf
    with pytest.raises(p.NumericalFailureError) as ref:
        p.solve(prm, p.VARIANTS["indexed-gpu-pairs"], grid=g, a0=a0)
    from paper_2012_03667_b200.distributed import close_solvers, iterate_once_sharded, solve_sharded
    with pytest.raises(p.NumericalFailureError) as got:
        solve_sharded(g, prm, p.VARIANTS["indexed-gpu-pairs"].with_gpus(1), a0, np.ones(g.n_ext), ())
    assert (got.value.iteration, got.value.row, got.value.radial, got.value.angular) == \
        (ref.value.iteration, ref.value.row, ref.value.radial, ref.value.angular)
    with pytest.raises(p.NumericalFailureError) as ref1:
        p.iterate_once(g, a0, np.ones(g.n_ext), prm, p.VARIANTS["indexed-gpu-pairs"])
    with pytest.raises(p.NumericalFailureError) as got1:
        iterate_once_sharded(g, a0, np.ones(g.n_ext), prm, p.VARIANTS["indexed-gpu-pairs"].with_gpus(1))
    assert (got1.value.row, got1.value.radial, got1.value.angular) == \
        (ref1.value.row, ref1.value.radial, ref1.value.angular)
    close_solvers()


def test_torchrun_world2_public_solve_bitwise(tmp_path):
    """W = 2 under torchrun (needs two GPUs: skipped on a one-GPU box): the
    public solve / iterate_once with gpus=2 equal the single-GPU results
    bitwise, through the peer-memory step and through the NCCL step."""
    import subprocess
    import sys

    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p2p in ("1", "0"):
        env = dict(os.environ, DSE_P2P=p2p, PYTHONPATH=root)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()),
               os.path.join(root, "scripts", "dist_solve_check.py")]
        res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-3000:]
        assert "dist_solve_check ok" in res.stdout
