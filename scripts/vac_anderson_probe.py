"""GPU probe: Anderson acceleration of the vacuum sweep map (config 0 and the
256^3 substitute) vs the reference's successive approximation."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402
from paper_2012_03667_b200 import _native as nat  # noqa: E402


def aa_solve(sw, n, xi, cap, depth, beta, dev):
    lib = nat.load()
    x = torch.cat([torch.ones(n, dtype=torch.float64, device=dev), torch.full((n,), 0.3, dtype=torch.float64, device=dev)])
    send = torch.zeros(2 * n, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    err = nat.DseErr()
    X, F = [], []
    for it in range(1, cap + 1):
        nat.raise_for(lib.dse_solve_load(sw.handle, x[:n].data_ptr(), x[n:].data_ptr(), st, ctypes.byref(err)), err)
        nat.raise_for(lib.dse_sharded_sweep_pack(sw.handle, send.data_ptr(), n, st, ctypes.byref(err)), err)
        f = send - x
        d = torch.stack([f[:n].abs().max(), f[n:].abs().max()]).cpu().numpy()
        if d[0] < xi and d[1] < xi:
            return send.cpu().numpy(), it
        X.append(x.clone())
        F.append(f)
        if len(F) > depth + 1:
            X.pop(0)
            F.pop(0)
        if len(F) == 1:
            x = x + beta * f
            continue
        dF = torch.stack([F[k + 1] - F[k] for k in range(len(F) - 1)], dim=1)
        dX = torch.stack([X[k + 1] - X[k] for k in range(len(X) - 1)], dim=1)
        gram = dF.T @ dF
        gram = gram + (1e-14 * torch.trace(gram) + 1e-300) * torch.eye(gram.shape[0], dtype=torch.float64, device=dev)
        gamma = torch.linalg.solve(gram, dF.T @ f)
        x = x + beta * f - (dX + beta * dF) @ gamma
    return x.cpu().numpy(), cap


dev = torch.device("cuda", 0)
for name, kw, arith in (("config0", dict(N=128, m_rad=128, m_ang=64), p.Arithmetic.FAST),
                        ("sub256", dict(N=256, m_rad=256, m_ang=256, relaxation=0.5), p.Arithmetic.PAIRS)):
    prm = p.ModelParams(xi=1e-10, max_iterations=20000, **kw)
    g = p.build_grid(prm.N, prm.m_rad, prm.m_ang, prm.p2_min, prm.p2_max)
    sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, arith)
    a_sa, b_sa, it_sa, conv, _ = sw.solve(np.ones(prm.N), np.full(prm.N, 0.3))
    for depth in (5, 10, 20):
        aa_solve(sw, prm.N, prm.xi, 3000, depth, 1.0, dev)
        torch.cuda.synchronize()
        t = time.perf_counter()
        x, it = aa_solve(sw, prm.N, prm.xi, 3000, depth, 1.0, dev)
        dt = time.perf_counter() - t
        diff = max(np.max(np.abs(x[:prm.N] - a_sa)), np.max(np.abs(x[prm.N:] - b_sa)))
        print(name, "SA", it_sa, "AA depth", depth, "its", it, f"{1e3 * dt:.1f} ms", f"maxdiff {diff:.2e}", flush=True)
    sw.close()
