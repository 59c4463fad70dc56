"""Debug: batched successive approximation vs standalone (small grid)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2012_03667_b200.finite_mu import MuSweeper, solve_mu, solve_mu_batch_sa
from paper_2012_03667_b200.mu_grid import MuParams, grid_for
from dataclasses import replace

SMALL = dict(n_s=10, n_4=12, m_s=14, m_4=16, m_ang=6)
p = MuParams(vertex="bcb", max_iterations=60, **SMALL)
g = grid_for(p)
mus = [0.02, 0.1433, 0.2667]
one = solve_mu(replace(p, mu=mus[0]), g)
print("standalone", one.iterations, one.converged, [(r.n, r.delta_a) for r in one.history[:6]])
b = solve_mu_batch_sa(mus, p, g, batch=4)
print("batched", b[0].iterations, b[0].converged, [(r.n, r.delta_a) for r in b[0].history[:6]])
# manual: two batch sweeps vs two single sweeps
pm = replace(p, mode="moments")
with MuSweeper(g, pm) as sw:
    n = g.n_ext
    x = torch.cat([torch.full((n,), v, dtype=torch.complex128) for v in (1.0, 0.3, 1.0)]).cuda().repeat(4, 1).contiguous()
    y = torch.empty_like(x)
    pl = [replace(pm, mu=m) for m in mus] + [replace(pm, mu=mus[-1])]
    A, B, C = np.ones((10, 12), complex), np.full((10, 12), 0.3 + 0j), np.ones((10, 12), complex)
    for it in range(3):
        sw.batch_sweep(x, y, pl)
        A, B, C = sw.sweep(A, B, C, pl[0])
        got = y[0].cpu().numpy()
        print(it, np.max(np.abs(got[:n] - A.reshape(-1))), np.max(np.abs(got[n:2*n] - B.reshape(-1))))
        x, y = y, x
