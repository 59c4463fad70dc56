"""GPU probe: Newton-Krylov settings for the full 'bc' vertex on mid and
config-3 grids (solve_mu_newton)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2012_03667_b200.finite_mu import solve_mu_newton  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402

for size, restart, mr, ls, nmax in [
        (dict(n_s=32, n_4=32, m_s=32, m_4=32, m_ang=16), 60, 4, 0, 20),
        (dict(n_s=64, n_4=64, m_s=64, m_4=64, m_ang=16), 60, 4, 0, 20),
        (dict(n_s=64, n_4=64, m_s=64, m_4=64, m_ang=16), 200, 2, 6, 15),
        (dict(), 300, 2, 6, 12)]:
    prm = MuParams(vertex="bc", mu=0.2, mode="moments", **size)
    g = grid_for(prm)
    t0 = time.time()
    sol, rep = solve_mu_newton(prm, g, restart=restart, max_restarts=mr, line_search=ls, max_newton=nmax)
    print(f"{size or 'config3'} restart={restart} ls={ls}: converged={sol.converged} newton={sol.iterations} "
          f"sweeps={rep.sweeps} {time.time() - t0:.1f}s", flush=True)
    for s in rep.steps:
        print("   step %d  |F| %.3e %.3e %.3e  gmres %d" % s, flush=True)
