"""GPU probe: finite-mu config 3 at full size -- per-iteration time and the
convergence trend of each vertex mode."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2012_03667_b200.finite_mu import MuSweeper  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 40
sizes = [dict(), dict(n_s=64, n_4=64, m_s=64, m_4=64, m_ang=16)]
for kw in sizes:
    for vertex in ("bc1", "bcb", "bc"):
        for relax in (1.0, 0.5):
            p = MuParams(vertex=vertex, max_iterations=cap, relaxation=relax, **kw)
            g = grid_for(p)
            with MuSweeper(g, p) as sw:
                t = time.perf_counter()
                try:
                    sol = sw.solve(p)
                except Exception as e:  # noqa: BLE001
                    print(json.dumps(dict(vertex=vertex, relax=relax, size=kw, error=str(e)[:200])), flush=True)
                    continue
                dt = time.perf_counter() - t
                st = sw.stats()
            h = sol.history
            print(json.dumps(dict(vertex=vertex, relax=relax, size=kw or "config3", its=sol.iterations,
                                  conv=sol.converged, sec=dt, ms_per_it=1e3 * dt / sol.iterations,
                                  evaluated=st["evaluated_points"], nominal=st["nominal_points"],
                                  dA=[f"{r.delta_a:.2e}" for r in h[1::max(1, len(h) // 12)]],
                                  A0=str(sol.A[0, g.n_4 // 2]), B0=str(sol.B[0, g.n_4 // 2]),
                                  C0=str(sol.C[0, g.n_4 // 2]))), flush=True)
