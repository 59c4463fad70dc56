"""GPU probe: does the full in-medium BC vertex converge with a regularised
difference quotient?  Prints the max|dA| trend per eps^2 (DSE_MU_DQ_EPS2)."""
import json
import os
import sys

sys.path.insert(0, ".")
from paper_2012_03667_b200.finite_mu import MuSweeper  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402

for size in (dict(n_s=64, n_4=64, m_s=64, m_4=64, m_ang=16), dict()):
    for eps2 in ("0", "1e-6", "1e-4", "1e-3", "1e-2", "1e-1"):
        os.environ["DSE_MU_DQ_EPS2"] = eps2
        p = MuParams(vertex="bc", max_iterations=150, **size)
        g = grid_for(p)
        with MuSweeper(g, p) as sw:
            try:
                sol = sw.solve(p)
                h = [r.delta_a for r in sol.history[1:]]
                print(json.dumps(dict(size=size or "config3", eps2=eps2, its=sol.iterations, conv=sol.converged,
                                      dA=[f"{x:.1e}" for x in h[:: max(1, len(h) // 10)]],
                                      A0=str(sol.A[0, g.n_4 // 2]), C0=str(sol.C[0, g.n_4 // 2]))), flush=True)
            except Exception as e:  # noqa: BLE001
                print(json.dumps(dict(size=size or "config3", eps2=eps2, error=str(e)[:100])), flush=True)
