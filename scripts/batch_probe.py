"""Batched-solve throughput on config-0-sized grids (uniform scan: all converge)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402

g = p.build_grid(128, 128, 64, 1e-6, 1e4)
v = p.VARIANTS["indexed-gpu"]
for S in (1, 4, 16, 32, 64):
    ds = np.linspace(0.40, 0.50, S)
    plist = [p.ModelParams(N=128, m_rad=128, m_ang=64, D=float(d), xi=1e-10, max_iterations=20000) for d in ds]
    b0s = np.full((S, 128), 0.3)
    p.solve_batch(plist[:1], v, grid=g, b0s=b0s[:1])
    t0 = time.perf_counter()
    sols = p.solve_batch(plist, v, grid=g, b0s=b0s)
    tb = time.perf_counter() - t0
    t0 = time.perf_counter()
    for prm in plist:
        p.solve(prm, v, grid=g, b0=np.full(128, 0.3))
    ts = time.perf_counter() - t0
    its = [s.iterations for s in sols]
    print(f"S={S:3d} batched {tb:.3f}s sequential {ts:.3f}s speedup {ts/tb:.2f}x  iterations {min(its)}..{max(its)} "
          f"converged {sum(s.converged for s in sols)}/{S}  solve-iterations/s {sum(its)/tb:.3g}")
