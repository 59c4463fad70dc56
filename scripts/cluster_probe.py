"""Config-0 time to solution with and without the 2-CTA cluster layout (env DSE_NO_CLUSTER)."""
import os
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2012_03667_b200 as p

prm = p.ModelParams(N=128, m_rad=128, m_ang=64, xi=1e-10, max_iterations=20000)
g = p.build_grid(128, 128, 64, prm.p2_min, prm.p2_max)
for ar in (p.Arithmetic.FAST, p.Arithmetic.EXACT, p.Arithmetic.PAIRS):
    sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, ar)
    A = torch.ones(128, dtype=torch.float64, device="cuda")
    B = torch.full((128,), 0.3, dtype=torch.float64, device="cuda")
    sw.solve_device(A.data_ptr(), B.data_ptr(), prm.max_iterations)
    best = 1e9
    for _ in range(3):
        A.fill_(1.0); B.fill_(0.3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it, conv = sw.solve_device(A.data_ptr(), B.data_ptr(), prm.max_iterations)
        best = min(best, time.perf_counter() - t0)
    print(os.environ.get("DSE_NO_CLUSTER", "-"), ar.value, it, conv, f"{best*1e3:.2f} ms", sw.layout())
    sw.close()
