"""Sweeper set-up time per arithmetic (config 0 and config 2 grids), warm."""
import os, sys, time
sys.path.insert(0, ".")
import torch
import paper_2012_03667_b200 as p
for (n, m, k) in ((128, 128, 64), (1024, 1024, 256)):
    g = p.build_grid(n, m, k, 1e-6, 1e4)
    prm = p.ModelParams(N=n, m_rad=m, m_ang=k)
    for ar in (p.Arithmetic.MOMENTS, p.Arithmetic.FAST, p.Arithmetic.PAIRS, p.Arithmetic.EXACT):
        for r in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, ar)
            t1 = time.perf_counter()
            sw.close()
            t2 = time.perf_counter()
            print(n, ar.value, r, "create %.2f ms close %.2f ms" % (1e3 * (t1 - t0), 1e3 * (t2 - t1)), flush=True)
