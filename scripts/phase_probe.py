"""Phase timing of the persistent loop (needs build/libdse_timing.so, DSE_TIMING=1)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ["DSE_LIB"] = os.path.abspath("build/libdse_timing.so")
import paper_2012_03667_b200 as p  # noqa: E402
from paper_2012_03667_b200 import _native as nat  # noqa: E402

for arith in (p.Arithmetic.FAST,):
    for (n, m, k, it) in ((128, 128, 64, 200), (1024, 1024, 256, 8)):
        prm = p.ModelParams(N=n, m_rad=m, m_ang=k, xi=1e-14, max_iterations=it)
        g = p.build_grid(n, m, k, prm.p2_min, prm.p2_max)
        sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, arith)
        sw.solve(np.ones(n), np.full(n, 0.3))
        sw.solve(np.ones(n), np.full(n, 0.3))
        out = np.zeros((it, 9))
        lib = ctypes.CDLL(os.environ["DSE_LIB"])
        lib.dse_debug_phase_times.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int64]
        assert lib.dse_debug_phase_times(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), it) == 0
        o = out[5:]
        total = (out[6:, 0] - out[5:-1, 0])
        md = lambda x: np.median(x) / 1e3  # noqa: E731
        print(f"N={n} M={m} K={k} {arith.value}: per iteration {md(total):.2f} us; "
              f"prologue {md(o[:,1]-o[:,0]):.2f}, items {md(o[:,2]-o[:,1]):.2f} "
              f"[first item: begin {md(o[:,5]-o[:,1]):.2f}, leaves {md(o[:,6]-o[:,5]):.2f}, "
              f"barrier {md(o[:,7]-o[:,6]):.2f}, finish {md(o[:,8]-o[:,7]):.2f}], "
              f"grid.sync {md(o[:,3]-o[:,2]):.2f}, post {md(o[:,4]-o[:,3]):.2f} us (block 0)")
