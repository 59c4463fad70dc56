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
        out = np.zeros((it, 5))
        lib = ctypes.CDLL(os.environ["DSE_LIB"])
        lib.dse_debug_phase_times.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int64]
        assert lib.dse_debug_phase_times(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), it) == 0
        d = np.diff(out, axis=1)[5:]  # skip the first iterations
        total = (out[6:, 0] - out[5:-1, 0])
        print(f"N={n} M={m} K={k} {arith.value}: per iteration {np.median(total)/1e3:.2f} us; "
              f"prologue {np.median(d[:,0])/1e3:.2f}, items {np.median(d[:,1])/1e3:.2f}, "
              f"grid.sync {np.median(d[:,2])/1e3:.2f}, post {np.median(d[:,3])/1e3:.2f} us (block 0)")
