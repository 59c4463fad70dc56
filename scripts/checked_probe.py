"""Run every kernel path on the bounds-checked build and report the flags.
Usage: DSE_LIB=build/libdse_checked.so python scripts/checked_probe.py"""
import ctypes
import os
import runpy
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402
from paper_2012_03667_b200 import _native  # noqa: E402

assert os.environ.get("DSE_LIB", "").endswith("libdse_checked.so")
runpy.run_path("scripts/sanitize_probe.py")
for (n, m, k) in ((128, 128, 64), (1024, 1024, 256), (150, 100, 32), (37, 29, 5), (2, 2, 1)):
    g = p.build_grid(n, m, k, 1e-6, 1e4)
    prm = p.ModelParams(N=n, m_rad=m, m_ang=k, xi=1e-10, max_iterations=3)
    for v in ("indexed-gpu", "search-gpu-exact"):
        p.solve(prm, p.VARIANTS[v], grid=g, b0=np.full(n, 0.3))
os.environ["DSE_SPLIT_ROWS"] = "-1"
os.environ["DSE_CHUNK_LEAVES"] = "32"
p.solve_batch([p.ModelParams(N=64, m_rad=96, m_ang=64, max_iterations=3)] * 2, p.VARIANTS["indexed-gpu"])
p.iterate_once(p.build_grid(300, 200, 64, 1e-6, 1e4), np.ones(300), np.full(300, 0.3),
               p.ModelParams(), p.VARIANTS["indexed-gpu"])
# pairs arithmetic (dynamic items, angle chunks at small sizes, sharded rows)
for (n, m, k) in ((128, 128, 64), (300, 200, 64), (37, 29, 5), (2, 2, 1)):
    g = p.build_grid(n, m, k, 1e-6, 1e4)
    prm = p.ModelParams(N=n, m_rad=m, m_ang=k, xi=1e-10, max_iterations=3)
    p.solve(prm, p.VARIANTS["indexed-gpu-pairs"], grid=g, b0=np.full(n, 0.3))
    sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic.PAIRS, rows=(1 % n, 2))
    sw.sweep(np.ones(n), np.full(n, 0.3))
    sw.close()
# finite mu: direct and moments mode, all vertices, a sharded sweeper
from paper_2012_03667_b200.finite_mu import MuSweeper, solve_mu  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402
for dims in (dict(n_s=10, n_4=12, m_s=14, m_4=16, m_ang=6), dict(n_s=2, n_4=2, m_s=2, m_4=2, m_ang=1),
             dict(n_s=32, n_4=32, m_s=48, m_4=40, m_ang=8)):
    for vertex in ("bcb", "bc1", "bc"):
        for mode in ("direct", "moments"):
            mp = MuParams(vertex=vertex, mode=mode, max_iterations=3, **dims)
            solve_mu(mp, grid_for(mp))
    mp = MuParams(max_iterations=3, **dims)
    with MuSweeper(grid_for(mp), mp, row_start=0, row_stride=3) as sw:
        sw.sweep(np.ones((mp.n_s, mp.n_4)), np.full((mp.n_s, mp.n_4), 0.3), np.ones((mp.n_s, mp.n_4)))
# batched finite-mu sweeps (moments mode), S = 2 and 4
from paper_2012_03667_b200.finite_mu import solve_mu_batch_anderson  # noqa: E402
for bsz in (2, 4):
    mp = MuParams(max_iterations=3, mode="moments", n_s=10, n_4=12, m_s=14, m_4=16, m_ang=6)
    solve_mu_batch_anderson([0.1, 0.2, 0.3], mp, grid_for(mp), batch=bsz)
flags = ctypes.c_uint32(0)
assert _native.load().dse_debug_check_flags(ctypes.byref(flags)) == 0
print("CHECK_FLAGS", flags.value)
