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
flags = ctypes.c_uint32(0)
assert _native.load().dse_debug_check_flags(ctypes.byref(flags)) == 0
print("CHECK_FLAGS", flags.value)
