"""GPU probe: config-0 time to solution of the pairs kernel per angle-chunk
count (DSE_PAIRS_CHUNKS) next to the fast kernel."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402

prm = p.ModelParams(N=128, m_rad=128, m_ang=64, xi=1e-10, max_iterations=20000)
g = p.build_grid(128, 128, 64, prm.p2_min, prm.p2_max)
cases = [("fast", None)] + [("pairs", c) for c in ("1", "2", "4", "8", "16")]
for ar, c in cases:
    if c is None:
        os.environ.pop("DSE_PAIRS_CHUNKS", None)
    else:
        os.environ["DSE_PAIRS_CHUNKS"] = c
    sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic(ar))
    best = 1e9
    for rep in range(3):
        t0 = time.perf_counter()
        _, _, its, conv, _ = sw.solve(np.ones(128), np.full(128, 0.3))
        best = min(best, time.perf_counter() - t0)
    print(ar, c, its, f"{1e3 * best:.2f} ms", f"{1e6 * best / its:.2f} us/it", flush=True)
    sw.close()
