"""GPU probe: one batched moments-mode sweep (S = 2, 4) vs single sweeps."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from dataclasses import replace  # noqa: E402

from paper_2012_03667_b200.finite_mu import MuSweeper  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402

p = MuParams(mode="moments")
g = grid_for(p)
dev = torch.device("cuda", 0)
n = g.n_ext
with MuSweeper(g, p) as sw:
    sw.solve(replace(p, max_iterations=1), history=False)
    for S in (2, 4):
        plist = [replace(p, mu=0.1 + 0.05 * s) for s in range(S)]
        x = torch.cat([torch.full((n,), v, dtype=torch.complex128) for v in (1.0, 0.3, 1.0)]).to(dev).repeat(S, 1)
        y = torch.empty_like(x)
        ts = []
        for r in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sw.batch_sweep(x, y, plist)
            e1.record()
            torch.cuda.synchronize()
            if r >= 1:
                ts.append(e0.elapsed_time(e1))
        print("S", S, "ms", round(float(np.median(ts)), 3), "per solve", round(float(np.median(ts)) / S, 3), flush=True)
