"""GPU probe: finite-mu sweep outputs (direct and moments mode, every vertex,
a batched S = 4 sweep) of the current build saved to an npz, so that two
builds can be compared bitwise.  Usage: mu_bitwise_probe.py out.npz"""
import sys
from dataclasses import replace

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2012_03667_b200.finite_mu import MuSweeper, iterate_mu_once  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402

SMALL = dict(n_s=10, n_4=12, m_s=14, m_4=16, m_ang=6)
rng = np.random.default_rng(3)
out = {}
for vertex in ("bcb", "bc1", "bc"):
    p = MuParams(mu=0.2, vertex=vertex, **SMALL)
    g = grid_for(p)
    shape = (g.n_s, g.n_4)
    A = 1.0 + 0.8 * rng.random(shape) + 0.1j * rng.standard_normal(shape)
    B = 0.1 + 0.5 * rng.random(shape) + 0.05j * rng.standard_normal(shape)
    C = 1.0 + 0.8 * rng.random(shape) + 0.1j * rng.standard_normal(shape)
    for mode in ("direct", "moments"):
        r = iterate_mu_once(g, A, B, C, replace(p, mode=mode))
        for k, x in zip("ABC", r):
            out[f"{vertex}_{mode}_{k}"] = x
p = MuParams(mode="moments", **SMALL)
g = grid_for(p)
n = g.n_ext
with MuSweeper(g, p) as sw:
    plist = [replace(p, mu=0.1 + 0.05 * s, interaction_D=0.5 + 0.1 * s) if hasattr(p, "interaction_D")
             else replace(p, mu=0.1 + 0.05 * s) for s in range(4)]
    x = torch.from_numpy(1.0 + 0.3 * rng.random((4, 3 * n)) + 0.05j * rng.standard_normal((4, 3 * n))).cuda()
    y = torch.empty_like(x)
    sw.batch_sweep(x, y, plist)
    torch.cuda.synchronize()
    out["batch"] = y.cpu().numpy()
np.savez(sys.argv[1], **out)
print("saved", len(out))
