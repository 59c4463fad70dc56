"""Dump exact-arithmetic sweeps/solves with whichever library DSE_LIB names,
for a bitwise A/B between builds: python scripts/exact_ab.py out.npz"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402

out = {}
rng = np.random.default_rng(11)
import os
v = p.VARIANTS[os.environ.get("DSE_AB_VARIANT", "indexed-gpu-exact")]
for (n, m, k) in ((128, 128, 64), (1024, 1024, 256), (150, 100, 32), (37, 29, 5), (2, 2, 1), (256, 256, 256)):
    g = p.build_grid(n, m, k, 1e-6, 1e4)
    for si, (a, b) in enumerate([(np.ones(n), np.full(n, 0.3)), (rng.uniform(0.8, 2.5, n), rng.uniform(0, 1.6, n)),
                                 (rng.uniform(-3, 3, n), rng.uniform(-2, 2, n))]):
        for pi, prm in enumerate([p.ModelParams(), p.ModelParams(m0=0.004, z1=1.2, D=0.9, omega=0.5)]):
            try:
                x = p.iterate_once(g, a, b, prm, v)
            except p.NumericalFailureError as exc:
                x = (np.array([exc.row, exc.radial, exc.angular], float), np.zeros(1))
            out[f"{n}_{m}_{k}_{si}_{pi}_A"], out[f"{n}_{m}_{k}_{si}_{pi}_B"] = x
# extra random states (DSE_AB_EXTRA=n): wide value ranges, including the
# UV-tail-like tiny B values and a chiral (B = 0) state
extra = int(os.environ.get("DSE_AB_EXTRA", "0"))
if extra:
    g = p.build_grid(1024, 1024, 256, 1e-6, 1e4)
    rng = np.random.default_rng(123)
    for t in range(extra):
        a = rng.uniform(0.5, 3.0, 1024)
        b = rng.uniform(0.0, 2.0, 1024) * 10.0 ** rng.uniform(-250, 0, 1024) if t % 3 else rng.uniform(0, 2, 1024)
        if t == 5:
            b = np.zeros(1024)
        prm = p.ModelParams(D=float(rng.uniform(0.3, 1.0)), omega=float(rng.uniform(0.4, 0.9)),
                            m0=float(rng.choice([0.0, 0.005])))
        try:
            x = p.iterate_once(g, a, b, prm, v)
        except p.NumericalFailureError as exc:
            x = (np.array([exc.row, exc.radial, exc.angular], float), np.zeros(1))
        out[f"x{t}_A"], out[f"x{t}_B"] = x
g = p.build_grid(128, 128, 64, 1e-6, 1e4)
sol = p.solve(p.ModelParams(N=128, m_rad=128, m_ang=64, xi=1e-10, max_iterations=20000), v, grid=g,
              b0=np.full(128, 0.3))
out["c0_A"], out["c0_B"], out["c0_it"] = sol.A, sol.B, np.array(sol.iterations)
np.savez(sys.argv[1], **out)
print("dumped", len(out))
