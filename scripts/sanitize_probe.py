"""Small end-to-end exercise of every kernel for compute-sanitizer."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import paper_2012_03667_b200 as p  # noqa: E402
from paper_2012_03667_b200 import _native  # noqa: E402

g = p.build_grid(37, 29, 5, 1e-4, 1e3)
prm = p.ModelParams(N=37, m_rad=29, m_ang=5, xi=1e-8, max_iterations=40, relaxation=0.8)
for v in ("indexed-gpu", "search-gpu-exact"):
    sol = p.solve(prm, p.VARIANTS[v], grid=g, b0=np.full(37, 0.3))
    a, b = p.iterate_once(g, sol.A, sol.B, prm, p.VARIANTS[v])
g2 = p.build_grid(64, 128, 64, 1e-6, 1e4)
p.iterate_once(g2, np.ones(64), np.full(64, 0.3), p.ModelParams(), p.VARIANTS["indexed-gpu"])
p.solve_batch([prm, prm], p.VARIANTS["indexed-gpu"], grid=g)
aq = p.interp_indexed_many(g, sol.A)
p.row_rhs(g.p2_ext[3], sol.A[3], sol.B[3], aq, p.interp_indexed_many(g, sol.B), g, prm, row=3)
x = np.logspace(-4, 4, 512)
q = np.exp(np.random.default_rng(0).uniform(np.log(1e-4), np.log(1e4), 10001))
for mode in ("search", "direct"):
    p.interp_linear_batch(x, 1.0 / (1.0 + x), q, mode=mode, with_index=True, counter=p.ComparisonCounter())
_native.debug_pairwise_sum(np.random.default_rng(1).standard_normal((3, 16, 8)), chunk_leaves=1)
a0 = np.ones(20)
a0[7] = np.nan
try:
    p.iterate_once(p.build_grid(20, 16, 8, 1e-6, 1e4), a0, np.ones(20), p.ModelParams(), p.VARIANTS["indexed-gpu"])
except p.NumericalFailureError as exc:
    print("expected failure", exc.row, exc.radial, exc.angular)
print("sanitize probe done")
