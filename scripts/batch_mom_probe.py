"""The bench's 32-solve D scan on the config-0 grid: fast vs moments variant through solve_batch."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2012_03667_b200 as p
g = p.build_grid(128, 128, 64, 1e-6, 1e4)
ds = np.linspace(0.40, 0.50, 32)
plist = [p.ModelParams(N=128, m_rad=128, m_ang=64, D=float(d), xi=1e-10, max_iterations=20000) for d in ds]
b0s = np.full((32, 128), 0.3)
out = {}
ref = None
for name in ("indexed-gpu", "indexed-gpu-moments", "indexed-gpu-pairs"):
    v = p.VARIANTS[name]
    p.solve_batch(plist[:2], v, grid=g, b0s=b0s[:2])
    ts = []
    for r in range(2):
        t0 = time.perf_counter()
        sols = p.solve_batch(plist, v, grid=g, b0s=b0s)
        ts.append(time.perf_counter() - t0)
    its = [s.iterations for s in sols]
    if ref is None:
        ref = sols
    dev = max(float(np.max(np.abs(s.A - r.A) / np.abs(r.A))) for s, r in zip(sols, ref))
    out[name] = {"seconds": ts, "iterations_equal_fast": its == [s.iterations for s in ref], "max_rel_vs_fast": dev}
print(json.dumps(out))
