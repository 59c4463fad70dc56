"""Public-API time to solution (solve(), host arrays, history with the default probes) for config 0 and the 256^3 substitute."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2012_03667_b200 as p
out = {}
for name, kw in {"c0": dict(N=128, m_rad=128, m_ang=64, xi=1e-10, max_iterations=20000),
                 "s256": dict(N=256, m_rad=256, m_ang=256, xi=1e-10, max_iterations=2000, relaxation=0.5)}.items():
    prm = p.ModelParams(**kw)
    g = p.build_grid(prm.N, prm.m_rad, prm.m_ang, prm.p2_min, prm.p2_max)
    for v in ("indexed-gpu", "indexed-gpu-pairs", "indexed-gpu-moments", "indexed-seq"):
        b0 = np.full(prm.N, 0.3)
        p.solve(prm, p.VARIANTS[v], grid=g, b0=b0)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            sol = p.solve(prm, p.VARIANTS[v], grid=g, b0=b0)
            ts.append(time.perf_counter() - t0)
        out[f"{name}/{v}"] = (round(min(ts) * 1e3, 2), sol.iterations)
print(json.dumps(out))
