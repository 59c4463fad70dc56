"""Python-side cost of iterate_once at config 0 (tiny sweep): cProfile of 300 calls."""
import cProfile, pstats, io, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2012_03667_b200 as p
g = p.build_grid(1024, 1024, 256, 1e-6, 1e4)
prm = p.ModelParams(N=1024, m_rad=1024, m_ang=256, xi=1e-10)
v = p.VARIANTS["indexed-gpu-pairs"]
a, b = np.ones(1024), np.full(1024, 0.3)
for _ in range(5):
    p.iterate_once(g, a, b, prm, v)
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    p.iterate_once(g, a, b, prm, v)
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(15)
print(s.getvalue()[:4000])
