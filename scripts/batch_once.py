import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2012_03667_b200 as p
g = p.build_grid(128, 128, 64, 1e-6, 1e4)
ds = np.linspace(0.40, 0.50, 32)
plist = [p.ModelParams(N=128, m_rad=128, m_ang=64, D=float(d), xi=1e-10, max_iterations=20000) for d in ds]
v = p.VARIANTS[sys.argv[1] if len(sys.argv) > 1 else "indexed-gpu-moments"]
p.solve_batch(plist, v, grid=g, b0s=np.full((32, 128), 0.3))
