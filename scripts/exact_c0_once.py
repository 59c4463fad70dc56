"""One config-0 solve in the exact arithmetic (device loop) for ncu."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2012_03667_b200 as p
prm = p.ModelParams(N=128, m_rad=128, m_ang=64, xi=1e-10, max_iterations=20000)
g = p.build_grid(128, 128, 64, prm.p2_min, prm.p2_max)
sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic(sys.argv[1] if len(sys.argv) > 1 else "exact"))
A = torch.ones(128, dtype=torch.float64, device="cuda")
B = torch.full((128,), 0.3, dtype=torch.float64, device="cuda")
print(sw.solve_device(A.data_ptr(), B.data_ptr(), prm.max_iterations), sw.layout())
