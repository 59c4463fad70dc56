"""256^3 substitute (relaxation 0.5, 421 iterations): device time to solution, pairs arithmetic,
for the launch shape DSE_PAIRS_LAUNCH_THREADS selects."""
import json, os, sys
sys.path.insert(0, ".")
import torch
import paper_2012_03667_b200 as p
prm = p.ModelParams(N=256, m_rad=256, m_ang=256, xi=1e-10, relaxation=0.5, max_iterations=20000)
g = p.build_grid(256, 256, 256, prm.p2_min, prm.p2_max)
sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic("pairs"))
A = torch.ones(256, dtype=torch.float64, device="cuda"); B = torch.full((256,), 0.3, dtype=torch.float64, device="cuda")
sw.solve_device(A.data_ptr(), B.data_ptr(), prm.max_iterations)
ts = []
for r in range(3):
    A.fill_(1.0); B.fill_(0.3); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); it, conv = sw.solve_device(A.data_ptr(), B.data_ptr(), prm.max_iterations); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(json.dumps({"threads": os.environ.get("DSE_PAIRS_LAUNCH_THREADS"), "ms": round(min(ts), 3), "iterations": it, "layout": sw.layout()}))
