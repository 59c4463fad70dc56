"""Config-0 device time to solution per arithmetic (solve_device, no history)."""
import json, os, sys
sys.path.insert(0, ".")
import torch
import paper_2012_03667_b200 as p
prm = p.ModelParams(N=128, m_rad=128, m_ang=64, xi=1e-10, max_iterations=20000)
g = p.build_grid(128, 128, 64, prm.p2_min, prm.p2_max)
out = {"lib": os.environ.get("DSE_LIB")}
for ar in ("fast", "exact", "pairs", "moments"):
    sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic(ar))
    A = torch.ones(128, dtype=torch.float64, device="cuda"); B = torch.full((128,), 0.3, dtype=torch.float64, device="cuda")
    sw.solve_device(A.data_ptr(), B.data_ptr(), prm.max_iterations)
    ts = []
    for r in range(3):
        A.fill_(1.0); B.fill_(0.3); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); it, conv = sw.solve_device(A.data_ptr(), B.data_ptr(), prm.max_iterations); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    out[ar] = (round(min(ts), 3), it)
    sw.close()
print(json.dumps(out))
