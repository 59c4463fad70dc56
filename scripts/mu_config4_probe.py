import sys, time
sys.path.insert(0, ".")
import torch
from paper_2012_03667_b200.finite_mu import solve_mu_batch_anderson, MuSweeper
from paper_2012_03667_b200.mu_grid import MuParams, grid_for
p = MuParams(mode="moments"); g = grid_for(p)
mus = [0.4 * (k + 0.5) / 32 for k in range(32)]
solve_mu_batch_anderson(mus[:4], p, g); torch.cuda.synchronize()
for r in range(4):
    t0 = time.perf_counter(); bb = solve_mu_batch_anderson(mus, p, g, batch=4); torch.cuda.synchronize()
    print("batched", round(time.perf_counter() - t0, 4), sum(s.iterations for s in bb), flush=True)
t0 = time.perf_counter()
with MuSweeper(g, p) as sw:
    sw.solve(MuParams(mode="moments", max_iterations=1))
    torch.cuda.synchronize(); t1 = time.perf_counter()
print("sweeper+table", round(t1 - t0, 4), "close", round(time.perf_counter() - t1, 4))
