"""Config 4 by batched successive approximation (solve_mu_batch_sa): whole
32-solve job timed 3 times; batch 4 and batch 2."""
import sys, time, json
sys.path.insert(0, ".")
import torch
from paper_2012_03667_b200.finite_mu import solve_mu_batch_sa
from paper_2012_03667_b200.mu_grid import MuParams, grid_for
p = MuParams(mode="moments"); g = grid_for(p)
mus = [0.4 * (k + 0.5) / 32 for k in range(32)]
for batch in (4, 2):
    solve_mu_batch_sa(mus[:batch], p, g, batch=batch); torch.cuda.synchronize()
    ts = []
    for r in range(3):
        t0 = time.perf_counter(); bb = solve_mu_batch_sa(mus, p, g, batch=batch); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"batch": batch, "seconds": ts, "iterations": [s.iterations for s in bb],
                      "converged": sum(s.converged for s in bb)}), flush=True)
