"""One config-4 group (4 mu values, batch 4) by solve_mu_batch_sa: ms per sweep."""
import sys, time, json, os
sys.path.insert(0, ".")
import torch
from paper_2012_03667_b200.finite_mu import solve_mu_batch_sa
from paper_2012_03667_b200.mu_grid import MuParams, grid_for
p = MuParams(mode="moments"); g = grid_for(p)
mus = [0.4 * (k + 0.5) / 32 for k in range(32)][12:16]
solve_mu_batch_sa(mus, p, g, batch=4); torch.cuda.synchronize()
ts = []
for r in range(3):
    t0 = time.perf_counter(); bb = solve_mu_batch_sa(mus, p, g, batch=4); torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
it = max(s.iterations for s in bb)
print(json.dumps({"lib": os.environ.get("DSE_LIB"), "ms_per_sweep": 1e3 * min(ts) / it, "s": ts, "its": it}))
