"""GPU probe: where the batched-Anderson config-4 time goes (kernel vs host
algebra).  Prints the wall time of one group of 4 solves, the number of
sweeps, and the torch profiler's top CUDA/CPU ops."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2012_03667_b200.finite_mu import solve_mu_batch_anderson  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402

p = MuParams(mode="moments")
g = grid_for(p)
mus = [0.05, 0.1, 0.15, 0.2]
solve_mu_batch_anderson(mus, p, g)  # warm-up (table build, cuBLAS/cuSOLVER handles)
torch.cuda.synchronize()
t0 = time.perf_counter()
sols = solve_mu_batch_anderson(mus, p, g)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
its = max(s.iterations for s in sols)
print(f"wall {wall:.4f} s, sweeps {its}, per sweep {1e3 * wall / its:.3f} ms")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    solve_mu_batch_anderson(mus, p, g)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
