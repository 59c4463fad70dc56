"""torchrun check (tests/test_gpu_distributed.py, needs >= 2 GPUs): the
public multi-GPU solve and iterate_once with gpus = WORLD equal the
single-GPU results bitwise on every rank."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_03667_b200 as p  # noqa: E402
from paper_2012_03667_b200.distributed import close_solvers  # noqa: E402

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
os.environ["DSE_DEVICE"] = str(local)
dist.init_process_group("nccl")
world = dist.get_world_size()
for n, m, k, relax in ((256, 256, 256, 0.5), (128, 128, 64, 1.0)):
    prm = p.ModelParams(N=n, m_rad=m, m_ang=k, xi=1e-10, relaxation=relax, max_iterations=5000)
    g = p.build_grid(n, m, k, prm.p2_min, prm.p2_max)
    b0 = np.full(n, 0.3)
    for vname in ("indexed-gpu-pairs", "indexed-seq"):
        ref = p.solve(prm, p.VARIANTS[vname], grid=g, b0=b0)
        sol = p.solve(prm, p.VARIANTS[vname].with_gpus(world), grid=g, b0=b0)
        assert sol.iterations == ref.iterations and sol.converged == ref.converged, (vname, sol.iterations)
        assert np.array_equal(sol.A, ref.A) and np.array_equal(sol.B, ref.B), vname
        rng = np.random.default_rng(3)
        a, b = rng.uniform(1, 2, n), rng.uniform(0, 1, n)
        x = p.iterate_once(g, a, b, prm, p.VARIANTS[vname].with_gpus(world))
        y = p.iterate_once(g, a, b, prm, p.VARIANTS[vname])
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1]), vname
close_solvers()
dist.barrier()
if dist.get_rank() == 0:
    print("dist_solve_check ok", world)
dist.destroy_process_group()
