"""Break down one row-sharded step (torchrun, 1..N ranks) with CUDA events."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402
from paper_2012_03667_b200 import distributed as D  # noqa: E402

dist.init_process_group("nccl")
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
g = p.build_grid(1024, 1024, 256, 1e-6, 1e4)
prm = p.ModelParams(N=1024, m_rad=1024, m_ang=256, xi=1e-10)
v = p.VARIANTS["indexed-gpu"].with_gpus(dist.get_world_size())
sw, dev, rank, world, sweep_rows, gather, probe_fn, _ = D._device_loop(g, prm, v)
loop = D.ShardedLoop(g.n_ext, rank, world, sweep_rows, gather, probe_fn(()), xp=torch)
a = torch.ones(1024, dtype=torch.float64, device=dev)
b = torch.full((1024,), 0.3, dtype=torch.float64, device=dev)


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


out = {}
out["sweep_rows"] = timed(lambda: sweep_rows(a, b))
ar, br = sweep_rows(a, b)
out["assemble"] = timed(lambda: loop._assemble(ar, br))
out["full_step"] = timed(lambda: loop.sweep(a, b))
if rank == 0:
    print({k: round(v, 4) for k, v in out.items()})
dist.destroy_process_group()
