"""Why does a bench step cost more than a back-to-back sweep?  A/B timings."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402

dev = torch.device("cuda", 0)
g = p.build_grid(1024, 1024, 256, 1e-6, 1e4)
prm = p.ModelParams(N=1024, m_rad=1024, m_ang=256, xi=1e-10)
sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic.FAST, 0)
a = torch.ones(1024, dtype=torch.float64, device=dev)
b = torch.full((1024,), 0.3, dtype=torch.float64, device=dev)
ao, bo = torch.empty_like(a), torch.empty_like(b)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream().cuda_stream


def ev_time(pre, fn, n=20):
    ts = []
    for _ in range(3):
        pre()
        fn()
    torch.cuda.synchronize()
    for _ in range(n):
        pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return round(ts[len(ts) // 2], 4), round(ts[0], 4)


nop = lambda: None  # noqa: E731
fl = lambda: flush.fill_(1)  # noqa: E731
load = lambda: sw.load_device(a.data_ptr(), b.data_ptr(), s)  # noqa: E731
print("sweep_device, no flush   ", ev_time(nop, lambda: sw.sweep_device(a.data_ptr(), b.data_ptr(), ao.data_ptr(), bo.data_ptr(), s)))
print("sweep_device, flush      ", ev_time(fl, lambda: sw.sweep_device(a.data_ptr(), b.data_ptr(), ao.data_ptr(), bo.data_ptr(), s)))
print("load+resume, no flush    ", ev_time(load, lambda: sw.resume(1, s)))
print("load+resume, flush       ", ev_time(lambda: (load(), fl()), lambda: sw.resume(1, s)))
print("load+resume x2 (2 iters) ", ev_time(load, lambda: sw.resume(2, s)))
print("load+resume x10 (10 iters)", ev_time(load, lambda: sw.resume(10, s)))
