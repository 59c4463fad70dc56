import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402

dev = torch.device("cuda", 0)
g = p.build_grid(1024, 1024, 256, 1e-6, 1e4)
prm = p.ModelParams(N=1024, m_rad=1024, m_ang=256, xi=1e-10)
sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic.FAST, 0)
print("stats", sw.stats())
a = torch.ones(1024, dtype=torch.float64, device=dev)
b = torch.full((1024,), 0.3, dtype=torch.float64, device=dev)
ao, bo = torch.zeros_like(a), torch.zeros_like(b)
s = torch.cuda.current_stream().cuda_stream
ref = sw.sweep(np.ones(1024), np.full(1024, 0.3))
for trial in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sw.sweep_device(a.data_ptr(), b.data_ptr(), ao.data_ptr(), bo.data_ptr(), s)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print("sweep_device wall ms", round((t1 - t0) * 1e3, 3), "match", np.array_equal(ao.cpu().numpy(), ref[0]),
          float(ao[0]), ref[0][0])
    sw.check()
for trial in range(3):
    sw.load_device(a.data_ptr(), b.data_ptr(), s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sw.resume(1, s)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print("resume wall ms", round((t1 - t0) * 1e3, 3))
    sw.check()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
sw.sweep_device(a.data_ptr(), b.data_ptr(), ao.data_ptr(), bo.data_ptr(), s)
e1.record()
torch.cuda.synchronize()
print("event ms", e0.elapsed_time(e1))
