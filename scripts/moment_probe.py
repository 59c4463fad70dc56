"""Moments arithmetic: config 2 per-iteration (L2 flushed) and config 0 solve
loop timings, for A/B builds (DSE_LIB) and ncu."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402

tag = sys.argv[2] if len(sys.argv) > 2 else ""
g = p.build_grid(1024, 1024, 256, 1e-6, 1e4)
prm = p.ModelParams(N=1024, m_rad=1024, m_ang=256, xi=1e-10)
sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic.MOMENTS)
a = torch.ones(1024, dtype=torch.float64, device="cuda")
b = torch.full((1024,), 0.3, dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
ts = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    sw.load_device(a.data_ptr(), b.data_ptr())
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sw.resume(1)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
sw.check()
ts.sort()
g0 = p.build_grid(128, 128, 64, 1e-6, 1e4)
p0 = p.ModelParams(N=128, m_rad=128, m_ang=64, xi=1e-10, max_iterations=20000)
s0 = p.GpuSweeper(g0, p0, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic.MOMENTS)
A = torch.ones(128, dtype=torch.float64, device="cuda")
B = torch.full((128,), 0.3, dtype=torch.float64, device="cuda")
s0.solve_device(A.data_ptr(), B.data_ptr(), 20000)
A.fill_(1.0)
B.fill_(0.3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
it, conv = s0.solve_device(A.data_ptr(), B.data_ptr(), 20000)
e1.record()
torch.cuda.synchronize()
print(f"{tag:>8} config2 ms/iter median {ts[len(ts) // 2]:.4f} min {ts[0]:.4f} | config0 loop {e0.elapsed_time(e1):.2f} ms "
      f"({it} it) | wpr c2 {sw.layout()}")
