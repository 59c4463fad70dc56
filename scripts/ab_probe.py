"""A/B timing of library builds: DSE_LIB=<so> python scripts/ab_probe.py <tag>.
Config 2 fast sweep (load + flush + resume(1), median of 30) and the per-sweep
hybrid error against the exact-arithmetic build of the same library."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402

dev = torch.device("cuda", 0)
g = p.build_grid(1024, 1024, 256, 1e-6, 1e4)
prm = p.ModelParams(N=1024, m_rad=1024, m_ang=256, xi=1e-10)
a = torch.ones(1024, dtype=torch.float64, device=dev)
b = torch.full((1024,), 0.3, dtype=torch.float64, device=dev)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream().cuda_stream
out = {}
for arith in (p.Arithmetic.FAST, p.Arithmetic.EXACT):
    sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, arith, 0)
    ts = []
    for i in range(33):
        sw.load_device(a.data_ptr(), b.data_ptr(), s)
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sw.resume(1, s)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    ao, bo = sw.sweep(np.ones(1024), np.full(1024, 0.3))
    out[arith] = (ts[len(ts) // 2], ts[0], ao, bo)
    sw.close()


def hyb(x, r):
    m = np.max(np.abs(r))
    big = np.abs(r) >= 1e-6 * m
    return max(np.max(np.abs(x - r)[big] / np.abs(r)[big]), np.max(np.abs(x - r)[~big]) / m if (~big).any() else 0)


f, e = out[p.Arithmetic.FAST], out[p.Arithmetic.EXACT]
print(f"{sys.argv[1]:>10} fast {f[0]:.4f} ms (min {f[1]:.4f})  exact {e[0]:.4f} ms  "
      f"fast-vs-exact hybrid A {hyb(f[2], e[2]):.2e} B {hyb(f[3], e[3]):.2e}")
