"""GPU probe: where the e2e (iterate_once with host arrays) time goes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402
from paper_2012_03667_b200 import _native as nat  # noqa: E402
from paper_2012_03667_b200.solver import _make_sweeper  # noqa: E402

g = p.build_grid(1024, 1024, 256, 1e-6, 1e4)
prm = p.ModelParams(N=1024, m_rad=1024, m_ang=256, xi=1e-10)
v = p.VARIANTS["indexed-gpu-pairs"]
a = torch.ones(1024, dtype=torch.float64).pin_memory().numpy()
b = torch.full((1024,), 0.3, dtype=torch.float64).pin_memory().numpy()
for _ in range(5):
    p.iterate_once(g, a, b, prm, v)
n = 200
t = time.perf_counter()
for _ in range(n):
    p.iterate_once(g, a, b, prm, v)
t_api = (time.perf_counter() - t) / n
sw = _make_sweeper(g, prm, v)
ao, bo = np.empty(1024), np.empty(1024)
err = nat.DseErr()
fn = nat.sweep_raw()
import ctypes  # noqa: E402
t = time.perf_counter()
for _ in range(n):
    fn(sw.handle, a.ctypes.data, b.ctypes.data, ao.ctypes.data, bo.ctypes.data, ctypes.byref(err))
t_raw = (time.perf_counter() - t) / n
t = time.perf_counter()
for _ in range(n):
    _make_sweeper(g, prm, v)
t_lookup = (time.perf_counter() - t) / n
print(f"api {1e6 * t_api:.1f} us  raw C call {1e6 * t_raw:.1f} us  sweeper lookup {1e6 * t_lookup:.1f} us")
