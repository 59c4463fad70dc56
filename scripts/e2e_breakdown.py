"""Where the e2e iterate_once time goes at config 2 (pairs): Python API vs the
C call vs the device sweep (no L2 flush, back to back)."""
import json, sys, time, ctypes
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2012_03667_b200 as p
from paper_2012_03667_b200 import _native as nat
g = p.build_grid(1024, 1024, 256, 1e-6, 1e4)
prm = p.ModelParams(N=1024, m_rad=1024, m_ang=256, xi=1e-10)
v = p.VARIANTS["indexed-gpu-pairs"]
a = torch.ones(1024, dtype=torch.float64).pin_memory().numpy()
b = torch.full((1024,), 0.3, dtype=torch.float64).pin_memory().numpy()
for _ in range(5):
    p.iterate_once(g, a, b, prm, v)
sw = p.solver._make_sweeper(g, prm, v)
R = 50
out = {}
t0 = time.perf_counter()
for _ in range(R):
    p.iterate_once(g, a, b, prm, v)
out["iterate_once_ms"] = (time.perf_counter() - t0) / R * 1e3
t0 = time.perf_counter()
for _ in range(R):
    sw.sweep(a, b)
out["sweeper_sweep_ms"] = (time.perf_counter() - t0) / R * 1e3
ao, bo = np.empty(1024), np.empty(1024)
err = nat.DseErr()
fn = nat.sweep_raw()
t0 = time.perf_counter()
for _ in range(R):
    fn(sw.handle, a.ctypes.data, b.ctypes.data, ao.ctypes.data, bo.ctypes.data, ctypes.byref(err))
out["c_call_ms"] = (time.perf_counter() - t0) / R * 1e3
dev = torch.device("cuda", 0)
A = torch.ones(1024, dtype=torch.float64, device=dev)
B = torch.full((1024,), 0.3, dtype=torch.float64, device=dev)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(3):
        sw.load_device(A.data_ptr(), B.data_ptr(), st.cuda_stream); sw.resume(1, st.cuda_stream)
    st.synchronize()
    ev = []
    for _ in range(R):
        sw.load_device(A.data_ptr(), B.data_ptr(), st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); sw.resume(1, st.cuda_stream); e1.record(st)
        ev.append((e0, e1))
    st.synchronize()
out["device_resume_no_flush_ms"] = float(np.median([x.elapsed_time(y) for x, y in ev]))
print(json.dumps(out))
