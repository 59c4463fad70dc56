"""GPU probe: device time of one finite-mu iteration at config 3 (state
resident, L2 flushed between steps).  Usage: mu_step_probe.py [vertex] [steps]"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2012_03667_b200.finite_mu import MuSweeper  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402

vertex = sys.argv[1] if len(sys.argv) > 1 else "bcb"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
p = MuParams(vertex=vertex, max_iterations=3)
g = grid_for(p)
dev = torch.device("cuda", 0)
n = g.n_ext
with MuSweeper(g, p) as sw:
    sol = sw.solve(p)  # counts evaluated points; gives a realistic state
    A = torch.from_numpy(sol.A.reshape(-1)).to(dev)
    B = torch.from_numpy(sol.B.reshape(-1)).to(dev)
    C = torch.from_numpy(sol.C.reshape(-1)).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.Stream()
    ts = []
    with torch.cuda.stream(st):
        for i in range(steps + 2):
            sw.load_device(A.data_ptr(), B.data_ptr(), C.data_ptr(), st.cuda_stream)
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            sw.resume(1, st.cuda_stream)
            e1.record(st)
            st.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
    s = sw.stats()
print(json.dumps(dict(vertex=vertex, ms=sorted(ts)[len(ts) // 2], ms_all=ts, **s,
                      nominal_pts_per_s=s["nominal_points"] / (sorted(ts)[len(ts) // 2] / 1e3),
                      evaluated_pts_per_s=s["evaluated_points"] / (sorted(ts)[len(ts) // 2] / 1e3))))
