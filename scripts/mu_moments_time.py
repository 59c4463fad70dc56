"""GPU probe: median device time of one config-3 iteration in moments mode."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2012_03667_b200.finite_mu import MuSweeper  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
p = MuParams(mode="moments", max_iterations=3)
g = grid_for(p)
dev = torch.device("cuda", 0)
with MuSweeper(g, p) as sw:
    sol = sw.solve(p)
    A, B, C = (torch.from_numpy(x.reshape(-1)).to(dev) for x in (sol.A, sol.B, sol.C))
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
print(round(float(np.median(ts)), 3))
