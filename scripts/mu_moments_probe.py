"""GPU probe: one config-3 iteration in moments mode (table built first)."""
import sys

import torch

sys.path.insert(0, ".")
from dataclasses import replace  # noqa: E402

from paper_2012_03667_b200.finite_mu import MuSweeper  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402

p = MuParams(mode="moments", max_iterations=2)
g = grid_for(p)
dev = torch.device("cuda", 0)
with MuSweeper(g, p) as sw:
    sol = sw.solve(p)
    A = torch.from_numpy(sol.A.reshape(-1)).to(dev)
    B = torch.from_numpy(sol.B.reshape(-1)).to(dev)
    C = torch.from_numpy(sol.C.reshape(-1)).to(dev)
    st = torch.cuda.Stream()
    for _ in range(3):
        sw.load_device(A.data_ptr(), B.data_ptr(), C.data_ptr(), st.cuda_stream)
        sw.resume(1, st.cuda_stream)
    st.synchronize()
print("ok")
