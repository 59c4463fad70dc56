"""Config-1 interpolation kernel driver for ncu (device-resident arrays)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2012_03667_b200 import _native as nat  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "direct"
cubic = arg.startswith("cubic_")
mode = {"search": nat.BATCH_SEARCH, "direct": nat.BATCH_DIRECT}[arg.replace("cubic_", "")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = 1 << 26
x = np.logspace(-4, 4, 512)
v = 1.0 / (1.0 + x) + 0.1 * np.log1p(x)
q = np.exp(np.random.default_rng(0).uniform(np.log(1e-4), np.log(1e4), n))
dev = torch.device("cuda", 0)
dx, dv, dq = (torch.from_numpy(a).to(dev) for a in (x, v, q))
out = torch.empty(n, dtype=torch.float64, device=dev)
idx = torch.empty(n, dtype=torch.int32, device=dev)
lib = nat.load()
if cubic:
    from paper_2012_03667_b200.interpolation import natural_cubic_coefficients
    dc = torch.from_numpy(natural_cubic_coefficients(x, v)).to(dev)
for _ in range(reps):
    err = nat.DseErr()
    if cubic:
        rc = lib.dse_interp_cubic_batch_device(dx.data_ptr(), dv.data_ptr(), dc.data_ptr(), 512, dq.data_ptr(), n, mode,
                                               out.data_ptr(), idx.data_ptr(), 0, ctypes.byref(err))
    else:
        rc = lib.dse_interp_linear_batch_device(dx.data_ptr(), dv.data_ptr(), 512, dq.data_ptr(), n, mode,
                                                out.data_ptr(), idx.data_ptr(), 0, ctypes.byref(err))
    nat.raise_for(rc, err)
torch.cuda.synchronize()
print("ok", float(out[12345]), int(idx[12345]))
