"""Config-1 interpolation: device time per mode for the current build
(DSE_INTERP_REP / DSE_INTERP_THREADS from the environment), HBM fraction."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2012_03667_b200 import _native as nat  # noqa: E402
from paper_2012_03667_b200.interpolation import natural_cubic_coefficients  # noqa: E402

n = 1 << 26
x = np.logspace(-4, 4, 512)
v = 1.0 / (1.0 + x) + 0.1 * np.log1p(x)
q = np.exp(np.random.default_rng(0).uniform(np.log(1e-4), np.log(1e4), n))
dev = torch.device("cuda", 0)
dx, dv, dq = (torch.from_numpy(a).to(dev) for a in (x, v, q))
dc = torch.from_numpy(natural_cubic_coefficients(x, v)).to(dev)
out = torch.empty(n, dtype=torch.float64, device=dev)
idx = torch.empty(n, dtype=torch.int32, device=dev)
lib = nat.load()
hbm = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6550.0
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}
for cubic in (False, True):
    for mode, mname in ((nat.BATCH_DIRECT, "direct"), (nat.BATCH_SEARCH, "search")):
        ts = []
        for rep in range(6):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            err = nat.DseErr()
            e0.record()
            if cubic:
                rc = lib.dse_interp_cubic_batch_device(dx.data_ptr(), dv.data_ptr(), dc.data_ptr(), 512, dq.data_ptr(),
                                                       n, mode, out.data_ptr(), idx.data_ptr(), 0, ctypes.byref(err))
            else:
                rc = lib.dse_interp_linear_batch_device(dx.data_ptr(), dv.data_ptr(), 512, dq.data_ptr(), n, mode,
                                                        out.data_ptr(), idx.data_ptr(), 0, ctypes.byref(err))
            e1.record()
            nat.raise_for(rc, err)
            torch.cuda.synchronize()
            if rep:
                ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts)) / 1e3
        name = ("cubic_" if cubic else "linear_") + mname
        res[name] = {"ms": 1e3 * t, "hbm_frac": 20.0 * n / t / 1e9 / hbm, "gq_s": n / t / 1e9}
print(json.dumps({"rep": os.environ.get("DSE_INTERP_REP", "auto"), "threads": os.environ.get("DSE_INTERP_THREADS", "auto"),
                  **res}))
