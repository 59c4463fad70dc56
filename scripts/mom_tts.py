"""Moments-mode time to solution (config 0, 256^3 substitute): setup wall + device loop; cluster vs grid kernel."""
import json, os, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2012_03667_b200 as p
dev = torch.device("cuda", 0)
cases = {"c0": dict(N=128, m_rad=128, m_ang=64, xi=1e-10, max_iterations=20000),
         "s256": dict(N=256, m_rad=256, m_ang=256, xi=1e-10, max_iterations=2000, relaxation=0.5)}
for mc in ("0",):
    os.environ["DSE_MOM_CLUSTER"] = mc
    for name, kw in cases.items():
        prm = p.ModelParams(**kw)
        g = p.build_grid(prm.N, prm.m_rad, prm.m_ang, prm.p2_min, prm.p2_max)
        p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic.MOMENTS).close()
        res = []
        for r in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic.MOMENTS)
            setup = time.perf_counter() - t0
            A = torch.ones(prm.N, dtype=torch.float64, device=dev)
            B = torch.full((prm.N,), 0.3, dtype=torch.float64, device=dev)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            it, conv = sw.solve_device(A.data_ptr(), B.data_ptr(), prm.max_iterations)
            e1.record()
            torch.cuda.synchronize()
            res.append((setup, e0.elapsed_time(e1) / 1e3, it, conv))
            sw.close()
        print(json.dumps({"cluster_env": mc, "case": name, "runs": res}), flush=True)
