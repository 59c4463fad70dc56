"""Config-2 per-iteration device time of one arithmetic (default exact) with
whichever library DSE_LIB names: python scripts/exact_time.py [arith]"""
import json, os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2012_03667_b200 as p
arith = p.Arithmetic(sys.argv[1] if len(sys.argv) > 1 else "exact")
dev = torch.device("cuda", 0)
g = p.build_grid(1024, 1024, 256, 1e-6, 1e4)
prm = p.ModelParams(N=1024, m_rad=1024, m_ang=256, xi=1e-10)
sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, arith, 0)
A = torch.ones(1024, dtype=torch.float64, device=dev)
B = torch.full((1024,), 0.3, dtype=torch.float64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.Stream()
ts = []
with torch.cuda.stream(st):
    for r in range(13):
        sw.load_device(A.data_ptr(), B.data_ptr(), st.cuda_stream)
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sw.resume(1, st.cuda_stream)
        e1.record(st)
        st.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1))
print(json.dumps({"lib": os.environ.get("DSE_LIB"), "arith": arith.value, "ms": float(np.median(ts)), "min": min(ts)}))
