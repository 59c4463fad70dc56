"""Pairs kernel: where does the time above the FP64-pipe floor go?  Per-iteration
time across shapes (more rows = more items per warp, more angles = longer
items) and across iterations per launch, against the pipe floor
(evaluated points x 23.42 FP64 instructions / (148 SMs x 64 lanes/clk))."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2012_03667_b200 as p  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream().cuda_stream
arith = getattr(p.Arithmetic, (sys.argv[1] if len(sys.argv) > 1 else "PAIRS").upper())
FP64_PER_POINT = {"PAIRS": 23.42, "EXACT": 102.45, "FAST": 30.0}[arith.name]


def med(fn, pre, n=15):
    for _ in range(3):
        pre(); fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


for (N, M, K) in [(1024, 1024, 256), (2048, 1024, 256), (4096, 1024, 256), (1024, 1024, 1024), (1024, 2048, 256),
                  (512, 1024, 256), (256, 256, 256)]:
    g = p.build_grid(N, M, K, 1e-6, 1e4)
    prm = p.ModelParams(N=N, m_rad=M, m_ang=K, xi=1e-300, max_iterations=100000)
    sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, arith, 0)
    a = torch.ones(N, dtype=torch.float64, device=dev)
    b = torch.full((N,), 0.3, dtype=torch.float64, device=dev)
    ev = sw.stats()["evaluated_points"]
    floor_ms = ev * FP64_PER_POINT / (148 * 64) / 1.965e9 * 1e3
    load = lambda: sw.load_device(a.data_ptr(), b.data_ptr(), s)  # noqa: E731
    t1 = med(lambda: sw.resume(1, s), lambda: (load(), flush.fill_(1)))
    t1n = med(lambda: sw.resume(1, s), load)
    t4 = med(lambda: sw.resume(4, s), load) / 4
    print(f"{arith.name} N={N} M={M} K={K} evaluated={ev} floor={floor_ms:.4f} ms | 1 it flushed {t1:.4f} ({floor_ms/t1:.3f}) "
          f"| 1 it {t1n:.4f} ({floor_ms/t1n:.3f}) | per it of 4 {t4:.4f} ({floor_ms/t4:.3f}) | {sw.layout()}", flush=True)
    sw.close()
