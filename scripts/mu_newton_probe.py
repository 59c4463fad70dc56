"""GPU probe: the full in-medium Ball-Chiu vertex ('bc') by Newton-Krylov
(finite_mu.solve_mu_newton) -- config 3 at mu = 0.2, the same grid at mu = 0
against the vacuum solution (O(4) symmetry: A = C = A_vac(|p|^2 + p4^2)),
and a small grid checked against the C oracle's sweep (residual of the
oracle's own map at the GPU's solution)."""
import sys
import time
from dataclasses import replace

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import paper_2012_03667_b200 as p  # noqa: E402
from paper_2012_03667_b200.finite_mu import solve_mu_newton, solve_mu  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("small", "all"):
    import mu_oracle as mo
    for mu in (0.2, 0.0):
        prm = MuParams(vertex="bc", mu=mu, n_s=12, n_4=12, m_s=16, m_4=16, m_ang=8, xi=1e-10)
        g = grid_for(prm)
        t0 = time.time()
        sol, rep = solve_mu_newton(prm, g)
        out = mo.sweep_rows_c(g, prm, sol.A, sol.B, sol.C, np.arange(g.n_ext))
        res = max(np.max(np.abs(out[:, 0] - sol.A.reshape(-1))), np.max(np.abs(out[:, 1] - sol.B.reshape(-1))),
                  np.max(np.abs(out[:, 2] - sol.C.reshape(-1))))
        print(f"small mu={mu}: converged={sol.converged} newton={sol.iterations} sweeps={rep.sweeps} "
              f"start_its={rep.start_iterations} oracle_residual={res:.3e} {time.time() - t0:.2f}s", flush=True)
        for s in rep.steps:
            print("   step", s)

if which in ("c3", "all"):
    for mu in (0.2, 0.0):
        prm = MuParams(vertex="bc", mu=mu, mode="moments")
        g = grid_for(prm)
        t0 = time.time()
        sol, rep = solve_mu_newton(prm, g)
        t1 = time.time()
        print(f"config3 bc mu={mu}: converged={sol.converged} newton={sol.iterations} sweeps={rep.sweeps} "
              f"start_its={rep.start_iterations} {t1 - t0:.2f}s", flush=True)
        for s in rep.steps:
            print("   step", s, flush=True)
        b = solve_mu(replace(prm, vertex="bcb"), g)
        print("  max|A_bc - A_bcb| %.3e  max|B| diff %.3e  max|C| diff %.3e" % (
            np.max(np.abs(sol.A - b.A)), np.max(np.abs(sol.B - b.B)), np.max(np.abs(sol.C - b.C))))
        i0 = np.argsort(np.abs(g.p4_ext))[0]
        print("  IR (p=%.3g, p4=%.3g): A_bc %s C_bc %s B_bc %s | bcb A %s B %s" % (
            g.p_ext[0], g.p4_ext[i0], sol.A[0, i0], sol.C[0, i0], sol.B[0, i0], b.A[0, i0], b.B[0, i0]))
        if mu == 0.0:
            vp = p.ModelParams(N=128, m_rad=128, m_ang=64, xi=1e-10, max_iterations=20000)
            vg = p.build_grid(128, 128, 64, 1e-6, 1e4)
            vs = p.solve(vp, p.VARIANTS["indexed-gpu-moments"], grid=vg, b0=np.full(128, 0.3))
            p2 = g.p_ext[:, None] ** 2 + g.p4_ext[None, :] ** 2
            Av = np.interp(np.log(p2), np.log(vg.p2_ext), vs.A)
            Bv = np.interp(np.log(p2), np.log(vg.p2_ext), vs.B)
            for lim in (1.0, 4.0, 1e4):
                m = (p2 < lim) & (p2 > 1e-6)
                print("  mu=0 vs vacuum, p2<%g: max|A-Av| %.3e max|C-Av| %.3e max|B-Bv| %.3e max|A-C| %.3e" % (
                    lim, np.max(np.abs(sol.A - Av)[m]), np.max(np.abs(sol.C - Av)[m]), np.max(np.abs(sol.B - Bv)[m]),
                    np.max(np.abs(sol.A - sol.C)[m])))
            E = np.abs(sol.C - Av)
            i, j = np.unravel_index(np.argmax(E), E.shape)
            print("  worst C at p=%.3g p4=%.3g: C=%s A=%s Av=%.5f" % (g.p_ext[i], g.p4_ext[j], sol.C[i, j], sol.A[i, j],
                                                                  Av[i, j]))
            np.savez("gpurun_out/mu_newton_mu0.npz", A=sol.A, B=sol.B, C=sol.C, Av=Av, Bv=Bv)
        else:
            np.savez("gpurun_out/mu_newton_mu02.npz", A=sol.A, B=sol.B, C=sol.C, Ab=b.A, Bb=b.B, Cb=b.C)
