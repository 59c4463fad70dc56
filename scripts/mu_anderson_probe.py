"""GPU experiment: Anderson acceleration of the full in-medium BC vertex
(which diverges under plain successive approximation).  x = (A, B, C) complex;
g(x) = one sweep; AA(m) on the residual f = g(x) - x."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2012_03667_b200.finite_mu import MuSweeper  # noqa: E402
from paper_2012_03667_b200.mu_grid import MuParams, grid_for  # noqa: E402

m_hist = int(sys.argv[1]) if len(sys.argv) > 1 else 8
beta = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
size = dict(n_s=64, n_4=64, m_s=64, m_4=64, m_ang=16) if (len(sys.argv) > 3 and sys.argv[3] == "small") else {}
vertex = sys.argv[4] if len(sys.argv) > 4 else "bc"
p = MuParams(vertex=vertex, **size)
g = grid_for(p)
shape = (g.n_s, g.n_4)
x = np.concatenate([np.ones(g.n_ext, complex), np.full(g.n_ext, 0.3 + 0j), np.ones(g.n_ext, complex)])
X, F = [], []
t0 = time.time()
with MuSweeper(g, p) as sw:
    for it in range(1, 301):
        A, B, C = (x[k * g.n_ext:(k + 1) * g.n_ext].reshape(shape) for k in range(3))
        try:
            gx = np.concatenate([v.reshape(-1) for v in sw.sweep(A, B, C)])
        except Exception as e:  # noqa: BLE001
            print("fail", it, str(e)[:80])
            break
        f = gx - x
        res = np.max(np.abs(f))
        if it % 10 == 0 or res < 1e-9:
            print(it, f"{res:.3e}", f"{time.time() - t0:.1f}s", flush=True)
        if res < 1e-9:
            print("converged", it)
            break
        X.append(x.copy())
        F.append(f)
        if len(F) > m_hist + 1:
            X.pop(0)
            F.pop(0)
        if len(F) == 1:
            x = x + beta * f
            continue
        dF = np.stack([F[k + 1] - F[k] for k in range(len(F) - 1)], axis=1)
        dX = np.stack([X[k + 1] - X[k] for k in range(len(X) - 1)], axis=1)
        gam, *_ = np.linalg.lstsq(dF, f, rcond=None)
        x = x + beta * f - (dX + beta * dF) @ gam
print("A0", x[0], "C0", x[2 * g.n_ext])
