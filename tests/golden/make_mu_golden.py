"""Generate tests/golden/mu_vacuum_points.npz by RUNNING THE REFERENCE.

The finite-mu path has no reference implementation; its one
reference anchor is the mu = 0 limit.  With mu = 0, C = A and A, B functions
of the 4-D p^2 only, the finite-mu projections must reduce pointwise to the
reference's vacuum integrand:

  P_A(e = p_vec) + p4 P_C(e = unit_4)  ==  IA2 + IA3        (kernels.py:158-161)
  P_B                                   ==  IB1 + IB2 + IB3  (kernels.py:162-165)

This script draws seeded (|p|, p4, |q|, q4, cos theta) points and dressing
values, maps each to the reference's 4-D kinematics (p2, q2, z4) and records
the reference's own `integrand_terms(kinematics(p2, q2, z4), a_p, a_q, b_p, b_q)`.
Run once in the build container (the reference is not on the GPU box).

--config3 / --config4 write the full-size converged fixtures instead
(mu_full_<tag>.npz).  There is no reference for finite mu, so these come from
the C oracle (oracle/mu_oracle_c.c through oracle/mu_oracle.solve_c:
explicit 4-vector projections, sequential sums, exact-zero node skip that is
bitwise neutral) run on the grid arrays stored in the same file:
  config3       mu = 0.2 GeV, BASELINE config 3 (MuParams defaults, vertex bcb)
  config4_k<k>  mu = 0.4 (k + 1/2) / 32, the k-th of config 4's 32 values
Each holds the MuGrid arrays, A, B, C, iterations, converged, history.

Usage:  python tests/golden/make_mu_golden.py [--config3] [--config4 K ...] [--threads T]
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    from dsegap.kernels import integrand_terms, kinematics
    rng = np.random.default_rng(20121036)
    n = 400
    P = np.exp(rng.uniform(np.log(1e-2), np.log(10.0), n))
    Qs = np.exp(rng.uniform(np.log(1e-2), np.log(10.0), n))
    p4 = rng.uniform(-3.0, 3.0, n)
    q4 = rng.uniform(-3.0, 3.0, n)
    z = rng.uniform(-0.99, 0.99, n)
    ap, aq = rng.uniform(0.8, 2.0, n), rng.uniform(0.8, 2.0, n)
    bp, bq = rng.uniform(0.0, 1.5, n), rng.uniform(0.0, 1.5, n)
    ia, ib, p2s, q2s, z4s = [], [], [], [], []
    for i in range(n):
        p2 = P[i] ** 2 + p4[i] ** 2
        q2 = Qs[i] ** 2 + q4[i] ** 2
        pq = P[i] * Qs[i] * z[i] + p4[i] * q4[i]
        z4 = pq / np.sqrt(p2 * q2)
        t = integrand_terms(kinematics(p2, q2, z4), ap[i], aq[i], bp[i], bq[i])
        ia.append(t.IA2 + t.IA3)
        ib.append(t.IB1 + t.IB2 + t.IB3)
        p2s.append(p2), q2s.append(q2), z4s.append(z4)
    np.savez(os.path.join(HERE, "mu_vacuum_points.npz"), P=P, Qs=Qs, p4=p4, q4=q4, z=z, ap=ap, aq=aq,
             bp=bp, bq=bq, p2=np.array(p2s), q2=np.array(q2s), z4=np.array(z4s), ia=np.array(ia), ib=np.array(ib),
             call=np.array("dsegap.kernels.integrand_terms(kinematics(p2, q2, z4), a_p, a_q, b_p, b_q); "
                           "IA2+IA3, IB1+IB2+IB3"))
    print("wrote mu_vacuum_points.npz", n)


GRID_FIELDS = ("p_ext", "ps2_ext", "p4_ext", "q_int", "qs2_int", "q4_int", "meas_s", "meas_4", "z_nodes",
               "z_weights", "brk_s", "brk_4", "node_measure")


def full_solve(tag: str, mu: float, threads: int):
    import time
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import mu_oracle
    from paper_2012_03667_b200.mu_grid import MuParams, grid_for
    prm = MuParams(mu=mu)
    g = grid_for(prm)
    t0 = time.perf_counter()

    def log(n, d):
        print(f"{tag} iteration {n}: {d[0]:.3e} {d[1]:.3e} {d[2]:.3e} ({time.perf_counter() - t0:.0f} s)", flush=True)

    A, B, C, n, conv, hist = mu_oracle.solve_c(g, prm, threads=threads, on_iteration=log)
    path = os.path.join(HERE, f"mu_full_{tag}.npz")
    np.savez_compressed(path, A=A, B=B, C=C, iterations=np.array(n), converged=np.array(conv),
                        history=np.array(hist, dtype=np.float64),
                        params=np.array([prm.D, prm.omega, prm.m0, prm.z1, prm.mu, prm.xi, prm.max_iterations,
                                         prm.relaxation]),
                        vertex=np.array(prm.vertex), seconds=np.array(time.perf_counter() - t0),
                        call=np.array(f"mu_oracle.solve_c(grid_for(MuParams(mu={mu!r})), MuParams(mu={mu!r}))"),
                        **{f"grid_{k}": getattr(g, k) for k in GRID_FIELDS})
    print(f"wrote {path}: {n} iterations, converged={conv}, {time.perf_counter() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--config3", action="store_true")
    ap.add_argument("--config4", type=int, nargs="*", default=[])
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    args = ap.parse_args()
    if not args.config3 and not args.config4:
        main()
    if args.config3:
        full_solve("config3", 0.2, args.threads)
    for k in args.config4:
        full_solve(f"config4_k{k:02d}", 0.4 * (k + 0.5) / 32, args.threads)
