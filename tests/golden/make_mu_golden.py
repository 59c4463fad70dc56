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

Usage:  python tests/golden/make_mu_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from dsegap.kernels import integrand_terms, kinematics  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
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


if __name__ == "__main__":
    main()
