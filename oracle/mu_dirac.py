"""Explicit Dirac-matrix evaluation of the finite-mu self-energy projections.

TEST INFRASTRUCTURE ONLY (tests/test_mu_oracle.py).  An independent check of
oracle/mu_oracle.point_projections: builds Euclidean hermitian gamma matrices
({gamma_mu, gamma_nu} = 2 delta_mu_nu), inverts S^-1(q~) = i gamma.q A +
i gamma_4 q~4 C + B numerically, forms the in-medium Ball-Chiu vertex and the
Landau-gauge transverse projector, and takes the traces

  P_A = tr[-i gamma.p_vec X]/4,  P_C = tr[-i gamma_4 X]/4,  P_B = tr[X]/4,
  X   = T_mu_nu(k) gamma_mu S(q~) Gamma_nu(q~, p~)

with the Delta_B vertex structure removed from the A and C channels (as the
reference removes it from A, kernels.py:1-14).  Results are multiplied by
den = q^2 A^2 + q~4^2 C^2 + B^2 to compare with point_projections, which
leaves 1/den to the caller.  Also checks the Ward-Takahashi identity
k_nu Gamma_nu = -i (S^-1(q~) - S^-1(p~)).
"""
from __future__ import annotations

import numpy as np

_s = [np.array([[0, 1], [1, 0]], complex), np.array([[0, -1j], [1j, 0]], complex),
      np.array([[1, 0], [0, -1]], complex)]
_Z = np.zeros((2, 2), complex)
_I2 = np.eye(2, dtype=complex)
GAMMA = [np.block([[_Z, -1j * s], [1j * s, _Z]]) for s in _s] + [np.block([[_I2, _Z], [_Z, -_I2]])]
ONE = np.eye(4, dtype=complex)


def slash(v):
    return sum(v[m] * GAMMA[m] for m in range(4))


def s_inv(vec3, v4, A, B, C):
    return 1j * sum(vec3[m] * GAMMA[m] for m in range(3)) * A + 1j * GAMMA[3] * v4 * C + B * ONE


def vertex_fn(nu, t, sA, sC, dA, dC, dB, with_db=True):
    D = (dA * t[0], dA * t[1], dA * t[2], dC * t[3])
    g = (sA if nu < 3 else sC) * GAMMA[nu] + 0.5 * t[nu] * slash(D)
    if with_db:
        g = g - 1j * t[nu] * dB * ONE
    return g


def projections(P, p4t, Qs, z, q4t, q4r, p4r, Ap, Bp, Cp, Aq, Bq, Cq, vertex="bc"):
    pv = (P, 0.0, 0.0)
    qv = (Qs * z, Qs * np.sqrt(1.0 - z * z), 0.0)
    k = (qv[0] - pv[0], qv[1] - pv[1], 0.0, q4r - p4r)
    t = (qv[0] + pv[0], qv[1] + pv[1], 0.0, q4t + p4t)
    k2 = sum(x * x for x in k)
    dq = (Qs * Qs - P * P) + (q4t * q4t - p4t * p4t)
    sA, sC = 0.5 * (Ap + Aq), 0.5 * (Cp + Cq)
    dA, dC, dB = (Aq - Ap) / dq, (Cq - Cp) / dq, (Bq - Bp) / dq
    S = np.linalg.inv(s_inv(qv, q4t, Aq, Bq, Cq))
    den = (Qs * Qs) * Aq * Aq + (q4t * q4t) * Cq * Cq + Bq * Bq
    T = np.eye(4) - np.outer(k, k) / k2

    fac, fb, fdb = vertex == "bc", vertex in ("bc", "bcb"), vertex == "bc"

    def X(qa, qc, qb):
        acc = np.zeros((4, 4), complex)
        for m in range(4):
            for n in range(4):
                if T[m, n] != 0.0:
                    acc += T[m, n] * GAMMA[m] @ S @ vertex_fn(n, t, sA, sC, qa, qc, qb, True)
        return acc

    Xn = X(dA if fac else 0.0, dC if fac else 0.0, 0.0)       # A and C channels
    Xf = X(dA if fb else 0.0, dC if fb else 0.0, dB if fdb else 0.0)  # B channel
    PA = np.trace(-1j * slash((pv[0], pv[1], pv[2], 0.0)) @ Xn) / 4.0
    PC = np.trace(-1j * GAMMA[3] @ Xn) / 4.0
    PB = np.trace(Xf) / 4.0
    # Ward-Takahashi identity of the vertex
    lhs = sum(k[n] * vertex_fn(n, t, sA, sC, dA, dC, dB) for n in range(4))
    pvec4 = (pv[0], pv[1], pv[2])
    rhs = -1j * (s_inv(qv, q4t, Aq, Bq, Cq) - s_inv(pvec4, p4t, Ap, Bp, Cp))
    wti = float(np.max(np.abs(lhs - rhs)))
    return k2, PA * den, PC * den, PB * den, wti
