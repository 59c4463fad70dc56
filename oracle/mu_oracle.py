"""CPU oracle of the finite chemical potential sweep (BASELINE configs 3-4).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline leg.  The product package never imports
it.

PARITY UNPINNED AGAINST THE REFERENCE: the reference has no finite-mu code
(SPEC.md:16).  This is a self-derived
restatement of the equations in DESIGN.md "Finite chemical potential", which
extend the reference's vacuum equation (kernels.py:178-226) to
S^-1(p~) = i gamma.p A + i gamma_4 p~4 C + B with p~ = (p, p4 + i mu):

  Sigma(p~) = sum_q  w_q g(k^2)/k^2 T_{mu nu}(k) gamma_mu S(q~) Gamma_nu(q~, p~)
  Gamma_nu  = Sigma_F gamma_nu + 1/2 t~_nu gamma.D - i t~_nu Delta_B      (Ball-Chiu, in medium)
  A = z1 + P_A/|p|^2,  C = z1 + P_C/p~4,  B = m0 z1 + P_B

What pins it instead:
  * the projections are checked against an explicit 4x4 Dirac-matrix
    evaluation of the traces (tests/test_mu_oracle.py, oracle/mu_dirac.py);
  * at mu = 0 with C = A and A, B functions of p^2, the full 4-D projection
    P_A + p4 P_C reduces POINTWISE to the reference's vacuum integrand
    IA2 + IA3 and IB1 + IB2 + IB3 (kernels.py:152-175, checked against the
    reference's own integrand_terms in tests/golden/mu_vacuum_points.npz);
  * at mu = 0 a converged solve restores O(4) symmetry, A = C, up to the
    2-D discretisation (tests/test_mu_oracle.py).  (A solution-level
    comparison with the vacuum solver would need the full "bc" vertex, the
    only mode whose mu = 0 equation IS the reference's; on a 2-D grid it
    diverges under successive approximation.)

Here every point is formed from explicit 4-vector components
p = (|p|, 0, 0, p~4), q = (|q| z, |q| sqrt(1-z^2), 0, q~4) and bilinear dot
products -- not from the kernel's factored polynomial form -- so the GPU path
and this oracle are independent evaluations.  The Delta_B structure is kept
in the B channel only, as the reference does for A (kernels.py:1-14).
"""
from __future__ import annotations

import numpy as np

__all__ = ["interp2d", "point_projections", "sweep_row", "sweep", "solve", "delta", "sweep_rows_c"]


def _lin(xi, xi1, vi, vi1, q):
    # interpolation.py:71-72 _linear_eval op order, real arrays
    return vi + ((q - xi) * (vi1 - vi)) / (xi1 - xi)


def _axis(x, idx, q):
    """Per-axis (lo, hi, clamp) for the reference's clamped linear rule
    (interpolation.py:125-132): idx < 0 -> node 0, idx >= n-1 -> node n-1."""
    n = x.size
    lo = np.clip(idx, 0, n - 1)
    hi = np.clip(idx + 1, 0, n - 1)
    inside = (idx >= 0) & (idx < n - 1)
    return lo, hi, inside


def interp2d(grid, F: np.ndarray) -> np.ndarray:
    """Complex values at the internal (|q|, q4) nodes, shape (m_s, m_4):
    linear in |p|^2 (as the vacuum interpolates linearly in p^2,
    SPEC.md:223) along each of the two bracketing p4 rows, then linear in p4;
    real and imaginary parts separately, reference op order, per-axis
    clamping at the ends."""
    F = np.asarray(F, dtype=np.complex128).reshape(grid.n_s, grid.n_4)
    xs, x4 = grid.ps2_ext, grid.p4_ext
    slo, shi, sin_ = _axis(xs, grid.brk_s, None)
    tlo, thi, tin = _axis(x4, grid.brk_4, None)
    qs = grid.qs2_int[:, None]
    q4 = grid.q4_int[None, :]
    out = []
    for part in (F.real, F.imag):
        part = np.ascontiguousarray(part)

        def along_s(t_idx):
            v0 = part[slo[:, None], t_idx[None, :]]
            v1 = part[shi[:, None], t_idx[None, :]]
            xs0 = xs[slo][:, None]
            xs1 = xs[shi][:, None]
            with np.errstate(invalid="ignore", divide="ignore"):
                lin = _lin(xs0, xs1, v0, v1, qs)
            return np.where(sin_[:, None], lin, v0)

        f0 = along_s(tlo)
        f1 = along_s(thi)
        x40 = x4[tlo][None, :]
        x41 = x4[thi][None, :]
        with np.errstate(invalid="ignore", divide="ignore"):
            lin = _lin(x40, x41, f0, f1, q4)
        out.append(np.where(tin[None, :], lin, f0))
    return out[0] + 1j * out[1]


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + a[3] * b[3]


VERTICES = ("bc", "bc1", "bcb")


def point_projections(P, p4t, Qs, z, q4t, q4r, p4r, Ap, Bp, Cp, Aq, Bq, Cq, vertex="bc"):
    """(k^2, P_A(e = p), P_C(e = unit 4), P_B) at broadcastable points.

    P, Qs, z, q4r, p4r real; p4t = p4 + i mu, q4t = q4 + i mu complex; the
    dressing values complex.  The quark propagator numerator is -i gamma.Q +
    Bq with Q = (Aq q_vec, Cq q~4); the 1/den factor is applied by the caller.
    vertex: "bc" the in-medium Ball-Chiu vertex (Delta_B in the B channel
    only), "bc1" its Sigma structure only, "bcb" Sigma everywhere plus the
    Delta_A/Delta_C structures in the B channel only.
    """
    fac = vertex == "bc"           # Delta_A, Delta_C in the A and C channels
    fb = vertex in ("bc", "bcb")   # Delta_A, Delta_C in the B channel
    fdb = vertex == "bc"           # Delta_B in the B channel
    zero = np.zeros(np.broadcast(P, Qs, z, q4r, p4r).shape)
    sperp = np.sqrt(1.0 - z * z)
    qx, qy = Qs * z, Qs * sperp
    # real gluon momentum k = q - p (the i mu cancels), t = q~ + p~
    k = (qx - P + zero, qy + zero, zero, q4r - p4r + zero)
    t = (qx + P + zero, qy + zero, zero, q4t + p4t + zero)
    k2 = k[0] * k[0] + k[1] * k[1] + k[3] * k[3]
    kk_s = k[0] * k[0] + k[1] * k[1]
    sA = 0.5 * (Ap + Aq)
    sC = 0.5 * (Cp + Cq)
    dq = (Qs * Qs - P * P) + (q4t * q4t - p4t * p4t)        # q~^2 - p~^2
    dA = (Aq - Ap) / dq
    dC = (Cq - Cp) / dq
    dB = (Bq - Bp) / dq
    Q = (Aq * qx, Aq * qy, zero, Cq * q4t)
    Qp = (sA * Aq * qx, sA * Aq * qy, zero, sC * Cq * q4t)
    D = (dA * t[0], dA * t[1], zero, dC * t[3])
    D0 = (zero, zero, zero, zero)
    Dac = D if fac else D0
    Db = D if fb else D0
    kt = _dot(k, t)
    u = tuple(t[m] - k[m] * kt / k2 for m in range(4))
    trT = sA * (3.0 - kk_s / k2) + sC * (1.0 - k[3] * k[3] / k2)

    def T(a, b):
        return _dot(a, b) - _dot(k, a) * _dot(k, b) / k2

    QD, uD, uQ = _dot(Q, Dac), _dot(u, Dac), _dot(u, Q)

    def proj(e, e_scaled):
        term1 = -(T(e, Qp) + T(Q, e_scaled) - _dot(e, Q) * trT)
        term2 = -0.5 * (_dot(e, u) * QD - _dot(e, Q) * uD + _dot(e, Dac) * uQ)
        return term1 + term2

    eA = (P + zero, zero, zero, zero)
    eC = (zero, zero, zero, 1.0 + zero)
    PA = proj(eA, tuple(sA * c for c in eA))
    PC = proj(eC, tuple(sC * c for c in eC))
    PB = Bq * trT - (dB * uQ if fdb else 0.0) + 0.5 * Bq * _dot(u, Db)
    return k2, PA, PC, PB


def sweep_row(grid, params, i: int, A, B, C, Aq, Bq, Cq):
    """(A', B', C') at external point i given the dressing values at the
    internal nodes (shape (m_s, m_4)).  Sums with np.sum over the full
    (m_s, m_4, m_ang) block like the reference's row_rhs (kernels.py:217-218)."""
    i_s, i_4 = divmod(int(i), grid.n_4)
    P = grid.p_ext[i_s]
    p4r = grid.p4_ext[i_4]
    p4t = p4r + 1j * params.mu
    Ap, Bp, Cp = A.reshape(-1)[i], B.reshape(-1)[i], C.reshape(-1)[i]
    Qs = grid.q_int[:, None, None]
    q4r = grid.q4_int[None, :, None]
    q4t = q4r + 1j * params.mu
    z = grid.z_nodes[None, None, :]
    aq, bq, cq = (x[:, :, None] for x in (Aq, Bq, Cq))
    k2, PA, PC, PB = point_projections(P, p4t, Qs, z, q4t, q4r, p4r, Ap, Bp, Cp, aq, bq, cq, params.vertex)
    den = (Qs * Qs) * aq * aq + (q4t * q4t) * cq * cq + bq * bq
    w = grid.node_measure[:, :, None] * grid.z_weights[None, None, :]
    g = params.interaction_coeff * np.exp(-k2 / (params.omega * params.omega))
    core = (w * g) / (k2 * den)
    with np.errstate(all="ignore"):
        a_new = params.z1 + np.sum(core * PA) / (P * P)
        c_new = params.z1 + np.sum(core * PC) / p4t
        b_new = params.m0 * params.z1 + np.sum(core * PB)
    return a_new, b_new, c_new, (core, PA, PB, PC)


class MuNumericalFailure(RuntimeError):
    def __init__(self, row, radial, angular):
        super().__init__(f"non-finite integrand in finite-mu sweep at row={row}, radial={radial}, angular={angular}")
        self.row, self.radial, self.angular = row, radial, angular


def sweep(grid, params, A, B, C, rows=None):
    """One Jacobi sweep over all (or the listed) external points.  Raises
    MuNumericalFailure(row, radial j = j_s*m_4 + j_4, angular k) at the
    lowest failing row, first non-finite point in row-major order
    (kernels.py:219-225)."""
    A = np.asarray(A, np.complex128).reshape(grid.n_s, grid.n_4)
    B = np.asarray(B, np.complex128).reshape(grid.n_s, grid.n_4)
    C = np.asarray(C, np.complex128).reshape(grid.n_s, grid.n_4)
    Aq, Bq, Cq = interp2d(grid, A), interp2d(grid, B), interp2d(grid, C)
    An, Bn, Cn = A.copy().reshape(-1), B.copy().reshape(-1), C.copy().reshape(-1)
    rows = range(grid.n_ext) if rows is None else rows
    for i in rows:
        a, b, c, (core, PA, PB, PC) = sweep_row(grid, params, i, A, B, C, Aq, Bq, Cq)
        if not (np.isfinite(a) and np.isfinite(b) and np.isfinite(c)):
            bad = ~np.isfinite(core * (PA + PB + PC))
            if bad.any():
                js, j4, k = (int(v) for v in np.argwhere(bad)[0])
                raise MuNumericalFailure(int(i), js * grid.m_4 + j4, k)
            raise MuNumericalFailure(int(i), -1, -1)
        An[i], Bn[i], Cn[i] = a, b, c
    shape = (grid.n_s, grid.n_4)
    return An.reshape(shape), Bn.reshape(shape), Cn.reshape(shape)


def delta(new, old) -> float:
    """max |new - old| (complex modulus), iteration.py:34 on complex state."""
    return float(np.max(np.abs(np.asarray(new) - np.asarray(old))))


def solve(grid, params, A0=None, B0=None, C0=None):
    """Successive approximation (iteration.py:18-40, solver.py:247-252) on
    the complex state (A, B, C).  Returns (A, B, C, iterations, converged,
    history[(n, dA, dB, dC)])."""
    shape = (grid.n_s, grid.n_4)
    A = np.ones(shape, np.complex128) if A0 is None else np.array(A0, np.complex128).reshape(shape)
    B = np.full(shape, 0.3, np.complex128) if B0 is None else np.array(B0, np.complex128).reshape(shape)
    C = np.ones(shape, np.complex128) if C0 is None else np.array(C0, np.complex128).reshape(shape)
    relax = params.relaxation
    hist = [(0, np.nan, np.nan, np.nan)]
    for n in range(1, params.max_iterations + 1):
        An, Bn, Cn = sweep(grid, params, A, B, C)
        if relax != 1.0:
            An = relax * An + (1.0 - relax) * A
            Bn = relax * Bn + (1.0 - relax) * B
            Cn = relax * Cn + (1.0 - relax) * C
        d = (delta(An, A), delta(Bn, B), delta(Cn, C))
        A, B, C = An, Bn, Cn
        hist.append((n, *d))
        if all(x < params.xi for x in d):
            return A, B, C, n, True, hist
    return A, B, C, params.max_iterations, False, hist


_CLIB = None


def _clib():
    """liboracle_mu.so (mu_oracle_c.c, the same per-point formula in C with
    OpenMP over points; built by oracle/Makefile)."""
    global _CLIB
    if _CLIB is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        path = os.path.join(here, "liboracle_mu.so")
        src = os.path.join(here, "mu_oracle_c.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", here, "liboracle_mu.so"], check=True)
        lib = ctypes.CDLL(path)
        f64 = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        lib.mu_sweep_rows.restype = ctypes.c_int
        lib.mu_sweep_rows.argtypes = [f64, f64, i64, i64, f64, f64, f64, i64, i64, f64, f64, i64,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_int, f64, f64, f64, f64, f64, f64,
                                      ctypes.POINTER(ctypes.c_int64), i64, f64, ctypes.c_int, ctypes.c_int]
        _CLIB = lib
    return _CLIB


def sweep_rows_c(grid, params, A, B, C, rows, threads: int | None = None, skip: bool = True):
    """(A', B', C') at the listed external points, C restatement (sequential
    sums over (j_s, j_4, k) per point; np.sum's pairwise order in sweep_row
    differs at the rounding level).  Returns complex array [len(rows), 3].
    skip: the exact-zero node skip (bitwise equal to skip=False)."""
    import ctypes
    import os
    lib = _clib()
    shape = (grid.n_s, grid.n_4)
    A, B, C = (np.ascontiguousarray(np.asarray(x, np.complex128).reshape(shape)) for x in (A, B, C))
    Aq, Bq, Cq = (np.ascontiguousarray(interp2d(grid, X)) for X in (A, B, C))
    rows = np.ascontiguousarray(np.asarray(rows, np.int64))
    out = np.empty((rows.size, 3), np.complex128)
    f = lambda a: np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    keep = [np.ascontiguousarray(getattr(grid, n), dtype=np.float64) for n in
            ("p_ext", "p4_ext", "q_int", "q4_int", "node_measure", "z_nodes", "z_weights")]
    ptr = [k.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for k in keep]
    cv = lambda a: a.view(np.float64).ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
    vertex = ("bc", "bc1", "bcb").index(params.vertex)
    bad = lib.mu_sweep_rows(ptr[0], ptr[1], grid.n_s, grid.n_4, ptr[2], ptr[3], ptr[4], grid.m_s, grid.m_4, ptr[5],
                            ptr[6], grid.m_ang, params.interaction_coeff, params.omega, params.mu, params.z1,
                            params.m0, vertex, cv(A), cv(B), cv(C), cv(Aq), cv(Bq), cv(Cq),
                            rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), rows.size, cv(out),
                            int(threads or os.cpu_count() or 1), int(bool(skip)))
    del f
    if bad:
        raise MuNumericalFailure(-1, -1, -1)
    return out


def solve_c(grid, params, A0=None, B0=None, C0=None, threads: int | None = None, skip: bool = True,
            on_iteration=None):
    """solve() with every sweep done by the C restatement (sweep_rows_c over
    all external points; sequential sums over (j_s, j_4, k)): the oracle for
    full-size configs 3-4, where the numpy sweep is too slow.  Same loop,
    relaxation, deltas, stop rule and history as solve()."""
    shape = (grid.n_s, grid.n_4)
    A = np.ones(shape, np.complex128) if A0 is None else np.array(A0, np.complex128).reshape(shape)
    B = np.full(shape, 0.3, np.complex128) if B0 is None else np.array(B0, np.complex128).reshape(shape)
    C = np.ones(shape, np.complex128) if C0 is None else np.array(C0, np.complex128).reshape(shape)
    relax = params.relaxation
    rows = np.arange(grid.n_ext)
    hist = [(0, np.nan, np.nan, np.nan)]
    for n in range(1, params.max_iterations + 1):
        out = sweep_rows_c(grid, params, A, B, C, rows, threads=threads, skip=skip)
        An, Bn, Cn = (out[:, c].reshape(shape) for c in range(3))
        if relax != 1.0:
            An = relax * An + (1.0 - relax) * A
            Bn = relax * Bn + (1.0 - relax) * B
            Cn = relax * Cn + (1.0 - relax) * C
        d = (delta(An, A), delta(Bn, B), delta(Cn, C))
        A, B, C = An, Bn, Cn
        hist.append((n, *d))
        if on_iteration is not None:
            on_iteration(n, d)
        if all(x < params.xi for x in d):
            return A, B, C, n, True, hist
    return A, B, C, params.max_iterations, False, hist
