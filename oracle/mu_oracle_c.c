/* mu_oracle_c.c -- C restatement of oracle/mu_oracle.py's finite-mu sweep rows.
 *
 * TEST INFRASTRUCTURE ONLY (tests/ and bench.py's CPU-baseline leg): the
 * product never links it.  Same per-point formula as point_projections in
 * mu_oracle.py (explicit 4-vector components p = (|p|, 0, 0, p4 + i mu),
 * q = (|q| z, |q| sqrt(1 - z^2), 0, q4 + i mu), bilinear complex dot
 * products), summed sequentially over (j_s, j_4, k) per external point and
 * parallel over points with OpenMP.  PARITY UNPINNED AGAINST THE REFERENCE
 * (there is no finite-mu reference path); checked against the numpy oracle
 * in tests/test_mu_oracle.py.
 *
 * skip != 0: a (j_s, j_4) node whose every angular point has
 * exp(-k^2/w^2) == 0 exactly (lower bound of k^2 over the angles,
 * ((|q| - |p|)^2 + (q4 - p4)^2) / w^2 > 760, well past the underflow at
 * 745.13) is not evaluated -- the GPU kernels' exact-zero window skip.  It is
 * taken only when every value entering the node's summands is finite and
 * den != 0, so each skipped summand would have been an exact +-0: the sums
 * are bitwise those of skip = 0 (tested).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>

#include <omp.h>

typedef double complex cx;

static inline int cfin(cx v) { return isfinite(creal(v)) && isfinite(cimag(v)); }

static inline cx dot4(const cx a[4], const cx b[4]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + a[3] * b[3]; }

/* vertex: 0 bc, 1 bc1, 2 bcb (mu_grid.VERTICES order) */
int mu_sweep_rows(const double *p_ext, const double *p4_ext, int64_t n_s, int64_t n_4, const double *q_int,
                  const double *q4_int, const double *node_measure, int64_t m_s, int64_t m_4, const double *z,
                  const double *wz, int64_t K, double coeff, double omega, double mu, double z1, double m0,
                  int vertex, const double *A_, const double *B_, const double *C_, const double *Aq_,
                  const double *Bq_, const double *Cq_, const int64_t *rows, int64_t nrows, double *out_,
                  int threads, int skip) {
    const cx *A = (const cx *)A_, *B = (const cx *)B_, *C = (const cx *)C_;
    const cx *Aq = (const cx *)Aq_, *Bq = (const cx *)Bq_, *Cq = (const cx *)Cq_;
    cx *out = (cx *)out_;
    const int fac = vertex == 0, fb = vertex == 0 || vertex == 2, fdb = vertex == 0;
    const double w2 = omega * omega;
    (void)n_s;
    int bad = 0;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1) reduction(| : bad)
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t i = rows[r];
        const int64_t is = i / n_4, i4 = i % n_4;
        const double P = p_ext[is], p4r = p4_ext[i4];
        const cx p4t = p4r + I * mu;
        const cx Ap = A[i], Bp = B[i], Cp = C[i];
        cx sA_ = 0, sB_ = 0, sC_ = 0;
        for (int64_t js = 0; js < m_s; ++js) {
            const double Qs = q_int[js];
            for (int64_t j4 = 0; j4 < m_4; ++j4) {
                const int64_t j = js * m_4 + j4;
                const double q4r = q4_int[j4];
                const cx q4t = q4r + I * mu;
                const cx aq = Aq[j], bq = Bq[j], cq = Cq[j];
                const cx den = (Qs * Qs) * aq * aq + (q4t * q4t) * cq * cq + bq * bq;
                const cx sA = 0.5 * (Ap + aq), sC = 0.5 * (Cp + cq);
                const cx dq = (Qs * Qs - P * P) + (q4t * q4t - p4t * p4t);
                cx dA = (aq - Ap) / dq, dC = (cq - Cp) / dq, dB = (bq - Bp) / dq;
                if (skip) {
                    const double dqs = Qs - P, dq4 = q4r - p4r;
                    const double lb = dqs * dqs + dq4 * dq4;
                    if (lb > 760.0 * w2 && cfin(Ap) && cfin(Bp) && cfin(Cp) && cfin(aq) && cfin(bq) && cfin(cq) &&
                        cfin(den) && den != 0 && cfin(dA) && cfin(dB) && cfin(dC) && cfin(sA) && cfin(sC))
                        continue;
                }
                for (int64_t k = 0; k < K; ++k) {
                    const double zz = z[k];
                    const double sperp = sqrt(1.0 - zz * zz);
                    const double qx = Qs * zz, qy = Qs * sperp;
                    const cx kv[4] = {qx - P, qy, 0.0, q4r - p4r};
                    const cx tv[4] = {qx + P, qy, 0.0, q4t + p4t};
                    const double k2 = creal(kv[0]) * creal(kv[0]) + creal(kv[1]) * creal(kv[1]) +
                                      creal(kv[3]) * creal(kv[3]);
                    const double kks = creal(kv[0]) * creal(kv[0]) + creal(kv[1]) * creal(kv[1]);
                    const cx Q[4] = {aq * qx, aq * qy, 0.0, cq * q4t};
                    const cx Qp[4] = {sA * aq * qx, sA * aq * qy, 0.0, sC * cq * q4t};
                    const cx D[4] = {dA * tv[0], dA * tv[1], 0.0, dC * tv[3]};
                    const cx Z4[4] = {0, 0, 0, 0};
                    const cx *Dac = fac ? D : Z4;
                    const cx *Db = fb ? D : Z4;
                    const cx kt = dot4(kv, tv);
                    cx u[4];
                    for (int m = 0; m < 4; ++m) u[m] = tv[m] - kv[m] * kt / k2;
                    const cx trT = sA * (3.0 - kks / k2) + sC * (1.0 - creal(kv[3]) * creal(kv[3]) / k2);
                    const cx QD = dot4(Q, Dac), uD = dot4(u, Dac), uQ = dot4(u, Q);
                    /* A channel: e = (P, 0, 0, 0), e' = sA e */
                    const cx eA[4] = {P, 0, 0, 0};
                    const cx eAs[4] = {sA * P, 0, 0, 0};
                    const cx eC[4] = {0, 0, 0, 1.0};
                    const cx eCs[4] = {0, 0, 0, sC};
                    cx PA, PC;
                    {
                        const cx T1 = dot4(eA, Qp) - dot4(kv, eA) * dot4(kv, Qp) / k2;
                        const cx T2 = dot4(Q, eAs) - dot4(kv, Q) * dot4(kv, eAs) / k2;
                        const cx term1 = -(T1 + T2 - dot4(eA, Q) * trT);
                        const cx term2 = -0.5 * (dot4(eA, u) * QD - dot4(eA, Q) * uD + dot4(eA, Dac) * uQ);
                        PA = term1 + term2;
                    }
                    {
                        const cx T1 = dot4(eC, Qp) - dot4(kv, eC) * dot4(kv, Qp) / k2;
                        const cx T2 = dot4(Q, eCs) - dot4(kv, Q) * dot4(kv, eCs) / k2;
                        const cx term1 = -(T1 + T2 - dot4(eC, Q) * trT);
                        const cx term2 = -0.5 * (dot4(eC, u) * QD - dot4(eC, Q) * uD + dot4(eC, Dac) * uQ);
                        PC = term1 + term2;
                    }
                    const cx PB = bq * trT - (fdb ? dB * uQ : 0.0) + 0.5 * bq * dot4(u, Db);
                    const double w = node_measure[j] * wz[k];
                    const double g = coeff * exp(-k2 / w2);
                    const cx core = (w * g) / (k2 * den);
                    sA_ += core * PA;
                    sB_ += core * PB;
                    sC_ += core * PC;
                }
            }
        }
        const cx a = z1 + sA_ / (P * P), b = m0 * z1 + sB_, c = z1 + sC_ / p4t;
        out[3 * r] = a;
        out[3 * r + 1] = b;
        out[3 * r + 2] = c;
        if (!(isfinite(creal(a)) && isfinite(cimag(a)) && isfinite(creal(b)) && isfinite(cimag(b)) &&
              isfinite(creal(c)) && isfinite(cimag(c))))
            bad = 1;
    }
    return bad;
}
