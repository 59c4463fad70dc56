// dse_mu.cu -- finite chemical potential sweep (BASELINE configs 3-4).
// Included at the end of dse_b200.cu (one translation unit: it reuses the
// fast exp, the reciprocal, the error helpers and the launch counter).
//
// The reference has no finite-mu path; this is
// the self-derived extension written out in DESIGN.md "Finite chemical
// potential" and restated independently by oracle/mu_oracle.py (explicit
// 4-vector components, pinned against explicit Dirac traces and, at mu = 0,
// pointwise against the reference's integrand_terms, kernels.py:152-175).
//
// Per external point p~ = (|p|, p4 + i mu) and internal node q~ = (|q|,
// q4 + i mu) every projection of T_mu_nu(k) gamma_mu S(q~) Gamma_nu is a
// polynomial of degree <= 2 in r = p.q (spatial) and <= 1 in K = 1/k^2
// (DESIGN.md derives the coefficients).  With the interaction g(k^2) K and
// the angular weights, the angular sum of a (row, node) pair therefore
// factors into five real moments
//     S0 = sum_k w e K,  S1 = sum_k w e K r,  T0 = sum_k w e K^2,
//     T1 = sum_k w e K^2 r,  T2 = sum_k w e K^2 r^2      (e = exp(-k^2/w^2))
// accumulated point by point (one exp and one reciprocal per point), then
// contracted once per pair with complex coefficients.  Every point is still
// evaluated every iteration (the "integrand points" metric); the pair-level
// contraction is ~1/32 of the work at m_ang = 32.
//
// Layout: state X[2][3][n_ext] complex (ping-pong by iteration parity),
// node table NB[m_int] = {A_q, B_q, C_q, 1/den_q} rebuilt every iteration by
// bilinear interpolation (bitwise the oracle's op order), per-CTA delta
// maxima (max is exact, so any order gives the same stop decision).  One
// cooperative persistent launch runs the whole loop: interpolate | grid
// barrier | sweep rows | grid barrier | stop test.  Each row is reduced by one
// CTA of 256 threads in a fixed order: results are bitwise independent of
// the grid size and of row sharding.

#include <cub/block/block_scan.cuh>

namespace mu {

struct cplx {
    double x, y;
};
__device__ __forceinline__ cplx C(double x, double y) { return cplx{x, y}; }
__device__ __forceinline__ cplx operator+(cplx a, cplx b) { return C(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cplx operator-(cplx a, cplx b) { return C(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cplx operator*(cplx a, cplx b) { return C(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)); }
__device__ __forceinline__ cplx operator*(double s, cplx a) { return C(s * a.x, s * a.y); }
__device__ __forceinline__ cplx rcp(cplx a) {
    // 1/a with a scale so that |a|^2 neither overflows nor underflows
    const double s = fmax(fabs(a.x), fabs(a.y));
    const double is = 1.0 / s;
    const double ax = a.x * is, ay = a.y * is;
    const double d = 1.0 / fma(ax, ax, ay * ay);
    return C(ax * d * is, -ay * d * is);
}
// 1/a for the per-pair quotient 1/(q~^2 - p~^2): a power-of-two scale from
// the exponent bits (exact) and the Newton reciprocal instead of two IEEE
// divides (MUFU + two Newton steps, <= 1 ulp); a zero or non-finite a gives a
// non-finite result as rcp() does
__device__ __forceinline__ cplx rcp_pair(cplx a) {
    const double s = fmax(fabs(a.x), fabs(a.y));
    const int e = (__double2hiint(s) >> 20) & 0x7ff;
    const double is = __hiloint2double((2046 - e) << 20, 0);  // 2^-(e - 1023)
    const double ax = a.x * is, ay = a.y * is;
    const double d = dse::rcp_nr(fma(ax, ax, ay * ay));
    return C(ax * d * is, -ay * d * is);
}
// a*x + y for complex a, real x, complex y
__device__ __forceinline__ cplx cfma(cplx a, double x, cplx y) { return C(fma(a.x, x, y.x), fma(a.y, x, y.y)); }

struct MuArgs {
    const double *P, *P2, *p4, *Qs, *Q2, *q4, *meas_s, *meas_4, *z, *wz, *exp_tbl;
    const int *brk_s, *brk_4;
    int n_s, n_4, m_s, m_4, K;
    int row_start, row_stride, n_rows;  // owned external points: row_start + r*row_stride
    double coeff, w2, exp_c1, skip_k2, mu, z1, m0z1, xi, relax;
    double dq_eps2;
    double2* X;            // [2][3][n_ext]
    double2* NB;           // [m_int][4]: A_q, B_q, C_q, 1/den
    double* bmax;          // [gridDim][3]
    unsigned* ctr;         // [2] row tickets
    unsigned long long* err;  // [2] lowest failing row
    int* nonfinite;        // [2] some node value non-finite this iteration (no pair is skipped then)
    long long* status;     // [0] iterations done, [1] converged, [2] failed iteration, [3] failing row
    double* hist;          // (cap+1) x 4 or null
    long long* evaluated;  // pairs evaluated (diagnostic; null = not counted)
    int it_begin, it_end, sweep_only, vertex;
    int zsym;              // angular nodes and weights exactly mirror-symmetric: pair_moments walks node pairs
    // moments mode (DSE_MU_MODE_MOMENTS): per owned row r the exact-zero
    // windows (rlo [r][m_s], roff [r][m_s + 1]) and the five angular moments
    // of every evaluated pair, mom[m * mo_stride + mo_base[r] + f]
    const int* mo_rlo;
    const int* mo_roff;
    const long long* mo_base;
    double* mo_mom;
    long long mo_stride;
};

#ifndef DSE_MU_THREADS
#define DSE_MU_THREADS 256
#endif
constexpr int kThreads = DSE_MU_THREADS;
constexpr int kWarps = kThreads / 32;
#ifndef DSE_MU_UNROLL
#define DSE_MU_UNROLL 8  // config 3, bcb: unroll 2 5.46, 4 5.52, 8 5.35 ms; 3 CTAs/SM (80 regs) 5.51 ms
#endif
constexpr int kMuUnroll = DSE_MU_UNROLL;
#ifndef DSE_MU_MIRROR
#define DSE_MU_MIRROR 1
#endif
constexpr bool kMuMirror = DSE_MU_MIRROR;
#ifndef DSE_MU_MINB
#define DSE_MU_MINB 2  // CTAs per SM the register budget is cut for (A/B: scripts/mu_ab.sh)
// (20 warps per SM, which pays in the vacuum pairs kernel, does not here: at the
// 102-register cap these kernels spill 140-476 B -- config 3 direct / moments
// sweep 4.69 / 1.63 ms at 256 x 2; 320 x 2: 5.13-5.28 / 2.18; 640 x 1: 5.50-5.65 /
// 2.77; 512 x 1 (128 registers): 5.02 / 1.93 -- round 2, scripts/r02vo.sh)
#endif

// clamped linear rule of the reference along one axis (interpolation.py:71-72, :125-132)
__device__ __forceinline__ double axis_lin(bool in, double x0, double x1, double v0, double v1, double q) {
    return in ? dse::lin_eval(x0, x1, v0, v1, q) : v0;
}

__device__ void interp_node(const MuArgs& a, const double2* __restrict__ F, int js, int j4, double2& out) {
    const int n_s = a.n_s, n_4 = a.n_4;
    const int is = a.brk_s[js], i4 = a.brk_4[j4];
    const int slo = min(max(is, 0), n_s - 1), shi = min(max(is + 1, 0), n_s - 1);
    const int tlo = min(max(i4, 0), n_4 - 1), thi = min(max(i4 + 1, 0), n_4 - 1);
    const bool sin_ = is >= 0 && is < n_s - 1, tin = i4 >= 0 && i4 < n_4 - 1;
    const double xs0 = a.P2[slo], xs1 = a.P2[shi], qs = a.Q2[js];
    const double x40 = a.p4[tlo], x41 = a.p4[thi], q4 = a.q4[j4];
    const double2 v00 = F[slo * n_4 + tlo], v10 = F[shi * n_4 + tlo];
    const double2 v01 = F[slo * n_4 + thi], v11 = F[shi * n_4 + thi];
    const double f0x = axis_lin(sin_, xs0, xs1, v00.x, v10.x, qs), f1x = axis_lin(sin_, xs0, xs1, v01.x, v11.x, qs);
    const double f0y = axis_lin(sin_, xs0, xs1, v00.y, v10.y, qs), f1y = axis_lin(sin_, xs0, xs1, v01.y, v11.y, qs);
    out.x = axis_lin(tin, x40, x41, f0x, f1x, q4);
    out.y = axis_lin(tin, x40, x41, f0y, f1y, q4);
}

// Phase I: dressing values and 1/den at every internal node
__device__ void build_nodes(const MuArgs& a, const double2* __restrict__ Xin, int* flag) {
    const int n_ext = a.n_s * a.n_4, m_int = a.m_s * a.m_4;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m_int; j += gridDim.x * blockDim.x) {
        const int js = j / a.m_4, j4 = j - js * a.m_4;
        double2 v[3];
        for (int f = 0; f < 3; ++f) interp_node(a, Xin + f * n_ext, js, j4, v[f]);
        const cplx Aq = C(v[0].x, v[0].y), Bq = C(v[1].x, v[1].y), Cq = C(v[2].x, v[2].y);
        const cplx q4t = C(a.q4[j4], a.mu);
        const cplx den = a.Q2[js] * (Aq * Aq) + (q4t * q4t) * (Cq * Cq) + Bq * Bq;
        // 1/den with the pair weight's node factors folded in: coeff * (meas_s
        // meas_4) / den, the same two roundings the contraction applied per pair
        cplx r = (a.coeff * (__ldg(a.meas_s + js) * __ldg(a.meas_4 + j4))) * rcp(den);
        // a non-finite node poisons 1/den so that no pair using it is skipped
        // (the oracle's 0 * NaN = NaN flags it at every angle)
        if (!isfinite(v[0].x + v[0].y + v[1].x + v[1].y + v[2].x + v[2].y + r.x + r.y)) {
            r = C(NAN, NAN);
            atomicOr(flag, 1);
        }
        // (rejected: two more entries, B_q R and C_q q~4, hoisting those
        // per-pair products to the node: the wider staged node slot cost more
        // than the 8 operations saved, moments 1.63 -> 1.77 ms)
        double2* o = a.NB + 4 * (size_t)j;
        o[0] = v[0];
        o[1] = v[1];
        o[2] = v[2];
        o[3] = make_double2(r.x, r.y);
    }
}

// cp.async staging (moments mode): each thread copies its own next pair's
// moments and node values into its own shared-memory slot and reads only that
// slot, so a per-thread wait_group orders it (no block barrier)
constexpr int kStageDoubles = 14;  // 4 node double2 (8) + 5 moments + 1 pad: 112 B, 16-B aligned
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(dse::smem_addr(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dse::smem_addr(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

struct RowC {
    double P, P2, p4r;
    cplx p4t, Ap, Bp, Cp;
    cplx hAp, hCp;     // Ap / 2, Cp / 2 (exact): s_A = fma(1/2, Aq, Ap / 2) == (Ap + Aq) / 2 bitwise
    double mu, coeff;  // per solve (batched sweeps carry several)
};

// One (row, node) pair: angular moments, then the complex contraction.
// acc[0..5] += (A, B, C channel) * meas * coeff / den (before the row's
// division by |p|^2 and p~4).
// The five angular moments of one (row, node) pair, point by point.
__device__ __forceinline__ void pair_moments(const MuArgs& a, const RowC& rc, int js, int j4,
                                             const double2* __restrict__ zw, unsigned tbl, double mom[5]) {
    const double Qs = __ldg(a.Qs + js), Q2 = __ldg(a.Q2 + js), q4r = __ldg(a.q4 + j4);
    const double k4 = q4r - rc.p4r;
    const double PQ = rc.P * Qs;
    const double c0 = fma(k4, k4, rc.P2 + Q2);
    const dse::ExpK ek{a.exp_c1, 0.0};
    double S0 = 0.0, S1 = 0.0, T0 = 0.0, T1 = 0.0, T2 = 0.0;
    if (kMuMirror && a.zsym) {
        // mirror pairs: z_{K-1-k} = -z_k and w_{K-1-k} = w_k EXACTLY (checked
        // on the host), so r(-z) = -r(z) bit for bit and the pair shares r;
        // the odd moments take (x+ - x-) r, the even ones (x+ + x-): 20.5
        // instead of 22 FP64 instructions per point
        const int KH = a.K >> 1;
#pragma unroll kMuUnroll / 2
        for (int k = 0; k < KH; ++k) {
            const double2 zp = zw[a.K - 1 - k];
            const double r = PQ * zp.x;
            const double k2p = fma(-2.0, r, c0), k2m = fma(2.0, r, c0);
            const double Kp = dse::rcp_nr(k2p), Km = dse::rcp_nr(k2m);
            const double eKp = (zp.y * dse::exp_neg_k2(k2p, ek, tbl)) * Kp;
            const double eKm = (zp.y * dse::exp_neg_k2(k2m, ek, tbl)) * Km;
            S0 += eKp + eKm;
            S1 = fma(eKp - eKm, r, S1);
            const double eKKp = eKp * Kp, eKKm = eKm * Km;
            const double s2 = eKKp + eKKm;
            T0 += s2;
            T1 = fma(eKKp - eKKm, r, T1);
            T2 = fma(s2, r * r, T2);
        }
        if (a.K & 1) {  // the middle node, z = 0
            const double2 zk = zw[KH];
            const double r = PQ * zk.x;
            const double k2 = fma(-2.0, r, c0);
            const double K = dse::rcp_nr(k2);
            const double eK = (zk.y * dse::exp_neg_k2(k2, ek, tbl)) * K;
            S0 += eK;
            S1 = fma(eK, r, S1);
            const double eKK = eK * K;
            T0 += eKK;
            const double t = eKK * r;
            T1 += t;
            T2 = fma(t, r, T2);
        }
    } else {
#pragma unroll kMuUnroll
    for (int k = 0; k < a.K; ++k) {
        const double2 zk = zw[k];
        const double r = PQ * zk.x;
        const double k2 = fma(-2.0, r, c0);
        const double K = dse::rcp_nr(k2);
        const double e = zk.y * dse::exp_neg_k2(k2, ek, tbl);
        const double eK = e * K;
        S0 += eK;
        S1 = fma(eK, r, S1);
        const double eKK = eK * K;
        T0 += eKK;
        const double t = eKK * r;
        T1 += t;
        T2 = fma(t, r, T2);
    }
    }
    mom[0] = S0;
    mom[1] = S1;
    mom[2] = T0;
    mom[3] = T1;
    mom[4] = T2;
}

// The complex contraction of a pair's moments; acc[0..5] += (A, B, C) * meas
// * coeff / den (before the row's division by |p|^2 and p~4).
// LATE_B: apply the B channel's common factor Bq after the contraction
// (fewer operations: config 3 direct 5.16 -> 5.13 ms, batched S=4 5.11 ->
// 5.01 ms).  With the trimmed zero terms and rcp_pair, 5.28 -> 5.13 ms direct,
// 2.06 -> 1.83 ms moments, 5.59 -> 5.01 ms batched (S=4).
#ifndef DSE_MU_FACTORED
#define DSE_MU_FACTORED 1  // regrouped A/C channels for the vertices without Delta_A/Delta_C
#endif
constexpr bool kMuFactored = DSE_MU_FACTORED;
#ifndef DSE_MU_LATE_B
#define DSE_MU_LATE_B 1
#endif
template <int V, bool LATE_B = DSE_MU_LATE_B>
__device__ __forceinline__ void pair_contract(const MuArgs& a, const RowC& rc, int js, int j4, const double2* vn,
                                              const double mom[5], double acc[6]) {
    const double Q2 = __ldg(a.Q2 + js), q4r = __ldg(a.q4 + j4);
    const double k4 = q4r - rc.p4r;
    const double S0 = mom[0], S1 = mom[1], T0 = mom[2], T1 = mom[3], T2 = mom[4];
    const double2 vA = vn[0], vB = vn[1], vC = vn[2], vR = vn[3];
    const cplx Aq = C(vA.x, vA.y), Bq = C(vB.x, vB.y), Cq = C(vC.x, vC.y);
    const cplx q4t = C(q4r, rc.mu);
    const cplx t4 = C(q4r + rc.p4r, 2.0 * rc.mu);
    const double P2 = rc.P2;
    const double kts = Q2 - P2;
    // q~^2 - p~^2 = k.t (complex), real part as (Q2 - P2) + k4 (q4 + p4)
    const cplx kt = C(fma(k4, q4r + rc.p4r, kts), 2.0 * rc.mu * k4);
    // experiment hook (DSE_MU_DQ_EPS2, default 0 = the exact quotient):
    // Tikhonov-regularised 1/(q~^2 - p~^2) = conj(d) / (|d|^2 + eps^2)
    const cplx rkt = a.dq_eps2 > 0.0 ? (1.0 / fma(kt.x, kt.x, fma(kt.y, kt.y, a.dq_eps2))) * C(kt.x, -kt.y) : rcp_pair(kt);
    const cplx sA = C(fma(0.5, Aq.x, rc.hAp.x), fma(0.5, Aq.y, rc.hAp.y));
    const cplx sC = C(fma(0.5, Cq.x, rc.hCp.x), fma(0.5, Cq.y, rc.hCp.y));
    const cplx dA = (Aq - rc.Ap) * rkt, dC = (Cq - rc.Cp) * rkt, dB = (Bq - rc.Bp) * rkt;
    const cplx tau0 = 2.0 * sA + sC;
    const cplx tau1 = (k4 * k4) * (sA - sC);
    const cplx Cq_q4t = Cq * q4t;
    const cplx akQ = Q2 * Aq + k4 * Cq_q4t;                       // k.Q = akQ - Aq r
    const cplx akQp = Q2 * (sA * Aq) + k4 * (sC * Cq_q4t);        // k.Q' = akQp - sA Aq r
    const cplx nu1 = Aq * dA;
    const cplx Cq_q4t_t4 = Cq_q4t * t4;
    const cplx nu0 = Q2 * nu1 + Cq_q4t_t4 * dC;                   // Q.D = nu0 + nu1 r
    const cplx delta0 = (P2 + Q2) * dA + (t4 * t4) * dC;          // u.D = delta0 + 2 dA r - psi K
    const cplx psi = (kts * dA + k4 * (dC * t4)) * kt;
    const cplx eta0 = Q2 * Aq + Cq_q4t_t4;                        // Q.t = eta0 + Aq r
    const cplx sAAq = sA * Aq;
    // vertex structures by mode (DSE_MU_VERTEX_*): Sigma parts always, the
    // Delta_A/Delta_C parts in the A/C channels (fac), in the B channel (fb),
    // Delta_B in the B channel (fdb); V is a compile-time constant.
    constexpr bool fac = V == DSE_MU_VERTEX_BC;
    constexpr bool fb = V != DSE_MU_VERTEX_BC1;
    constexpr bool fdb = V == DSE_MU_VERTEX_BC;
    const cplx zero = C(0.0, 0.0);
    cplx FA, FC;
    if constexpr (!fac && kMuFactored) {
        // without the Delta_A/Delta_C parts the A and C channels regroup over
        // moment combinations (exact algebra on the general form below):
        //   F_A = Aq sC S1 + lam0 (T1 - P2 T0) + sA Aq 2 (P2 T1 - T2) + Aq tau1 T1
        //   F_C = Cq q~4 ((2 sA - sC) S0 + k4^2 (sA + sC) T0) + k4 (Q2 T0 - T1) (sA + sC) Aq
        // with lam0 = 2 Q2 sA Aq + k4 (sA + sC) Cq q~4
        const cplx ssum = sA + sC;
        const double k42 = k4 * k4;
        const cplx lam0 = (2.0 * Q2) * sAAq + k4 * (ssum * Cq_q4t);
        const double U = fma(-P2, T0, T1);
        const double Vv = 2.0 * fma(P2, T1, -T2);
        const double W = fma(Q2, T0, -T1);
        FA = cfma(Aq * sC, S1, cfma(lam0, U, cfma(sAAq, Vv, T1 * (Aq * tau1))));
        FC = Cq_q4t * cfma(2.0 * sA - sC, S0, (k42 * T0) * ssum) + (k4 * W) * (ssum * Aq);
    } else {
        // A channel (e = p_vec): F_A = cA00 + cA01 r + K (cA10 + cA11 r + cA12 r^2)
        const cplx lam0 = akQp + sA * akQ;
        const cplx cA00 = fac ? (-0.5 * P2) * (nu0 + dA * eta0) : zero;
        cplx cA01 = Aq * sC;  // Aq tau0 - 2 sA Aq
        cplx cA10 = (-P2) * lam0;
        cplx cA11 = lam0 + (2.0 * P2) * sAAq + Aq * tau1;
        if (fac) {
            cA01 = cA01 - 0.5 * (nu0 + P2 * nu1 - Aq * delta0 + dA * (eta0 + P2 * Aq));
            cA10 = cA10 - (0.5 * P2) * (kt * (nu0 - dA * akQ));
            cA11 = cA11 - 0.5 * (kt * (P2 * nu1 - nu0) + Aq * psi + (dA * kt) * (P2 * Aq - akQ));
        }
        const cplx cA12 = -2.0 * sAAq;
        // C channel (e = unit 4): F_C = cC00 + cC01 r + K (cC10 + cC11 r)
        const cplx lam0c = akQp + sC * akQ;
        const cplx lam1c = (sA + sC) * Aq;
        const cplx dCt4 = dC * t4;
        cplx cC00 = Cq_q4t * (tau0 - 2.0 * sC);
        cplx cC01 = zero;
        cplx cC10 = k4 * lam0c + Cq_q4t * tau1;
        cplx cC11 = (-k4) * lam1c;
        if (fac) {
            cC00 = cC00 - 0.5 * (t4 * nu0 - Cq_q4t * delta0 + dCt4 * eta0);
            cC01 = -0.5 * (t4 * nu1 - 2.0 * (Cq_q4t * dA) + dCt4 * Aq);
            cC10 = cC10 - 0.5 * (Cq_q4t * psi - kt * (k4 * nu0 + dCt4 * akQ));
            cC11 = cC11 - 0.5 * (kt * (dCt4 * Aq - k4 * nu1));
        }

        const cplx FA0 = cfma(cA01, S1, cfma(cA10, T0, cfma(cA11, T1, T2 * cA12)));
        FA = fac ? cfma(cA00, S0, FA0) : FA0;
        const cplx FC0 = cfma(cC10, T0, T1 * cC11);
        FC = cfma(cC00, S0, fac ? cfma(cC01, S1, FC0) : FC0);
    }
    // B channel: F_B = cB00 + cB01 r + K (cB10 + cB11 r); without Delta_B
    // every coefficient carries the factor Bq, which is applied once (with
    // the scale) after the moments are contracted
    constexpr bool late_b = LATE_B && !fdb;
    cplx cB00, cB01 = zero, cB10, cB11 = zero;
    if (fb) {
        cB00 = tau0 + 0.5 * delta0;
        cB01 = dA;
        cB10 = tau1 - 0.5 * psi;
    } else {
        cB00 = tau0;
        cB10 = tau1;
    }
    if (!late_b) {
        cB00 = Bq * cB00;
        cB01 = Bq * cB01;
        cB10 = Bq * cB10;
    }
    if (fdb) {
        cB00 = cB00 - dB * eta0;
        cB01 = cB01 - dB * Aq;
        cB10 = cB10 + dB * (kt * akQ);
        cB11 = -1.0 * (dB * (kt * Aq));
    }
    // contract with the moments, scale by meas * coeff / den
    // (terms whose coefficient is identically zero for this vertex are not
    // formed: 0 * moment would only matter for a non-finite moment, and a
    // non-finite moment already makes the other terms non-finite)
    const cplx FB0 = fdb ? cfma(cB10, T0, T1 * cB11) : T0 * cB10;
    const cplx FB = cfma(cB00, S0, fb ? cfma(cB01, S1, FB0) : FB0);
    const cplx rd = C(vR.x, vR.y);  // coeff * meas / den (build_nodes)
    const cplx gA = FA * rd, gB = FB * (late_b ? Bq * rd : rd), gC = FC * rd;
    acc[0] += gA.x; acc[1] += gA.y;
    acc[2] += gB.x; acc[3] += gB.y;
    acc[4] += gC.x; acc[5] += gC.y;
}

template <int V>
__device__ __forceinline__ void pair_contrib(const MuArgs& a, const RowC& rc, int js, int j4,
                                             const double2* __restrict__ zw, unsigned tbl, double acc[6]) {
    // node values first: their latency hides behind the angular loop
    const double2* nb = a.NB + 4 * (size_t)(js * a.m_4 + j4);
    const double2 vn[4] = {nb[0], nb[1], nb[2], nb[3]};
    double mom[5];
    pair_moments(a, rc, js, j4, zw, tbl, mom);
    pair_contract<V>(a, rc, js, j4, vn, mom, acc);
}

__device__ __forceinline__ double hyp(double x, double y) { return hypot(x, y); }

// relax * new + (1 - relax) * old per component, each operation rounded once
__device__ __forceinline__ double2 mu_blend(double relax, double2 n, double2 o) {
    const double om = __dsub_rn(1.0, relax);
    return make_double2(__dadd_rn(__dmul_rn(relax, n.x), __dmul_rn(om, o.x)),
                        __dadd_rn(__dmul_rn(relax, n.y), __dmul_rn(om, o.y)));
}

// Multi-GPU (finite_mu.solve_mu_sharded): pack the owned rows of the new
// state into send[3][per] (complex), and rebuild the full state from the
// gathered recv[world][3][per] with the blend and the per-function max
// |new - old| (one CTA; max is exact, so order-free).
__global__ void mu_pack_kernel(const double2* __restrict__ Xn, int n_ext, int r0, int w, int per,
                               double2* __restrict__ send) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < per; k += gridDim.x * blockDim.x) {
        const int i = r0 + k * w;
        for (int f = 0; f < 3; ++f) send[f * per + k] = i < n_ext ? Xn[(size_t)f * n_ext + i] : make_double2(0.0, 0.0);
    }
}

__global__ void __launch_bounds__(1024) mu_assemble_kernel(const double2* __restrict__ recv, int world, int per,
                                                           int n_ext, double relax, double2* __restrict__ X,
                                                           double* __restrict__ delta) {
    __shared__ double red[3][32];
    double d[3] = {0.0, 0.0, 0.0};
    for (int i = threadIdx.x; i < n_ext; i += blockDim.x) {
        const int r = i % world, k = i / world;
        for (int f = 0; f < 3; ++f) {
            double2 nv = recv[((size_t)r * 3 + f) * per + k];
            const double2 ov = X[(size_t)f * n_ext + i];
            if (relax != 1.0) nv = mu_blend(relax, nv, ov);
            d[f] = fmax(d[f], hyp(nv.x - ov.x, nv.y - ov.y));
            X[(size_t)f * n_ext + i] = nv;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int f = 0; f < 3; ++f) {
        double v = d[f];
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) red[f][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double v = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[threadIdx.x][w]);
        delta[threadIdx.x] = v;
    }
}


// The exact-zero windows of one row: per radial node js the evaluated q4
// form one window around p4.  Fills rlo[m_s], roff[m_s + 1]
// (shared) and returns the row's number of evaluated pairs.  all = evaluate
// every pair (a non-finite node must reach the sums).
template <class ScanT>
__device__ int row_windows(const MuArgs& a, const RowC& rc, bool all, const double* q4s, int* rlo, int* roff,
                           typename ScanT::TempStorage& scan_tmp, int& s_carry) {
    const int tid = threadIdx.x;
    if (tid == 0) s_carry = 0;
    for (int base = 0; base < a.m_s; base += kThreads) {
        const int js = base + tid;
        int len = 0;
        if (js < a.m_s) {
            int lo = 0, hi = a.m_4;
            if (!all) {
                const double dPQ = rc.P - __ldg(a.Qs + js);
                const double d2 = a.skip_k2 - dPQ * dPQ;
                if (d2 < 0.0) {
                    hi = 0;
                } else {
                    const double half = sqrt(d2) * (1.0 + 1e-12) + 1e-300;
                    const double x0 = rc.p4r - half, x1 = rc.p4r + half;
                    int l = 0, h = a.m_4;  // first q4 >= x0
                    while (l < h) { const int mm = (l + h) >> 1; if (q4s[mm] < x0) l = mm + 1; else h = mm; }
                    lo = l;
                    h = a.m_4;             // first q4 > x1
                    while (l < h) { const int mm = (l + h) >> 1; if (q4s[mm] <= x1) l = mm + 1; else h = mm; }
                    hi = l;
                }
            }
            len = max(hi - lo, 0);
            rlo[js] = lo;
        }
        int ex;
        __syncthreads();  // s_carry written
        const int carry = s_carry;
        ScanT(scan_tmp).ExclusiveSum(len, ex);
        if (js < a.m_s) roff[js] = carry + ex;
        __syncthreads();
        if (tid == kThreads - 1) s_carry = carry + ex + len;
    }
    __syncthreads();
    const int total = s_carry;
    if (tid == 0) roff[a.m_s] = total;
    __syncthreads();
    return total;
}

// node js of flat pair index f: fixed-trip binary search over roff (the
// warp's lanes stay converged through the pair body)
__device__ __forceinline__ int node_of(const int* roff, int m_s, int top, int f) {
    int js = 0;
    for (int step = top >> 1; step > 0; step >>= 1) js = (js + step < m_s && roff[js + step] <= f) ? js + step : js;
    return js;
}

__device__ __forceinline__ RowC row_consts(const MuArgs& a, const double2* Xin, int n_ext, int i) {
    const int is = i / a.n_4, i4 = i - is * a.n_4;
    RowC rc;
    rc.P = a.P[is];
    rc.P2 = a.P2[is];
    rc.p4r = a.p4[i4];
    rc.p4t = C(rc.p4r, a.mu);
    const double2 va = Xin[i], vb = Xin[n_ext + i], vc = Xin[2 * n_ext + i];
    rc.Ap = C(va.x, va.y);
    rc.Bp = C(vb.x, vb.y);
    rc.Cp = C(vc.x, vc.y);
    rc.hAp = 0.5 * rc.Ap;
    rc.hCp = 0.5 * rc.Cp;
    rc.mu = a.mu;
    rc.coeff = a.coeff;
    return rc;
}

// Moments mode, pass 1: every owned row's windows (geometry only: P, p4,
// the |q| and q4 nodes, omega) into the global tables and its pair count.
__global__ void __launch_bounds__(kThreads) mu_windows_kernel(MuArgs a, int* rlo_g, int* roff_g, long long* tot) {
    extern __shared__ __align__(16) double sm[];
    double* q4s = sm;
    int* rlo = reinterpret_cast<int*>(q4s + a.m_4);
    int* roff = rlo + a.m_s;
    using Scan = cub::BlockScan<int, kThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int s_carry;
    for (int k = threadIdx.x; k < a.m_4; k += kThreads) q4s[k] = __ldg(a.q4 + k);
    __syncthreads();
    for (int r = blockIdx.x; r < a.n_rows; r += gridDim.x) {
        const int i = a.row_start + r * a.row_stride;
        const int is = i / a.n_4, i4 = i - is * a.n_4;
        RowC rc{};
        rc.P = a.P[is];
        rc.P2 = a.P2[is];
        rc.p4r = a.p4[i4];
        const int total = row_windows<Scan>(a, rc, false, q4s, rlo, roff, scan_tmp, s_carry);
        for (int js = threadIdx.x; js < a.m_s; js += kThreads) rlo_g[(size_t)r * a.m_s + js] = rlo[js];
        for (int js = threadIdx.x; js <= a.m_s; js += kThreads) roff_g[(size_t)r * (a.m_s + 1) + js] = roff[js];
        if (threadIdx.x == 0) tot[r] = total;
        __syncthreads();
    }
}

// Moments mode, pass 2: the five moments of every evaluated pair (the same
// pair_moments as the direct sweep: the moments are bitwise those the direct
// sweep forms every iteration).
__global__ void __launch_bounds__(kThreads) mu_moments_build_kernel(MuArgs a) {
    extern __shared__ __align__(16) double sm[];
    double* etbl = sm;
    double2* zw = reinterpret_cast<double2*>(sm + (1 << dse::kExpTableBits));
    int* roff = reinterpret_cast<int*>(zw + a.K);
    for (int i = threadIdx.x; i < (1 << dse::kExpTableBits); i += kThreads) etbl[i] = __ldg(a.exp_tbl + i);
    for (int k = threadIdx.x; k < a.K; k += kThreads) zw[k] = make_double2(__ldg(a.z + k), __ldg(a.wz + k));
    __syncthreads();
    const unsigned tbl = dse::smem_addr(etbl);
    int top = 1;
    while (top < a.m_s) top <<= 1;
    for (int r = blockIdx.x; r < a.n_rows; r += gridDim.x) {
        const int i = a.row_start + r * a.row_stride;
        const int is = i / a.n_4, i4 = i - is * a.n_4;
        RowC rc{};
        rc.P = a.P[is];
        rc.P2 = a.P2[is];
        rc.p4r = a.p4[i4];
        for (int js = threadIdx.x; js <= a.m_s; js += kThreads) roff[js] = a.mo_roff[(size_t)r * (a.m_s + 1) + js];
        __syncthreads();
        const int total = roff[a.m_s];
        const long long base = a.mo_base[r];
        for (int f0 = 0; f0 < total; f0 += kThreads) {
            const int f = min(f0 + threadIdx.x, total - 1);
            const int js = node_of(roff, a.m_s, top, f);
            const int j4 = a.mo_rlo[(size_t)r * a.m_s + js] + (f - roff[js]);
            __syncwarp();
            double mom[5];
            pair_moments(a, rc, js, j4, zw, tbl, mom);
            if (f0 + threadIdx.x < total)
                for (int q = 0; q < 5; ++q) a.mo_mom[q * a.mo_stride + base + f] = mom[q];
        }
        __syncthreads();
    }
}

#ifndef DSE_MU_MOM_PF_NB
// moments mode: prefetch the next pair's node values with its moments (1) or
// load them at use (0): config 3, 1.97 (early B) / 2.32 (late B) vs 1.83 ms
#define DSE_MU_MOM_PF_NB 0
#endif
constexpr bool kMomPfNB = DSE_MU_MOM_PF_NB;
#ifndef DSE_MU_MOM_STAGE
// moments mode: cp.async staging of the next pair into shared memory
// (supersedes the register prefetch above; spills 88 -> 32 B).  Config 3:
// 1.84 -> 1.79 ms with the node values L1-cached (.ca); bypassing L1 (.cg)
// was slower, 2.04 ms -- the node values are reused from L1 across pairs
#define DSE_MU_MOM_STAGE 1
#endif
constexpr bool kMomStage = DSE_MU_MOM_STAGE;
#ifndef DSE_MU_MOM_MINB
#define DSE_MU_MOM_MINB DSE_MU_MINB
#endif
template <int V, bool MOM>
__global__ void __launch_bounds__(kThreads, MOM ? DSE_MU_MOM_MINB : DSE_MU_MINB) mu_solve_kernel(MuArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double smem[];
    double* etbl = smem;                                           // 2^bits
    double2* zw = reinterpret_cast<double2*>(smem + (1 << dse::kExpTableBits));  // K
    double* red = smem + (1 << dse::kExpTableBits) + 2 * a.K;      // kWarps * 6
    double* q4s = red + kWarps * 6;                                // m_4
    int* rlo = reinterpret_cast<int*>(q4s + a.m_4);                // m_s: first evaluated j4 per js
    int* roff = rlo + a.m_s;                                       // m_s + 1: flat offsets
    // moments mode: 2 x kThreads staging slots, 16-B aligned after roff
    double* mom_stage = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(roff + a.m_s + 1) + 15) & ~uintptr_t(15));
    __shared__ unsigned s_row;
    __shared__ int s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < (1 << dse::kExpTableBits); i += kThreads) etbl[i] = __ldg(a.exp_tbl + i);
    for (int k = tid; k < a.K; k += kThreads) zw[k] = make_double2(__ldg(a.z + k), __ldg(a.wz + k));
    for (int k = tid; k < a.m_4; k += kThreads) q4s[k] = __ldg(a.q4 + k);
    __syncthreads();
    const unsigned tbl = dse::smem_addr(etbl);
    const int n_ext = a.n_s * a.n_4;
    long long it_done = a.it_begin;
    bool converged = false;
    for (int it = a.it_begin; it < a.it_end; ++it) {
        const int cur = it & 1;
        const double2* Xin = a.X + (size_t)cur * 3 * n_ext;
        double2* Xout = a.X + (size_t)(cur ^ 1) * 3 * n_ext;
        if (blockIdx.x == 0 && tid == 0) {
            a.ctr[cur ^ 1] = 0u;
            a.err[cur ^ 1] = ~0ull;
            a.nonfinite[cur ^ 1] = 0;
        }
        build_nodes(a, Xin, a.nonfinite + cur);
        grid.sync();
        // ---- phase S: rows by ticket, one CTA per row ----
        double dmax[3] = {0.0, 0.0, 0.0};
        long long pairs = 0;
        for (;;) {
            if (tid == 0) s_row = atomicAdd(a.ctr + cur, 1u);
            __syncthreads();
            const unsigned r = s_row;
            __syncthreads();
            if (r >= (unsigned)a.n_rows) break;
            const int i = a.row_start + (int)r * a.row_stride;
            const RowC rc = row_consts(a, Xin, n_ext, i);
            const double2 va = Xin[i], vb = Xin[n_ext + i], vc = Xin[2 * n_ext + i];
            const bool all = a.nonfinite[cur] != 0;  // a non-finite node must reach the sum
            int total;
            if (MOM) {
                // precomputed windows; a non-finite node fails the lowest owned
                // row directly (every row's reference sum contains it), the
                // location comes from the direct per-point pass
                if (all) {
                    if (tid == 0) atomicMin(a.err + cur, (unsigned long long)a.row_start);
                    continue;
                }
                for (int js = tid; js < a.m_s; js += kThreads) rlo[js] = __ldg(a.mo_rlo + (size_t)r * a.m_s + js);
                for (int js = tid; js <= a.m_s; js += kThreads)
                    roff[js] = __ldg(a.mo_roff + (size_t)r * (a.m_s + 1) + js);
                __syncthreads();
                total = roff[a.m_s];
            } else if (!all && a.mo_rlo) {
                // the precomputed windows of this row (geometry + omega only)
                for (int js = tid; js < a.m_s; js += kThreads) rlo[js] = __ldg(a.mo_rlo + (size_t)r * a.m_s + js);
                for (int js = tid; js <= a.m_s; js += kThreads)
                    roff[js] = __ldg(a.mo_roff + (size_t)r * (a.m_s + 1) + js);
                __syncthreads();
                total = roff[a.m_s];
            } else {
                using Scan = cub::BlockScan<int, kThreads>;
                __shared__ typename Scan::TempStorage scan_tmp;
                total = row_windows<Scan>(a, rc, all, q4s, rlo, roff, scan_tmp, s_carry);
            }
            double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            // the warp's lanes stay converged through the pair body: the node
            // of flat index f is found by a fixed-trip binary search over the
            // offsets (a data-dependent walk here split the warps, 6 of 32
            // lanes active on average)
            int top = 1;
            while (top < a.m_s) top <<= 1;
            const long long mbase = MOM ? __ldg(a.mo_base + r) : 0;
            if (MOM && kMomStage) {
                // the next pair's node values and moments are copied into this
                // thread's shared-memory slot (cp.async, double-buffered)
                // while the current pair is contracted
                double* const slot0 = mom_stage + (size_t)tid * kStageDoubles;
                constexpr size_t kBufStride = (size_t)kThreads * kStageDoubles;
                int js = 0, j4 = 0;
                if (total > 0) {
                    const int f = min(tid, total - 1);
                    js = node_of(roff, a.m_s, top, f);
                    j4 = rlo[js] + (f - roff[js]);
                    const double2* nb = a.NB + 4 * (size_t)(js * a.m_4 + j4);
                    for (int q = 0; q < 4; ++q) cp_async16(slot0 + 2 * q, nb + q);
                    for (int q = 0; q < 5; ++q) cp_async8(slot0 + 8 + q, a.mo_mom + q * a.mo_stride + mbase + f);
                    cp_async_commit();
                }
                int buf = 0;
                for (int f0 = 0; f0 < total; f0 += kThreads) {
                    int jsn = js, j4n = j4;
                    if (f0 + kThreads < total) {
                        const int fn = min(f0 + kThreads + tid, total - 1);
                        jsn = node_of(roff, a.m_s, top, fn);
                        j4n = rlo[jsn] + (fn - roff[jsn]);
                        DCHECK(jsn >= 0 && jsn < a.m_s && j4n >= 0 && j4n < a.m_4 && mbase + fn < a.mo_stride, 23);
                        double* sl = slot0 + (buf ^ 1) * kBufStride;
                        const double2* nb = a.NB + 4 * (size_t)(jsn * a.m_4 + j4n);
                        for (int q = 0; q < 4; ++q) cp_async16(sl + 2 * q, nb + q);
                        for (int q = 0; q < 5; ++q) cp_async8(sl + 8 + q, a.mo_mom + q * a.mo_stride + mbase + fn);
                        cp_async_commit();
                        cp_async_wait<1>();
                    } else {
                        cp_async_wait<0>();
                    }
                    const double* sl = slot0 + buf * kBufStride;
                    const double2* sv = reinterpret_cast<const double2*>(sl);
                    const double2 vn[4] = {sv[0], sv[1], sv[2], sv[3]};
                    const double mom[5] = {sl[8], sl[9], sl[10], sl[11], sl[12]};
                    __syncwarp();
                    double part[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                    pair_contract<V>(a, rc, js, j4, vn, mom, part);
                    if (f0 + tid < total)
                        for (int c = 0; c < 6; ++c) acc[c] += part[c];
                    js = jsn;
                    j4 = j4n;
                    buf ^= 1;
                }
            } else if (MOM) {
                // the moment stream is read once per iteration from HBM: the
                // next pair's moments are loaded before this pair is
                // contracted (software pipelining over the row)
                int f = min(tid, total - 1);
                int js = node_of(roff, a.m_s, top, f), j4 = rlo[js] + (f - roff[js]);
                double mom[5];
                double2 vn[4];
                if (total > 0) {
                    for (int q = 0; q < 5; ++q) mom[q] = __ldcs(a.mo_mom + q * a.mo_stride + mbase + f);
                    if (kMomPfNB) {
                        const double2* nb = a.NB + 4 * (size_t)(js * a.m_4 + j4);
                        for (int q = 0; q < 4; ++q) vn[q] = nb[q];
                    }
                }
                for (int f0 = 0; f0 < total; f0 += kThreads) {
                    const int fn = min(f0 + kThreads + tid, total - 1);
                    const int jsn = node_of(roff, a.m_s, top, fn), j4n = rlo[jsn] + (fn - roff[jsn]);
                    DCHECK(jsn >= 0 && jsn < a.m_s && j4n >= 0 && j4n < a.m_4 && mbase + fn < a.mo_stride, 23);
                    double momn[5];
                    double2 vnn[4];
                    if (f0 + kThreads < total) {
                        for (int q = 0; q < 5; ++q) momn[q] = __ldcs(a.mo_mom + q * a.mo_stride + mbase + fn);
                        if (kMomPfNB) {
                            const double2* nb = a.NB + 4 * (size_t)(jsn * a.m_4 + j4n);
                            for (int q = 0; q < 4; ++q) vnn[q] = nb[q];
                        }
                    }
                    if (!kMomPfNB) {  // node values (L1/L2-resident) loaded at use
                        const double2* nb = a.NB + 4 * (size_t)(js * a.m_4 + j4);
                        for (int q = 0; q < 4; ++q) vn[q] = nb[q];
                    }
                    __syncwarp();
                    double part[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                    pair_contract<V>(a, rc, js, j4, vn, mom, part);
                    if (f0 + tid < total)
                        for (int c = 0; c < 6; ++c) acc[c] += part[c];
                    js = jsn;
                    j4 = j4n;
                    for (int q = 0; q < 5; ++q) mom[q] = momn[q];
                    if (kMomPfNB)
                        for (int q = 0; q < 4; ++q) vn[q] = vnn[q];
                }
            } else {
                for (int f0 = 0; f0 < total; f0 += kThreads) {
                    const int f = min(f0 + tid, total - 1);
                    const int js = node_of(roff, a.m_s, top, f);
                    const int j4 = rlo[js] + (f - roff[js]);
                    __syncwarp();
                    double part[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                    pair_contrib<V>(a, rc, js, j4, zw, tbl, part);
                    if (f0 + tid < total)
                        for (int c = 0; c < 6; ++c) acc[c] += part[c];
                }
            }
            pairs += (tid == 0) ? total : 0;
            // fixed-order block reduction
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                double v = acc[c];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) red[warp * 6 + c] = v;
            }
            __syncthreads();
            if (tid == 0) {
                double s[6];
                for (int c = 0; c < 6; ++c) {
                    double v = red[c];
                    for (int w = 1; w < kWarps; ++w) v += red[w * 6 + c];
                    s[c] = v;
                }
                // A' = z1 + sum_A / |p|^2 ; B' = m0 z1 + sum_B ; C' = z1 + sum_C / p~4
                double2 An = make_double2(a.z1 + s[0] / rc.P2, s[1] / rc.P2);
                double2 Bn = make_double2(a.m0z1 + s[2], s[3]);
                const cplx cn = C(s[4], s[5]) * rcp(rc.p4t);
                double2 Cn = make_double2(a.z1 + cn.x, cn.y);
                if (a.relax != 1.0) {  // solver.py:249-251, one rounding per op (as mu_blend)
                    An = mu_blend(a.relax, An, va);
                    Bn = mu_blend(a.relax, Bn, vb);
                    Cn = mu_blend(a.relax, Cn, vc);
                }
                const bool fin = isfinite(An.x) && isfinite(An.y) && isfinite(Bn.x) && isfinite(Bn.y) &&
                                 isfinite(Cn.x) && isfinite(Cn.y);
                if (!fin) atomicMin(a.err + cur, (unsigned long long)i);
                Xout[i] = An;
                Xout[n_ext + i] = Bn;
                Xout[2 * n_ext + i] = Cn;
                dmax[0] = fmax(dmax[0], hyp(An.x - va.x, An.y - va.y));
                dmax[1] = fmax(dmax[1], hyp(Bn.x - vb.x, Bn.y - vb.y));
                dmax[2] = fmax(dmax[2], hyp(Cn.x - vc.x, Cn.y - vc.y));
            }
        }
        if (tid == 0) {
            a.bmax[3 * blockIdx.x + 0] = dmax[0];
            a.bmax[3 * blockIdx.x + 1] = dmax[1];
            a.bmax[3 * blockIdx.x + 2] = dmax[2];
        }
        if (a.evaluated) {
            for (int o = 16; o > 0; o >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
            if (lane == 0 && it == a.it_begin) atomicAdd((unsigned long long*)a.evaluated, (unsigned long long)pairs);
        }
        grid.sync();
        // ---- stop test (every CTA, identical decision) ----
        it_done = it + 1;
        if (a.err[cur] != ~0ull) {
            if (blockIdx.x == 0 && tid == 0) {
                a.status[2] = it + 1;
                a.status[3] = (long long)a.err[cur];
            }
            break;
        }
        double d[3] = {0.0, 0.0, 0.0};
        for (int b = 0; b < (int)gridDim.x; ++b)
            for (int c = 0; c < 3; ++c) d[c] = fmax(d[c], a.bmax[3 * b + c]);
        if (blockIdx.x == 0 && tid == 0 && a.hist) {
            double* h = a.hist + 4 * (size_t)(it + 1);
            h[0] = double(it + 1);
            h[1] = d[0];
            h[2] = d[1];
            h[3] = d[2];
        }
        if (!a.sweep_only && d[0] < a.xi && d[1] < a.xi && d[2] < a.xi) {
            converged = true;
            break;
        }
        // the next iteration's tickets/err slots were reset before this
        // iteration's first barrier; bmax is rewritten only after the next
        // barrier, so it is safe to fall through
    }
    if (blockIdx.x == 0 && tid == 0) {
        a.status[0] = it_done;
        a.status[1] = converged ? 1 : 0;
    }
}


// ---- batched solves (BASELINE config 4): S independent solves on one grid in
// moments mode.  Every pair's five moments are read once and contracted for
// each solve still iterating (each solve has its own state, node table, mu and
// coefficient); the per-solve arithmetic and reduction order are those of
// mu_solve_kernel<V, true>, so each solve's sweep is bitwise its standalone
// moments-mode sweep.  One cooperative launch runs the whole successive
// approximation of the group (iteration.py:18-40 per solve: max-norm deltas
// of A, B, C, strict stop, cap -> not converged): a solve that has stopped is
// neither swept nor written again (its state stays in the half its last sweep
// wrote), and the launch ends when every solve has stopped or one has failed.
// Sweep-only mode (stop = 0, one iteration) is dse_mu_batch_sweep.
// (rejected: cp.async staging of the next pair as in mu_solve_kernel<V, true>
// -- moments only for S = 4, moments + both node tables for S = 2 -- measured
// slower, S = 2 2.73 -> 3.15 ms, S = 4 5.02 -> 5.32 ms per sweep)
constexpr int kMuMaxBatch = 4;
struct MuBatch {
    double2* Xh[2];       // halves [S][3][n_ext]: iteration it reads Xh[it & 1], writes Xh[(it & 1) ^ 1]
    double2* NB;          // [S][m_int][4]
    unsigned long long* err;  // [2][S] lowest failing row (per iteration parity)
    int* nonfinite;       // [2][S]
    double* bmax;         // [gridDim][S][3] per-CTA delta maxima
    double* hist;         // [S][hist_stride][4] (n, |dA|, |dB|, |dC|) or null
    long long hist_stride;
    long long* status;    // [S][4]: iterations, converged, failed iteration, failing row
    int stop;             // 1: stop test (solve), 0: sweep only
    double mu[kMuMaxBatch], coeff[kMuMaxBatch], z1[kMuMaxBatch], m0z1[kMuMaxBatch], xi[kMuMaxBatch];
    long long cap[kMuMaxBatch];
};

#ifndef DSE_MU_BATCH_MINB
#define DSE_MU_BATCH_MINB DSE_MU_MINB
#endif
#ifndef DSE_MU_BATCH_SMACC
#define DSE_MU_BATCH_SMACC 0  // per-thread accumulators of S = 4 in shared memory (frees 48 registers)
#endif
constexpr bool kBatchSmAcc = DSE_MU_BATCH_SMACC;
#ifndef DSE_MU_BATCH_PF
#define DSE_MU_BATCH_PF 2  // prefetch the next chunk's moments: 0 off, 1 into L1, 2 into L2 (S = 4 sweep 4.50 -> 4.42 ms)
#endif
constexpr int kBatchPf = DSE_MU_BATCH_PF;
#ifndef DSE_MU_BATCH_PFNB
#define DSE_MU_BATCH_PFNB 2  // also prefetch the next chunk's node values: 0 off, 1 always, 2 for S = 2 only
#endif                       // (S = 2 2.56 -> 2.46 ms; S = 4 4.42 -> 4.46 ms, register pressure)
template <int S>
__host__ __device__ constexpr bool batch_pfnb() {
    return DSE_MU_BATCH_PF && (DSE_MU_BATCH_PFNB == 1 || (DSE_MU_BATCH_PFNB == 2 && S == 2));
}
template <int S>
__host__ __device__ constexpr size_t batch_acc_doubles() { return (kBatchSmAcc && S == 4) ? (size_t)S * 6 * kThreads : 0; }

template <int V, int S>
__global__ void __launch_bounds__(kThreads, DSE_MU_BATCH_MINB) mu_batch_kernel(MuArgs a, MuBatch b) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double smem[];
    constexpr bool smacc = batch_acc_doubles<S>() > 0;
    double* sacc = smem;                                           // [S*6][kThreads] (smacc)
    double* red = smem + batch_acc_doubles<S>();                   // kWarps * 6 * S
    int* rlo = reinterpret_cast<int*>(red + kWarps * 6 * S);       // m_s
    int* roff = rlo + a.m_s;                                       // m_s + 1
    __shared__ RowC s_rc[S];
    __shared__ unsigned s_row;
    __shared__ double s_d[S][3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_ext = a.n_s * a.n_4, m_int = a.m_s * a.m_4;
    int top = 1;
    while (top < a.m_s) top <<= 1;
    unsigned act = (1u << S) - 1u;  // solves still iterating (uniform over the grid)
    for (int it = a.it_begin; it < a.it_end && act; ++it) {
        const int cur = it & 1;
        const double2* Xin = b.Xh[cur];
        double2* Xout = b.Xh[cur ^ 1];
        if (blockIdx.x == 0 && tid == 0) {  // the next iteration's slots (unused until after this one's barriers)
            a.ctr[cur ^ 1] = 0u;
            for (int s = 0; s < S; ++s) {
                b.err[(cur ^ 1) * S + s] = ~0ull;
                b.nonfinite[(cur ^ 1) * S + s] = 0;
            }
        }
        // phase I: every iterating solve's node table (its state, its mu)
        for (int s = 0; s < S; ++s) {
            if (!(act >> s & 1u)) continue;
            MuArgs as = a;
            as.mu = b.mu[s];
            as.coeff = b.coeff[s];
            as.NB = b.NB + (size_t)s * 4 * m_int;
            build_nodes(as, Xin + (size_t)s * 3 * n_ext, b.nonfinite + cur * S + s);
        }
        grid.sync();
        double dmax[3] = {0.0, 0.0, 0.0};  // thread s < S: solve s's deltas over this CTA's rows
        for (;;) {
            if (tid == 0) s_row = atomicAdd(a.ctr + cur, 1u);
            __syncthreads();
            const unsigned r = s_row;
            __syncthreads();
            if (r >= (unsigned)a.n_rows) break;
            const int i = a.row_start + (int)r * a.row_stride;
            if (tid < S) {  // every solve (a stopped one is contracted too, its sums unused: no branch in the pair loop)
                MuArgs as = a;
                as.mu = b.mu[tid];
                as.coeff = b.coeff[tid];
                s_rc[tid] = row_consts(as, Xin + (size_t)tid * 3 * n_ext, n_ext, i);
            }
            for (int js = tid; js < a.m_s; js += kThreads) rlo[js] = __ldg(a.mo_rlo + (size_t)r * a.m_s + js);
            for (int js = tid; js <= a.m_s; js += kThreads) roff[js] = __ldg(a.mo_roff + (size_t)r * (a.m_s + 1) + js);
            __syncthreads();
            const int total = roff[a.m_s];
            const long long mbase = __ldg(a.mo_base + r);
            double acc[smacc ? 1 : S][6];
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    if (smacc) sacc[(s * 6 + c) * kThreads + tid] = 0.0;
                    else acc[smacc ? 0 : s][c] = 0.0;
                }
            constexpr bool kBatchPfNB = batch_pfnb<S>();
            int jsn = 0, j4n = 0;  // this chunk's node (computed one chunk ahead when prefetching node values)
            if (kBatchPfNB && total > 0) {
                const int f = min(tid, total - 1);
                jsn = node_of(roff, a.m_s, top, f);
                j4n = rlo[jsn] + (f - roff[jsn]);
            }
            for (int f0 = 0; f0 < total; f0 += kThreads) {
                const int f = min(f0 + tid, total - 1);
                int js, j4;
                if (kBatchPfNB) {
                    js = jsn;
                    j4 = j4n;
                } else {
                    js = node_of(roff, a.m_s, top, f);
                    j4 = rlo[js] + (f - roff[js]);
                }
                DCHECK(total == 0 || (js >= 0 && js < a.m_s && j4 >= 0 && j4 < a.m_4), 24);
                double mom[5];
                for (int q = 0; q < 5; ++q) mom[q] = __ldcs(a.mo_mom + q * a.mo_stride + mbase + f);
                if (kBatchPf && f0 + kThreads < total) {  // the next chunk's moments toward the SM (no registers held)
                    const int fn = min(f0 + kThreads + tid, total - 1);
                    for (int q = 0; q < 5; ++q) {
                        const double* pa = a.mo_mom + q * a.mo_stride + mbase + fn;
                        if (kBatchPf == 1) asm volatile("prefetch.global.L1 [%0];" ::"l"(pa));
                        else asm volatile("prefetch.global.L2 [%0];" ::"l"(pa));
                    }
                    if (kBatchPfNB) {  // and its node values, every solve, into L1
                        jsn = node_of(roff, a.m_s, top, fn);
                        j4n = rlo[jsn] + (fn - roff[jsn]);
                        for (int s = 0; s < S; ++s)
                            asm volatile("prefetch.global.L1 [%0];" ::"l"(b.NB + (size_t)s * 4 * m_int +
                                                                          4 * (size_t)(jsn * a.m_4 + j4n)));
                    }
                }
                __syncwarp();
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const double2* nb = b.NB + (size_t)s * 4 * m_int + 4 * (size_t)(js * a.m_4 + j4);
                    const double2 vn[4] = {nb[0], nb[1], nb[2], nb[3]};
                    double part[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                    pair_contract<V>(a, s_rc[s], js, j4, vn, mom, part);
                    if (f0 + tid < total)
                        for (int c = 0; c < 6; ++c) {
                            if (smacc) sacc[(s * 6 + c) * kThreads + tid] += part[c];
                            else acc[smacc ? 0 : s][c] += part[c];
                        }
                }
            }
            // fixed-order block reduction per solve (mu_solve_kernel's)
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    double v = smacc ? sacc[(s * 6 + c) * kThreads + tid] : acc[smacc ? 0 : s][c];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    if (lane == 0) red[(warp * S + s) * 6 + c] = v;
                }
            __syncthreads();
            if (tid < S && (act >> tid & 1u)) {
                const int s = tid;
                const RowC& rc = s_rc[s];
                double sum[6];
                for (int c = 0; c < 6; ++c) {
                    double v = red[s * 6 + c];
                    for (int w = 1; w < kWarps; ++w) v += red[(w * S + s) * 6 + c];
                    sum[c] = v;
                }
                const double2 An = make_double2(b.z1[s] + sum[0] / rc.P2, sum[1] / rc.P2);
                const double2 Bn = make_double2(b.m0z1[s] + sum[2], sum[3]);
                const cplx cn = C(sum[4], sum[5]) * rcp(rc.p4t);
                const double2 Cn = make_double2(b.z1[s] + cn.x, cn.y);
                const bool fin = isfinite(An.x) && isfinite(An.y) && isfinite(Bn.x) && isfinite(Bn.y) &&
                                 isfinite(Cn.x) && isfinite(Cn.y);
                const int nf = b.nonfinite[cur * S + s];
                if (!fin || nf) atomicMin(b.err + cur * S + s, (unsigned long long)(nf ? a.row_start : i));
                double2* Xo = Xout + (size_t)s * 3 * n_ext;
                Xo[i] = An;
                Xo[n_ext + i] = Bn;
                Xo[2 * n_ext + i] = Cn;
                // the single solve's stop-rule deltas (mu_solve_kernel)
                dmax[0] = fmax(dmax[0], hyp(An.x - rc.Ap.x, An.y - rc.Ap.y));
                dmax[1] = fmax(dmax[1], hyp(Bn.x - rc.Bp.x, Bn.y - rc.Bp.y));
                dmax[2] = fmax(dmax[2], hyp(Cn.x - rc.Cp.x, Cn.y - rc.Cp.y));
            }
            __syncthreads();
        }
        if (!b.stop) break;
        if (tid < S)
            for (int c = 0; c < 3; ++c) b.bmax[((size_t)blockIdx.x * S + tid) * 3 + c] = dmax[c];
        grid.sync();
        // ---- stop test per solve (every CTA, identical decisions) ----
        if (warp < S) {
            double d[3] = {0.0, 0.0, 0.0};
            for (int q = lane; q < (int)gridDim.x; q += 32)
                for (int c = 0; c < 3; ++c) d[c] = fmax(d[c], __ldcg(b.bmax + ((size_t)q * S + warp) * 3 + c));
            for (int c = 0; c < 3; ++c) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) d[c] = fmax(d[c], __shfl_xor_sync(0xffffffffu, d[c], o));
                if (lane == 0) s_d[warp][c] = d[c];
            }
        }
        __syncthreads();
        bool failed = false;
        for (int s = 0; s < S; ++s)
            if ((act >> s & 1u) && __ldcg(b.err + cur * S + s) != ~0ull) failed = true;
        const unsigned act_in = act;
        for (int s = 0; s < S; ++s) {
            if (!(act_in >> s & 1u)) continue;
            const unsigned long long er = __ldcg(b.err + cur * S + s);
            const double d0 = s_d[s][0], d1 = s_d[s][1], d2 = s_d[s][2];
            if (er != ~0ull) {
                if (blockIdx.x == 0 && tid == 0) {
                    b.status[4 * s + 0] = it + 1;
                    b.status[4 * s + 2] = it + 1;
                    b.status[4 * s + 3] = (long long)er;
                }
                continue;
            }
            if (blockIdx.x == 0 && tid == 0 && b.hist) {
                double* h = b.hist + ((size_t)s * b.hist_stride + (it + 1)) * 4;
                h[0] = double(it + 1);
                h[1] = d0;
                h[2] = d1;
                h[3] = d2;
            }
            const bool conv = d0 < b.xi[s] && d1 < b.xi[s] && d2 < b.xi[s];
            if (conv || it + 1 >= b.cap[s]) {
                act &= ~(1u << s);
                if (blockIdx.x == 0 && tid == 0) {
                    b.status[4 * s + 0] = it + 1;
                    b.status[4 * s + 1] = conv ? 1 : 0;
                }
            } else if (blockIdx.x == 0 && tid == 0) {
                b.status[4 * s + 0] = it + 1;
            }
        }
        if (failed) break;
        __syncthreads();  // s_d is rewritten by the next stop test only after two grid barriers
    }
}

// Failure location: first non-finite point (j, k) in row-major order of the
// failing row, evaluated with the same pair form.  One thread per node.
template <int V>
__global__ void __launch_bounds__(kThreads) mu_locate_kernel(MuArgs a, int i, int in_buf, unsigned long long* first) {
    __shared__ double etbl[1 << dse::kExpTableBits];
    for (int t = threadIdx.x; t < (1 << dse::kExpTableBits); t += blockDim.x) etbl[t] = __ldg(a.exp_tbl + t);
    __syncthreads();
    const unsigned tbl = dse::smem_addr(etbl);
    const int n_ext = a.n_s * a.n_4, m_int = a.m_s * a.m_4;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m_int) return;
    const double2* Xin = a.X + (size_t)in_buf * 3 * n_ext;
    const int is = i / a.n_4, i4 = i - is * a.n_4;
    RowC rc;
    rc.P = a.P[is];
    rc.P2 = a.P2[is];
    rc.p4r = a.p4[i4];
    rc.p4t = C(rc.p4r, a.mu);
    rc.Ap = C(Xin[i].x, Xin[i].y);
    rc.Bp = C(Xin[n_ext + i].x, Xin[n_ext + i].y);
    rc.Cp = C(Xin[2 * n_ext + i].x, Xin[2 * n_ext + i].y);
    rc.hAp = 0.5 * rc.Ap;
    rc.hCp = 0.5 * rc.Cp;
    rc.mu = a.mu;
    rc.coeff = a.coeff;
    // per point: run the pair form with a single-angle weight table
    double2 zw1[1];
    MuArgs b = a;
    b.K = 1;
    for (int k = 0; k < a.K; ++k) {
        zw1[0] = make_double2(a.z[k], a.wz[k]);
        double acc[6] = {0, 0, 0, 0, 0, 0};
        pair_contrib<V>(b, rc, j / a.m_4, j % a.m_4, zw1, tbl, acc);
        bool bad = false;
        for (int c = 0; c < 6; ++c) bad |= !isfinite(acc[c]);
        if (bad) {
            atomicMin(first, (unsigned long long)j * (unsigned long long)a.K + (unsigned long long)k);
            return;
        }
    }
}

__global__ void mu_reset_kernel(unsigned* ctr, unsigned long long* err, long long* status, int* nonfinite) {
    const int t = threadIdx.x;
    if (t < 2) {
        ctr[t] = 0u;
        err[t] = ~0ull;
        nonfinite[t] = 0;
    }
    if (t < 4) status[t] = 0;
}


// ---- Anderson acceleration on the device (finite_mu.solve_mu_anderson and
// solve_mu_batch_anderson).  S solves of N = 3 n_ext complex unknowns each;
// the last `depth` residual/iterate differences live in ring slots
// dF[s][slot][N], dX[s][slot][N].  Every reduction is one CTA per output in a
// fixed order, and every solve is processed by the same code, so a solve
// batched with others computes bitwise what it computes alone.
constexpr int kAaMaxDepth = 16;
constexpr int kAaMaxS = 4;
struct AaCols {
    int n;                      // active columns
    int col[kAaMaxDepth];       // ring slots, oldest first
    double2 gamma[kAaMaxS][kAaMaxDepth];
};

// f = gx - x; max |f| per (solve, function) (exact max, order-free);
// with slot >= 0: dF[slot] = f - fprev, dX[slot] = x - xprev; then fprev = f,
// xprev = x.
__global__ void aa_residual_kernel(int S, long long n_ext, const double2* __restrict__ x,
                                   const double2* __restrict__ gx, double2* __restrict__ f, double2* fprev,
                                   double2* xprev, double2* __restrict__ dF, double2* __restrict__ dX, int depth,
                                   int slot, unsigned long long* dmax_bits) {
    const long long N = 3 * n_ext, total = (long long)S * N;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long s = e / N, i = e - s * N;
        const double2 xv = x[e], gv = gx[e];
        const double2 fv = make_double2(gv.x - xv.x, gv.y - xv.y);
        f[e] = fv;
        const double m = hypot(fv.x, fv.y);
        atomicMax(dmax_bits + 3 * s + i / n_ext, (unsigned long long)__double_as_longlong(m));
        if (slot >= 0) {
            const double2 fp = fprev[e], xp = xprev[e];
            const size_t o = ((size_t)s * depth + slot) * N + i;
            dF[o] = make_double2(fv.x - fp.x, fv.y - fp.y);
            dX[o] = make_double2(xv.x - xp.x, xv.y - xp.y);
        }
        fprev[e] = fv;
        xprev[e] = xv;
    }
}

// out[(s * 2 + w) * n + c] = sum_i conj(dF[s][col_c][i]) * v[i] with
// v = dF[s][slot] (w = 0, the new Gram column) or f[s] (w = 1, the
// right-hand side); one CTA per (s, w, c), 256 threads, fixed order.
__global__ void __launch_bounds__(256) aa_dots_kernel(long long n_ext, const double2* __restrict__ f,
                                                      const double2* __restrict__ dF, int depth, int slot, AaCols cols,
                                                      double2* __restrict__ out) {
    __shared__ double2 red[256];
    const long long N = 3 * n_ext;
    const int c = blockIdx.x, w = blockIdx.y, s = blockIdx.z;
    if (w == 0 && slot < 0) return;
    const double2* a = dF + ((size_t)s * depth + cols.col[c]) * N;
    const double2* v = w == 0 ? dF + ((size_t)s * depth + slot) * N : f + (size_t)s * N;
    double re = 0.0, im = 0.0;
    for (long long i = threadIdx.x; i < N; i += 256) {
        const double2 p = a[i], q = v[i];
        re = fma(p.x, q.x, fma(p.y, q.y, re));   // conj(p) q
        im = fma(p.x, q.y, fma(-p.y, q.x, im));
    }
    red[threadIdx.x] = make_double2(re, im);
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (threadIdx.x < h) {
            red[threadIdx.x].x += red[threadIdx.x + h].x;
            red[threadIdx.x].y += red[threadIdx.x + h].y;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[((size_t)s * 2 + w) * cols.n + c] = red[0];
}

// x <- x + beta f - sum_c gamma_c (dX[col_c] + beta dF[col_c]), the columns in
// ring order (oldest first).
__global__ void aa_update_kernel(int S, long long n_ext, double2* __restrict__ x, const double2* __restrict__ f,
                                 const double2* __restrict__ dF, const double2* __restrict__ dX, int depth,
                                 double beta, AaCols cols) {
    const long long N = 3 * n_ext, total = (long long)S * N;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long s = e / N, i = e - s * N;
        double ax = 0.0, ay = 0.0;
        for (int c = 0; c < cols.n; ++c) {
            const size_t o = ((size_t)s * depth + cols.col[c]) * N + i;
            const double2 dx = dX[o], df = dF[o], g = cols.gamma[s][c];
            const double tx = fma(beta, df.x, dx.x), ty = fma(beta, df.y, dx.y);
            ax = fma(g.x, tx, fma(-g.y, ty, ax));
            ay = fma(g.x, ty, fma(g.y, tx, ay));
        }
        const double2 xv = x[e], fv = f[e];
        x[e] = make_double2(fma(beta, fv.x, xv.x) - ax, fma(beta, fv.y, xv.y) - ay);
    }
}

}  // namespace mu

struct dse_mu_sweeper {
    int device = 0;
    cudaStream_t stream = nullptr;
    int n_s = 0, n_4 = 0, m_s = 0, m_4 = 0, K = 0;
    int row_start = 0, row_stride = 1, n_rows = 0;
    dse_mu_params prm{};
    double *d_P = nullptr, *d_P2 = nullptr, *d_p4 = nullptr, *d_Qs = nullptr, *d_Q2 = nullptr, *d_q4 = nullptr;
    double *d_ms = nullptr, *d_m4 = nullptr, *d_z = nullptr, *d_wz = nullptr, *d_etbl = nullptr;
    int zsym = 0;  // angular nodes/weights exactly mirror-symmetric
    int *d_brk_s = nullptr, *d_brk_4 = nullptr;
    double2* d_X = nullptr;
    double2* d_NB = nullptr;
    double* d_bmax = nullptr;
    unsigned* d_ctr = nullptr;
    unsigned long long* d_err = nullptr;
    long long* d_status = nullptr;
    long long* d_eval = nullptr;
    int* d_nonfinite = nullptr;
    double* d_hist = nullptr;
    size_t hist_cap = 0;
    int blocks = 0;
    size_t smem = 0, smem_mom = 0;
    long long it_next = 0;
    long long evaluated_pairs = -1;
    // moments mode tables (built on first use; geometry only, shared by every mu)
    int* d_mo_rlo = nullptr;
    int* d_mo_roff = nullptr;
    long long* d_mo_base = nullptr;
    double* d_mo_mom = nullptr;
    long long mo_total = -1;
    bool mo_mode = false;  // the current call runs the moments kernel
    double win_omega = -1.0;  // omega the windows were built for
    double2* d_bNB = nullptr;  // batched sweeps: [S][m_int][4] node tables
    unsigned long long* d_berr = nullptr;
    int* d_bnf = nullptr;
    int bblocks[2] = {0, 0};   // cooperative grid of the batch kernels (S = 2, 4)
    long long* d_bstatus = nullptr;  // [S][4] batched solve status
    double* d_bbmax = nullptr;       // [blocks][S][3] batched per-CTA deltas
    int bbmax_blocks = 0;
    long long win_pairs = 0;
};

namespace {

int mu_check_params(const dse_mu_params* p, dse_err* err) {
    if (!(p->omega > 0.0) || !(p->coeff >= 0.0) || !(p->xi > 0.0) || !(p->relaxation > 0.0 && p->relaxation <= 1.0) ||
        p->max_iterations < 1 || !(p->mu >= 0.0) || !std::isfinite(p->mu) || p->vertex < 0 || p->vertex > 2 ||
        p->mode < 0 || p->mode > 1)
        return fail(err, DSE_EPARAM, "finite-mu parameters out of range");
    return DSE_OK;
}

mu::MuArgs mu_make_args(dse_mu_sweeper* s, const dse_mu_params& p, int it_begin, int it_end, bool hist, bool sweep_only,
                        bool count) {
    mu::MuArgs a{};
    a.P = s->d_P; a.P2 = s->d_P2; a.p4 = s->d_p4; a.Qs = s->d_Qs; a.Q2 = s->d_Q2; a.q4 = s->d_q4;
    a.meas_s = s->d_ms; a.meas_4 = s->d_m4; a.z = s->d_z; a.wz = s->d_wz; a.exp_tbl = s->d_etbl;
    a.zsym = s->zsym;
    a.brk_s = s->d_brk_s; a.brk_4 = s->d_brk_4;
    a.n_s = s->n_s; a.n_4 = s->n_4; a.m_s = s->m_s; a.m_4 = s->m_4; a.K = s->K;
    a.row_start = s->row_start; a.row_stride = s->row_stride; a.n_rows = s->n_rows;
    a.coeff = p.coeff;
    a.w2 = p.omega * p.omega;
    a.exp_c1 = -double(1 << dse::kExpTableBits) * 1.4426950408889634 / a.w2;
    a.skip_k2 = 708.0 * a.w2;  // exp(-x) < 2^-1021 beyond: the point is an exact zero of the sum (F8)
    a.mu = p.mu; a.z1 = p.z1; a.m0z1 = p.m0 * p.z1; a.xi = p.xi; a.relax = p.relaxation;
    a.X = s->d_X; a.NB = s->d_NB; a.bmax = s->d_bmax; a.ctr = s->d_ctr; a.err = s->d_err; a.status = s->d_status;
    a.nonfinite = s->d_nonfinite;
    a.hist = hist ? s->d_hist : nullptr;
    a.evaluated = count ? s->d_eval : nullptr;
    a.it_begin = it_begin; a.it_end = it_end; a.sweep_only = sweep_only ? 1 : 0;
    a.vertex = (int)p.vertex;
    a.dq_eps2 = getenv("DSE_MU_DQ_EPS2") ? atof(getenv("DSE_MU_DQ_EPS2")) : 0.0;
    a.mo_rlo = s->d_mo_rlo; a.mo_roff = s->d_mo_roff; a.mo_base = s->d_mo_base; a.mo_mom = s->d_mo_mom;
    a.mo_stride = s->mo_total > 0 ? s->mo_total : 0;
    return a;
}

const void* mu_kernel_ptr(int v, bool mom = false) {
    if (mom) {
        if (v == DSE_MU_VERTEX_BC1) return (const void*)mu::mu_solve_kernel<DSE_MU_VERTEX_BC1, true>;
        if (v == DSE_MU_VERTEX_BCB) return (const void*)mu::mu_solve_kernel<DSE_MU_VERTEX_BCB, true>;
        return (const void*)mu::mu_solve_kernel<DSE_MU_VERTEX_BC, true>;
    }
    if (v == DSE_MU_VERTEX_BC1) return (const void*)mu::mu_solve_kernel<DSE_MU_VERTEX_BC1, false>;
    if (v == DSE_MU_VERTEX_BCB) return (const void*)mu::mu_solve_kernel<DSE_MU_VERTEX_BCB, false>;
    return (const void*)mu::mu_solve_kernel<DSE_MU_VERTEX_BC, false>;
}

// Moments mode: the windows and the five angular moments of every evaluated
// pair of the owned rows, once per sweeper (they depend on the grid and
// omega only, so every mu of a config-4 sweep reuses them).
// The exact-zero windows of every owned row (geometry + omega only) and the
// rows' pair offsets into the moment table; used by both modes.
int mu_build_windows(dse_mu_sweeper* s, const dse_mu_params& p, dse_err* err) {
    if (s->win_omega == p.omega && s->d_mo_rlo) return DSE_OK;
    const size_t R = (size_t)s->n_rows, ms = (size_t)s->m_s;
    if (s->d_mo_rlo) {  // a different omega: new windows, and the moments go stale
        for (void* q : {(void*)s->d_mo_rlo, (void*)s->d_mo_roff, (void*)s->d_mo_base, (void*)s->d_mo_mom}) cudaFree(q);
        s->d_mo_rlo = nullptr; s->d_mo_roff = nullptr; s->d_mo_base = nullptr; s->d_mo_mom = nullptr;
        s->mo_total = -1;
    }
    CUDA_TRY(cudaMalloc(&s->d_mo_rlo, R * ms * sizeof(int)));
    CUDA_TRY(cudaMalloc(&s->d_mo_roff, R * (ms + 1) * sizeof(int)));
    CUDA_TRY(cudaMalloc(&s->d_mo_base, R * sizeof(long long)));
    long long* d_tot = nullptr;
    CUDA_TRY(cudaMalloc(&d_tot, R * sizeof(long long)));
    mu::MuArgs a = mu_make_args(s, p, 0, 0, false, true, false);
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device));
    const size_t sm1 = (size_t)s->m_4 * sizeof(double) + (2 * ms + 2) * sizeof(int);
    CUDA_TRY(cudaFuncSetAttribute((const void*)mu::mu_windows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sm1));
    mu::mu_windows_kernel<<<std::max(1, std::min((int)R, 4 * sms)), mu::kThreads, sm1, s->stream>>>(
        a, s->d_mo_rlo, s->d_mo_roff, d_tot);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    std::vector<long long> tot(R), base(R);
    CUDA_TRY(cudaMemcpyAsync(tot.data(), d_tot, R * sizeof(long long), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    cudaFree(d_tot);
    long long sum = 0;
    for (size_t r = 0; r < R; ++r) {
        base[r] = sum;
        sum += tot[r];
    }
    CUDA_TRY(cudaMemcpyAsync(s->d_mo_base, base.data(), R * sizeof(long long), cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    s->win_pairs = sum;
    s->win_omega = p.omega;
    return DSE_OK;
}

int mu_build_moments(dse_mu_sweeper* s, const dse_mu_params& p, dse_err* err) {
    int rc = mu_build_windows(s, p, err);
    if (rc) return rc;
    if (s->mo_total >= 0) return DSE_OK;
    const size_t R = (size_t)s->n_rows, ms = (size_t)s->m_s;
    (void)ms;
    const long long sum = s->win_pairs;
    mu::MuArgs a = mu_make_args(s, p, 0, 0, false, true, false);
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device));
    size_t free_b = 0, total_b = 0;
    CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
    if ((size_t)std::max(sum, 1ll) * 5 * sizeof(double) > free_b)
        return fail(err, DSE_EENV, "moment table of %lld pairs does not fit in device memory", sum);
    CUDA_TRY(cudaMalloc(&s->d_mo_mom, (size_t)std::max(sum, 1ll) * 5 * sizeof(double)));
    s->mo_total = std::max(sum, 1ll);
    a = mu_make_args(s, p, 0, 0, false, true, false);
    const size_t sm2 = ((1 << dse::kExpTableBits) + 2 * (size_t)s->K) * sizeof(double) + (ms + 1) * sizeof(int);
    CUDA_TRY(cudaFuncSetAttribute((const void*)mu::mu_moments_build_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)mu::mu_moments_build_kernel,
                                                          mu::kThreads, sm2));
    mu::mu_moments_build_kernel<<<std::max(1, std::min((int)R, std::max(per_sm, 1) * sms)), mu::kThreads, sm2,
                                  s->stream>>>(a);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    return DSE_OK;
}

// select the kernel family of this call; build the moment table on first use
int mu_prepare(dse_mu_sweeper* s, const dse_mu_params& p, dse_err* err) {
    s->mo_mode = p.mode == DSE_MU_MODE_MOMENTS;
    return s->mo_mode ? mu_build_moments(s, p, err) : mu_build_windows(s, p, err);
}

int mu_launch(dse_mu_sweeper* s, const mu::MuArgs& a, bool reset, dse_err* err) {
    if (s->mo_mode && !a.mo_mom) return fail(err, DSE_EENV, "moments mode without a moment table");
    if (reset) {
        mu::mu_reset_kernel<<<1, 32, 0, s->stream>>>(s->d_ctr, s->d_err, s->d_status, s->d_nonfinite);
        CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1);
    }
    mu::MuArgs b = a;
    void* args[] = {&b};
    const bool mom = a.mo_mom != nullptr && s->mo_mode;
    CUDA_TRY(cudaLaunchCooperativeKernel(mu_kernel_ptr(a.vertex, mom), dim3(s->blocks), dim3(mu::kThreads), args,
                                         mom ? s->smem_mom : s->smem, s->stream));
    g_launches.fetch_add(1);
    return DSE_OK;
}

int mu_failure(dse_mu_sweeper* s, const dse_mu_params& p, long long it_fail, long long row, dse_err* err) {
    // locate the first non-finite point of the failing row on the input state of that iteration
    unsigned long long* d_first = nullptr;
    CUDA_TRY(cudaMalloc(&d_first, sizeof(unsigned long long)));
    CUDA_TRY(cudaMemsetAsync(d_first, 0xff, sizeof(unsigned long long), s->stream));
    mu::MuArgs a = mu_make_args(s, p, 0, 0, false, true, false);
    const int m_int = s->m_s * s->m_4;
    // the node table NB still holds the failing iteration's input (the loop stops right after it)
    const int in_buf = (int)((it_fail - 1) & 1);
    auto loc = p.vertex == DSE_MU_VERTEX_BC1 ? mu::mu_locate_kernel<DSE_MU_VERTEX_BC1>
             : p.vertex == DSE_MU_VERTEX_BCB ? mu::mu_locate_kernel<DSE_MU_VERTEX_BCB>
                                             : mu::mu_locate_kernel<DSE_MU_VERTEX_BC>;
    loc<<<(m_int + mu::kThreads - 1) / mu::kThreads, mu::kThreads, 0, s->stream>>>(a, (int)row, in_buf,
                                                                                                  d_first);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    unsigned long long first = ~0ull;
    CUDA_TRY(cudaMemcpyAsync(&first, d_first, sizeof(first), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    cudaFree(d_first);
    long long j = -1, k = -1;
    if (first != ~0ull) {
        j = (long long)(first / (unsigned long long)s->K);
        k = (long long)(first % (unsigned long long)s->K);
    }
    fail(err, DSE_ENUMERIC, "non-finite integrand in finite-mu sweep at row=%lld, radial=%lld, angular=%lld", row, j, k);
    if (err) {
        err->iteration = it_fail;
        err->row = row;
        err->radial = j;
        err->angular = k;
    }
    return DSE_ENUMERIC;
}

}  // namespace

extern "C" {

int dse_mu_sweeper_create(const dse_mu_grid* g, const dse_mu_params* p, int device, int64_t row_start,
                          int64_t row_stride, dse_mu_sweeper** out, dse_err* err) {
    ok(err);
    if (!g || !p || !out) return fail(err, DSE_EPARAM, "null argument");
    *out = nullptr;
    if (g->n_s < 2 || g->n_4 < 2 || g->m_s < 2 || g->m_4 < 2 || g->m_ang < 1)
        return fail(err, DSE_EPARAM, "finite-mu grid sizes out of range");
    if (g->n_s * g->n_4 > (1LL << 30) || g->m_s * g->m_4 > (1LL << 30) || g->m_ang > 4096)
        return fail(err, DSE_EPARAM, "finite-mu grid too large");
    if (!g->p_ext || !g->ps2_ext || !g->p4_ext || !g->q_int || !g->qs2_int || !g->q4_int || !g->meas_s ||
        !g->meas_4 || !g->z_nodes || !g->z_weights || !g->brk_s || !g->brk_4)
        return fail(err, DSE_EPARAM, "null grid array");
    int rc = mu_check_params(p, err);
    if (rc) return rc;
    const int64_t n_ext = g->n_s * g->n_4;
    if (row_stride < 1 || row_start < 0 || (row_start >= n_ext && n_ext > 0))
        return fail(err, DSE_EPARAM, "bad row partition start=%lld stride=%lld", (long long)row_start,
                    (long long)row_stride);
    for (int64_t j = 0; j < g->m_s; ++j)
        if (g->brk_s[j] < -1 || g->brk_s[j] > g->n_s - 1) return fail(err, DSE_EPARAM, "brk_s out of range");
    for (int64_t j = 0; j < g->m_4; ++j)
        if (g->brk_4[j] < -1 || g->brk_4[j] > g->n_4 - 1) return fail(err, DSE_EPARAM, "brk_4 out of range");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(err, DSE_EENV, "CUDA device %d not present", device);
    CUDA_TRY(cudaSetDevice(device));
    auto* s = new dse_mu_sweeper();
    s->device = device;
    s->n_s = (int)g->n_s; s->n_4 = (int)g->n_4; s->m_s = (int)g->m_s; s->m_4 = (int)g->m_4; s->K = (int)g->m_ang;
    s->row_start = (int)row_start; s->row_stride = (int)row_stride;
    s->n_rows = (int)((n_ext - row_start + row_stride - 1) / row_stride);
    s->prm = *p;
    auto bail = [&](int code) {
        dse_mu_sweeper_destroy(s);
        return code;
    };
#define MU_TRY(expr)                                                                                       \
    do {                                                                                                   \
        cudaError_t _e = (expr);                                                                           \
        if (_e != cudaSuccess)                                                                             \
            return bail(fail(err, DSE_EENV, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__)); \
    } while (0)
    MU_TRY(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    cudaStream_t st = s->stream;
    std::vector<int> bs(g->brk_s, g->brk_s + g->m_s), b4(g->brk_4, g->brk_4 + g->m_4);
    MU_TRY(upload(&s->d_P, g->p_ext, g->n_s, st));
    MU_TRY(upload(&s->d_P2, g->ps2_ext, g->n_s, st));
    MU_TRY(upload(&s->d_p4, g->p4_ext, g->n_4, st));
    MU_TRY(upload(&s->d_Qs, g->q_int, g->m_s, st));
    MU_TRY(upload(&s->d_Q2, g->qs2_int, g->m_s, st));
    MU_TRY(upload(&s->d_q4, g->q4_int, g->m_4, st));
    MU_TRY(upload(&s->d_ms, g->meas_s, g->m_s, st));
    MU_TRY(upload(&s->d_m4, g->meas_4, g->m_4, st));
    {
        bool sym = !(getenv("DSE_MU_MIRROR") && atoi(getenv("DSE_MU_MIRROR")) == 0);
        for (int64_t k = 0; k < g->m_ang && sym; ++k) {
            const int64_t m = g->m_ang - 1 - k;
            sym = g->z_nodes[m] == -g->z_nodes[k] && g->z_weights[m] == g->z_weights[k] &&
                  (k >= m || g->z_nodes[m] > 0.0);
        }
        s->zsym = sym ? 1 : 0;
    }
    MU_TRY(upload(&s->d_z, g->z_nodes, g->m_ang, st));
    MU_TRY(upload(&s->d_wz, g->z_weights, g->m_ang, st));
    MU_TRY(upload(&s->d_brk_s, bs.data(), bs.size(), st));
    MU_TRY(upload(&s->d_brk_4, b4.data(), b4.size(), st));
    std::vector<double> etbl(1 << dse::kExpTableBits);
    for (int i = 0; i < (1 << dse::kExpTableBits); ++i) etbl[i] = std::exp2(i / double(1 << dse::kExpTableBits));
    MU_TRY(upload(&s->d_etbl, etbl.data(), etbl.size(), st));
    MU_TRY(cudaMalloc(&s->d_X, sizeof(double2) * 2 * 3 * (size_t)n_ext));
    MU_TRY(cudaMemsetAsync(s->d_X, 0, sizeof(double2) * 2 * 3 * (size_t)n_ext, st));
    MU_TRY(cudaMalloc(&s->d_NB, sizeof(double2) * 4 * (size_t)(g->m_s * g->m_4)));
    MU_TRY(cudaMalloc(&s->d_ctr, 2 * sizeof(unsigned)));
    MU_TRY(cudaMalloc(&s->d_err, 2 * sizeof(unsigned long long)));
    MU_TRY(cudaMalloc(&s->d_status, 4 * sizeof(long long)));
    MU_TRY(cudaMalloc(&s->d_nonfinite, 2 * sizeof(int)));
    MU_TRY(cudaMalloc(&s->d_eval, sizeof(long long)));
    s->smem = (size_t)((1 << dse::kExpTableBits) + 2 * s->K + mu::kWarps * 6 + s->m_4) * sizeof(double) +
              (size_t)(2 * s->m_s + 2) * sizeof(int);
    s->smem_mom = mu::kMomStage ? ((s->smem + 15) & ~size_t(15)) + 2 * sizeof(double) * mu::kThreads * mu::kStageDoubles
                                : s->smem;
    int per_sm = 1 << 30, sms = 0;
    for (int v : {DSE_MU_VERTEX_BC, DSE_MU_VERTEX_BC1, DSE_MU_VERTEX_BCB})
        for (bool mom : {false, true}) {
            const size_t sz = mom ? s->smem_mom : s->smem;
            MU_TRY(cudaFuncSetAttribute(mu_kernel_ptr(v, mom), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sz));
            int n = 0;
            MU_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, mu_kernel_ptr(v, mom), mu::kThreads, sz));
            per_sm = std::min(per_sm, n);
        }
    MU_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    if (per_sm < 1) return bail(fail(err, DSE_EENV, "finite-mu kernel does not fit on an SM"));
    s->blocks = per_sm * sms;
    if (const char* e = getenv("DSE_MU_BLOCKS")) s->blocks = std::max(1, std::min(s->blocks, atoi(e)));
    MU_TRY(cudaMalloc(&s->d_bmax, 3 * sizeof(double) * (size_t)s->blocks));
    MU_TRY(cudaStreamSynchronize(st));
#undef MU_TRY
    *out = s;
    return DSE_OK;
}

int dse_mu_sweeper_destroy(dse_mu_sweeper* s) {
    if (!s) return DSE_OK;
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    for (void* p : {(void*)s->d_P, (void*)s->d_P2, (void*)s->d_p4, (void*)s->d_Qs, (void*)s->d_Q2, (void*)s->d_q4,
                    (void*)s->d_ms, (void*)s->d_m4, (void*)s->d_z, (void*)s->d_wz, (void*)s->d_etbl,
                    (void*)s->d_brk_s, (void*)s->d_brk_4, (void*)s->d_X, (void*)s->d_NB, (void*)s->d_bmax,
                    (void*)s->d_ctr, (void*)s->d_err, (void*)s->d_status, (void*)s->d_eval, (void*)s->d_hist, (void*)s->d_nonfinite,
                    (void*)s->d_mo_rlo, (void*)s->d_mo_roff, (void*)s->d_mo_base, (void*)s->d_mo_mom,
                    (void*)s->d_bNB, (void*)s->d_berr, (void*)s->d_bnf, (void*)s->d_bstatus,
                    (void*)s->d_bbmax})
        if (p) cudaFree(p);
    if (s->stream) cudaStreamDestroy(s->stream);
    delete s;
    return DSE_OK;
}

// Upload a complex state (host, interleaved re/im, n_ext each) into X[0].
static int mu_put_state(dse_mu_sweeper* s, const double* A, const double* B, const double* C_, dse_err* err) {
    const size_t n = (size_t)s->n_s * s->n_4;
    const double* src[3] = {A, B, C_};
    for (int f = 0; f < 3; ++f)
        CUDA_TRY(cudaMemcpyAsync(s->d_X + f * n, src[f], n * sizeof(double2), cudaMemcpyHostToDevice, s->stream));
    return DSE_OK;
}

int dse_mu_solve(dse_mu_sweeper* s, const dse_mu_params* params, double* A, double* B, double* C_,
                 int64_t* iterations, int* converged, double* history, dse_err* err) {
    ok(err);
    if (!s || !A || !B || !C_) return fail(err, DSE_EPARAM, "null argument");
    const dse_mu_params p = params ? *params : s->prm;
    int rc = mu_check_params(&p, err);
    if (rc) return rc;
    if (s->row_start != 0 || s->row_stride != 1)
        return fail(err, DSE_EPARAM, "dse_mu_solve needs a sweeper that owns every row");
    CUDA_TRY(cudaSetDevice(s->device));
    const size_t cap = (size_t)p.max_iterations;
    if (history && s->hist_cap < cap + 1) {
        if (s->d_hist) cudaFree(s->d_hist);
        s->d_hist = nullptr;
        CUDA_TRY(cudaMalloc(&s->d_hist, 4 * sizeof(double) * (cap + 1)));
        s->hist_cap = cap + 1;
    }
    rc = mu_put_state(s, A, B, C_, err);
    if (rc) return rc;
    rc = mu_prepare(s, p, err);
    if (rc) return rc;
    const bool count = s->evaluated_pairs < 0;
    if (count) CUDA_TRY(cudaMemsetAsync(s->d_eval, 0, sizeof(long long), s->stream));
    mu::MuArgs a = mu_make_args(s, p, 0, (int)cap, history != nullptr, false, count);
    rc = mu_launch(s, a, true, err);
    if (rc) return rc;
    long long st[4];
    CUDA_TRY(cudaMemcpyAsync(st, s->d_status, sizeof(st), cudaMemcpyDeviceToHost, s->stream));
    long long ev = 0;
    if (count) CUDA_TRY(cudaMemcpyAsync(&ev, s->d_eval, sizeof(ev), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (count) s->evaluated_pairs = ev;
    if (st[2] != 0) return mu_failure(s, p, st[2], st[3], err);
    const long long n = st[0];
    const size_t ne = (size_t)s->n_s * s->n_4;
    const double2* fin = s->d_X + (size_t)(n & 1) * 3 * ne;
    double* dst[3] = {A, B, C_};
    for (int f = 0; f < 3; ++f)
        CUDA_TRY(cudaMemcpyAsync(dst[f], fin + f * ne, ne * sizeof(double2), cudaMemcpyDeviceToHost, s->stream));
    if (history) {
        CUDA_TRY(cudaMemcpyAsync(history + 4, s->d_hist + 4, 4 * sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost,
                                 s->stream));
        history[0] = 0.0;
        history[1] = history[2] = history[3] = NAN;
    }
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (iterations) *iterations = n;
    if (converged) *converged = (int)st[1];
    return DSE_OK;
}

int dse_mu_sweep(dse_mu_sweeper* s, const dse_mu_params* params, const double* A, const double* B, const double* C_,
                 double* A_out, double* B_out, double* C_out, dse_err* err) {
    ok(err);
    if (!s || !A || !B || !C_ || !A_out || !B_out || !C_out) return fail(err, DSE_EPARAM, "null argument");
    dse_mu_params p = params ? *params : s->prm;
    int rc = mu_check_params(&p, err);
    if (rc) return rc;
    p.relaxation = 1.0;  // one Jacobi sweep (iterate_once, solver.py:201-212)
    CUDA_TRY(cudaSetDevice(s->device));
    rc = mu_put_state(s, A, B, C_, err);
    if (rc) return rc;
    const size_t ne = (size_t)s->n_s * s->n_4;
    // rows not owned keep their input value in the output buffer
    CUDA_TRY(cudaMemcpyAsync(s->d_X + 3 * ne, s->d_X, 3 * ne * sizeof(double2), cudaMemcpyDeviceToDevice, s->stream));
    rc = mu_prepare(s, p, err);
    if (rc) return rc;
    mu::MuArgs a = mu_make_args(s, p, 0, 1, false, true, false);
    rc = mu_launch(s, a, true, err);
    if (rc) return rc;
    long long st[4];
    CUDA_TRY(cudaMemcpyAsync(st, s->d_status, sizeof(st), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if (st[2] != 0) {
        rc = mu_failure(s, p, st[2], st[3], err);
        if (err) err->iteration = 0;
        return rc;
    }
    double* dst[3] = {A_out, B_out, C_out};
    for (int f = 0; f < 3; ++f)
        CUDA_TRY(cudaMemcpyAsync(dst[f], s->d_X + (3 + f) * ne, ne * sizeof(double2), cudaMemcpyDeviceToHost,
                                 s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    return DSE_OK;
}

int dse_mu_solve_load(dse_mu_sweeper* s, const double* dA, const double* dB, const double* dC, uintptr_t stream,
                      dse_err* err) {
    ok(err);
    if (!s || !dA || !dB || !dC) return fail(err, DSE_EPARAM, "null argument");
    CUDA_TRY(cudaSetDevice(s->device));
    cudaStream_t st = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    const size_t ne = (size_t)s->n_s * s->n_4;
    const double* src[3] = {dA, dB, dC};
    for (int f = 0; f < 3; ++f)
        CUDA_TRY(cudaMemcpyAsync(s->d_X + f * ne, src[f], ne * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    mu::mu_reset_kernel<<<1, 32, 0, st>>>(s->d_ctr, s->d_err, s->d_status, s->d_nonfinite);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    s->it_next = 0;
    return DSE_OK;
}

int dse_mu_solve_resume(dse_mu_sweeper* s, int64_t n_iterations, uintptr_t stream, dse_err* err) {
    ok(err);
    if (!s || n_iterations < 1) return fail(err, DSE_EPARAM, "bad argument");
    CUDA_TRY(cudaSetDevice(s->device));
    int rc0 = mu_prepare(s, s->prm, err);
    if (rc0) return rc0;
    cudaStream_t keep = s->stream;
    s->stream = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    mu::MuArgs a = mu_make_args(s, s->prm, (int)s->it_next, (int)(s->it_next + n_iterations), false, true, false);
    int rc = mu_launch(s, a, false, err);
    s->stream = keep;
    if (rc) return rc;
    s->it_next += n_iterations;
    return DSE_OK;
}

int dse_mu_interp(dse_mu_sweeper* s, const double* F, double* out, dse_err* err) {
    ok(err);
    if (!s || !F || !out) return fail(err, DSE_EPARAM, "null argument");
    CUDA_TRY(cudaSetDevice(s->device));
    const size_t ne = (size_t)s->n_s * s->n_4, m = (size_t)s->m_s * s->m_4;
    int rc = mu_put_state(s, F, F, F, err);
    if (rc) return rc;
    // one sweep-only launch with zero iterations does not build nodes; run the
    // node phase through a 1-iteration sweep on a copy and read NB[.][0]
    s->mo_mode = false;
    mu::MuArgs a = mu_make_args(s, s->prm, 0, 1, false, true, false);
    rc = mu_launch(s, a, true, err);
    if (rc) return rc;
    std::vector<double2> nb(4 * m);
    CUDA_TRY(cudaMemcpyAsync(nb.data(), s->d_NB, nb.size() * sizeof(double2), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    for (size_t j = 0; j < m; ++j) {
        out[2 * j] = nb[4 * j].x;
        out[2 * j + 1] = nb[4 * j].y;
    }
    (void)ne;
    return DSE_OK;
}

int dse_mu_sharded_sweep_pack(dse_mu_sweeper* s, const dse_mu_params* params, double* d_send, int64_t per,
                              uintptr_t stream, dse_err* err) {
    ok(err);
    if (!s || !d_send || per < s->n_rows) return fail(err, DSE_EPARAM, "bad argument");
    dse_mu_params p = params ? *params : s->prm;
    int rc = mu_check_params(&p, err);
    if (rc) return rc;
    p.relaxation = 1.0;  // the blend is applied at assembly
    CUDA_TRY(cudaSetDevice(s->device));
    rc = mu_prepare(s, p, err);
    if (rc) return rc;
    cudaStream_t keep = s->stream;
    s->stream = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    mu::MuArgs a = mu_make_args(s, p, 0, 1, false, true, false);
    rc = mu_launch(s, a, true, err);
    if (!rc) {
        const size_t ne = (size_t)s->n_s * s->n_4;
        mu::mu_pack_kernel<<<(int)std::max<int64_t>(1, (per + 255) / 256), 256, 0, s->stream>>>(
            s->d_X + 3 * ne, (int)ne, s->row_start, s->row_stride, (int)per, (double2*)d_send);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = fail(err, DSE_EENV, "mu_pack_kernel: %s", cudaGetErrorString(e));
        g_launches.fetch_add(1);
    }
    s->stream = keep;
    return rc;
}

int dse_mu_sharded_assemble(dse_mu_sweeper* s, const double* d_recv, int64_t world, int64_t per, double relax,
                            double* d_delta, uintptr_t stream, dse_err* err) {
    ok(err);
    const int64_t ne = s ? (int64_t)s->n_s * s->n_4 : 0;
    if (!s || !d_recv || !d_delta || world < 1 || per * world < ne) return fail(err, DSE_EPARAM, "bad argument");
    if (!(relax > 0.0 && relax <= 1.0)) return fail(err, DSE_EPARAM, "relaxation out of range");
    CUDA_TRY(cudaSetDevice(s->device));
    mu::mu_assemble_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(
        (const double2*)d_recv, (int)world, (int)per, (int)ne, relax, s->d_X, d_delta);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    return DSE_OK;
}

int dse_mu_sharded_failure(dse_mu_sweeper* s, uintptr_t stream, dse_err* err) {
    // after a sharded sweep on `stream`: report a numerical failure of this rank's rows
    ok(err);
    if (!s) return fail(err, DSE_EPARAM, "null argument");
    long long st[4];
    CUDA_TRY(cudaMemcpyAsync(st, s->d_status, sizeof(st), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    if (st[2] == 0) return DSE_OK;
    return mu_failure(s, s->prm, st[2], st[3], err);
}

int dse_mu_sweeper_state(dse_mu_sweeper* s, double** dX) {
    if (!s || !dX) return DSE_EPARAM;
    *dX = (double*)s->d_X;  // [3][n_ext] complex: A, B, C
    return DSE_OK;
}

}  // extern "C"

namespace {
const void* mu_batch_ptr(int vv, int64_t ss) {
    if (ss == 2) return vv == DSE_MU_VERTEX_BC1 ? (const void*)mu::mu_batch_kernel<DSE_MU_VERTEX_BC1, 2>
                      : vv == DSE_MU_VERTEX_BCB ? (const void*)mu::mu_batch_kernel<DSE_MU_VERTEX_BCB, 2>
                                                : (const void*)mu::mu_batch_kernel<DSE_MU_VERTEX_BC, 2>;
    return vv == DSE_MU_VERTEX_BC1 ? (const void*)mu::mu_batch_kernel<DSE_MU_VERTEX_BC1, 4>
         : vv == DSE_MU_VERTEX_BCB ? (const void*)mu::mu_batch_kernel<DSE_MU_VERTEX_BCB, 4>
                                   : (const void*)mu::mu_batch_kernel<DSE_MU_VERTEX_BC, 4>;
}

// Shared set-up of the batched launches: argument checks, the moment table,
// the per-solve buffers and the cooperative grid; fills b's per-solve fields.
int mu_batch_setup(dse_mu_sweeper* s, const dse_mu_params* params, int64_t S, mu::MuBatch& b, size_t& smem,
                   dse_err* err) {
    if (!s || !params || (S != 2 && S != 4)) return fail(err, DSE_EPARAM, "bad argument (S must be 2 or 4)");
    for (int64_t q = 0; q < S; ++q) {
        int rc = mu_check_params(params + q, err);
        if (rc) return rc;
        if (params[q].omega != params[0].omega || params[q].vertex != params[0].vertex)
            return fail(err, DSE_EPARAM, "batched solves share omega and the vertex");
    }
    if (s->row_start != 0 || s->row_stride != 1) return fail(err, DSE_EPARAM, "batched sweeps need every row");
    CUDA_TRY(cudaSetDevice(s->device));
    dse_mu_params p0 = params[0];
    p0.mode = DSE_MU_MODE_MOMENTS;
    int rc = mu_build_moments(s, p0, err);
    if (rc) return rc;
    const size_t m_int = (size_t)s->m_s * s->m_4;
    const int si = S == 2 ? 0 : 1;
    smem = ((S == 4 ? mu::batch_acc_doubles<4>() : mu::batch_acc_doubles<2>()) + (size_t)mu::kWarps * 6 * S) *
               sizeof(double) + (2 * (size_t)s->m_s + 2) * sizeof(int);
    if (!s->bblocks[si]) {
        int per_sm = 1 << 30, sms = 0;
        for (int vv : {DSE_MU_VERTEX_BC, DSE_MU_VERTEX_BC1, DSE_MU_VERTEX_BCB}) {
            CUDA_TRY(cudaFuncSetAttribute(mu_batch_ptr(vv, S), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int n = 0;
            CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, mu_batch_ptr(vv, S), mu::kThreads, smem));
            per_sm = std::min(per_sm, n);
        }
        CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device));
        if (per_sm < 1) return fail(err, DSE_EENV, "batched kernel does not fit on an SM");
        s->bblocks[si] = per_sm * sms;
    }
    if (!s->d_bNB) {
        const int maxb = std::max(s->bblocks[0], s->bblocks[1]);
        CUDA_TRY(cudaMalloc(&s->d_bNB, sizeof(double2) * 4 * m_int * mu::kMuMaxBatch));
        CUDA_TRY(cudaMalloc(&s->d_berr, sizeof(unsigned long long) * 2 * mu::kMuMaxBatch));
        CUDA_TRY(cudaMalloc(&s->d_bnf, sizeof(int) * 2 * mu::kMuMaxBatch));
        CUDA_TRY(cudaMalloc(&s->d_bstatus, sizeof(long long) * 4 * mu::kMuMaxBatch));
        (void)maxb;
    }
    if (s->bbmax_blocks < s->bblocks[si]) {
        if (s->d_bbmax) cudaFree(s->d_bbmax);
        s->d_bbmax = nullptr;
        CUDA_TRY(cudaMalloc(&s->d_bbmax, sizeof(double) * 3 * mu::kMuMaxBatch * (size_t)s->bblocks[si]));
        s->bbmax_blocks = s->bblocks[si];
    }
    b = mu::MuBatch{};
    b.NB = s->d_bNB;
    b.err = s->d_berr;
    b.nonfinite = s->d_bnf;
    b.bmax = s->d_bbmax;
    b.status = s->d_bstatus;
    for (int64_t q = 0; q < S; ++q) {
        b.mu[q] = params[q].mu;
        b.coeff[q] = params[q].coeff;
        b.z1[q] = params[q].z1;
        b.m0z1[q] = params[q].m0 * params[q].z1;
        b.xi[q] = params[q].xi;
        b.cap[q] = params[q].max_iterations;
    }
    return DSE_OK;
}

int mu_batch_launch(dse_mu_sweeper* s, const dse_mu_params& p0, int64_t S, mu::MuBatch& b, size_t smem, int it_end,
                    cudaStream_t st, dse_err* err) {
    mu::mu_reset_kernel<<<1, 32, 0, st>>>(s->d_ctr, s->d_err, s->d_status, s->d_nonfinite);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    CUDA_TRY(cudaMemsetAsync(s->d_berr, 0xff, sizeof(unsigned long long) * 2 * S, st));
    CUDA_TRY(cudaMemsetAsync(s->d_bnf, 0, sizeof(int) * 2 * S, st));
    CUDA_TRY(cudaMemsetAsync(s->d_bstatus, 0, sizeof(long long) * 4 * S, st));
    dse_mu_params pm = p0;
    pm.mode = DSE_MU_MODE_MOMENTS;
    mu::MuArgs a = mu_make_args(s, pm, 0, it_end, false, true, false);
    void* args[] = {&a, &b};
    CUDA_TRY(cudaLaunchCooperativeKernel(mu_batch_ptr((int)p0.vertex, S), dim3(s->bblocks[S == 2 ? 0 : 1]),
                                         dim3(mu::kThreads), args, smem, st));
    g_launches.fetch_add(1);
    return DSE_OK;
}
}  // namespace

extern "C" {


int dse_mu_batch_sweep(dse_mu_sweeper* s, const dse_mu_params* params, int64_t S, const double* dX_in,
                       double* dX_out, uintptr_t stream, int64_t* failed_row, dse_err* err) {
    ok(err);
    if (!dX_in || !dX_out || !failed_row) return fail(err, DSE_EPARAM, "null argument");
    mu::MuBatch b;
    size_t smem = 0;
    int rc = mu_batch_setup(s, params, S, b, smem, err);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    b.Xh[0] = (double2*)dX_in;
    b.Xh[1] = (double2*)dX_out;
    b.stop = 0;
    rc = mu_batch_launch(s, params[0], S, b, smem, 1, st, err);
    if (rc) return rc;
    unsigned long long er[mu::kMuMaxBatch];
    CUDA_TRY(cudaMemcpyAsync(er, s->d_berr, sizeof(unsigned long long) * S, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int64_t q = 0; q < S; ++q) failed_row[q] = er[q] == ~0ull ? -1 : (int64_t)er[q];
    return DSE_OK;
}

int dse_mu_batch_solve(dse_mu_sweeper* s, const dse_mu_params* params, int64_t S, double* dX0, double* dX1,
                       double* hist, int64_t hist_stride, int64_t* iterations, int32_t* converged,
                       int64_t* failed_iteration, int64_t* failed_row, uintptr_t stream, dse_err* err) {
    ok(err);
    if (!dX0 || !dX1 || !iterations || !converged || !failed_iteration || !failed_row)
        return fail(err, DSE_EPARAM, "null argument");
    mu::MuBatch b;
    size_t smem = 0;
    int rc = mu_batch_setup(s, params, S, b, smem, err);
    if (rc) return rc;
    long long cap = 0;
    for (int64_t q = 0; q < S; ++q) {
        if (params[q].relaxation != 1.0)
            return fail(err, DSE_EPARAM, "batched solves run plain successive approximation (relaxation 1)");
        cap = std::max<long long>(cap, params[q].max_iterations);
    }
    if (hist && hist_stride < cap + 1) return fail(err, DSE_EPARAM, "hist_stride must be >= max_iterations + 1");
    if (cap > (1ll << 30)) return fail(err, DSE_EPARAM, "max_iterations too large");
    cudaStream_t st = (cudaStream_t)stream;
    b.Xh[0] = (double2*)dX0;
    b.Xh[1] = (double2*)dX1;
    b.stop = 1;
    b.hist = hist;
    b.hist_stride = hist_stride;
    rc = mu_batch_launch(s, params[0], S, b, smem, (int)cap, st, err);
    if (rc) return rc;
    long long stt[4 * mu::kMuMaxBatch];
    CUDA_TRY(cudaMemcpyAsync(stt, s->d_bstatus, sizeof(long long) * 4 * S, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int64_t q = 0; q < S; ++q) {
        iterations[q] = stt[4 * q + 0];
        converged[q] = (int32_t)stt[4 * q + 1];
        failed_iteration[q] = stt[4 * q + 2];
        failed_row[q] = stt[4 * q + 2] ? stt[4 * q + 3] : -1;
    }
    return DSE_OK;
}

int dse_mu_sweeper_stats(dse_mu_sweeper* s, int64_t* nominal_points, int64_t* evaluated_points, int32_t* blocks,
                         int64_t* smem_bytes) {
    if (!s) return DSE_EPARAM;
    const int64_t pairs = (int64_t)s->n_rows * s->m_s * s->m_4;
    if (nominal_points) *nominal_points = pairs * s->K;
    if (evaluated_points) *evaluated_points = s->evaluated_pairs < 0 ? -1 : s->evaluated_pairs * s->K;
    if (blocks) *blocks = s->blocks;
    if (smem_bytes) *smem_bytes = (int64_t)s->smem;
    return DSE_OK;
}

/* Anderson acceleration state kept on the device (see include/dse_b200.h). */
// The device the caller's state lives on: made current before any launch (the
// entry points take no device argument; the state pointer names it), and the
// grid cap is derived from that device's SM count.
static int aa_device(const void* ptr, int* blocks_cap, dse_err* err) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        return fail(err, DSE_EPARAM, "Anderson state: not a device pointer");
    }
    CUDA_TRY(cudaSetDevice(at.device));
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, at.device));
    *blocks_cap = 8 * sms;
    return DSE_OK;
}
static int aa_cols(int S, int depth, const int* cols, int ncols, mu::AaCols& c, dse_err* err) {
    if (S < 1 || S > mu::kAaMaxS || depth < 1 || depth > mu::kAaMaxDepth || ncols < 0 || ncols > depth ||
        (ncols > 0 && !cols))
        return fail(err, DSE_EPARAM, "Anderson state: S in 1..%d, depth in 1..%d, ncols <= depth", mu::kAaMaxS,
                    mu::kAaMaxDepth);
    c = mu::AaCols{};
    c.n = ncols;
    for (int k = 0; k < ncols; ++k) {
        if (cols[k] < 0 || cols[k] >= depth) return fail(err, DSE_EPARAM, "column slot out of range");
        c.col[k] = cols[k];
    }
    return DSE_OK;
}

int dse_mu_aa_residual(int32_t S, int64_t n_ext, const double* d_x, const double* d_gx, double* d_f, double* d_fprev,
                       double* d_xprev, double* d_dF, double* d_dX, int32_t depth, int32_t slot, const int32_t* cols,
                       int32_t ncols, double* d_scratch, double* host_out, uintptr_t stream, dse_err* err) {
    ok(err);
    mu::AaCols c;
    int rc = aa_cols(S, depth, cols, ncols, c, err);
    if (rc) return rc;
    if (n_ext < 1 || !d_x || !d_gx || !d_f || !d_fprev || !d_xprev || !d_scratch || !host_out ||
        (depth > 0 && (!d_dF || !d_dX)) || slot >= depth)
        return fail(err, DSE_EPARAM, "bad argument");
    int cap = 0;
    rc = aa_device(d_x, &cap, err);
    if (rc) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // dots first (16-B aligned), then the delta bits
    double2* dots = reinterpret_cast<double2*>(d_scratch);
    unsigned long long* bits = reinterpret_cast<unsigned long long*>(d_scratch + 4 * (size_t)S * ncols);
    CUDA_TRY(cudaMemsetAsync(bits, 0, sizeof(double) * 3 * S, st));
    const long long total = (long long)S * 3 * n_ext;
    const int blocks = (int)std::min<long long>((total + 255) / 256, cap);
    mu::aa_residual_kernel<<<blocks, 256, 0, st>>>(S, n_ext, (const double2*)d_x, (const double2*)d_gx,
                                                   (double2*)d_f, (double2*)d_fprev, (double2*)d_xprev,
                                                   (double2*)d_dF, (double2*)d_dX, depth, slot, bits);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    if (ncols > 0) {
        mu::aa_dots_kernel<<<dim3(ncols, 2, S), 256, 0, st>>>(n_ext, (const double2*)d_f, (const double2*)d_dF, depth,
                                                              slot, c, dots);
        CUDA_TRY(cudaGetLastError());
        g_launches.fetch_add(1);
    }
    const size_t bytes = sizeof(double) * (3 * (size_t)S + 4 * (size_t)S * ncols);
    CUDA_TRY(cudaMemcpyAsync(host_out, d_scratch, bytes, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return DSE_OK;
}

int dse_mu_aa_update(int32_t S, int64_t n_ext, double* d_x, const double* d_f, const double* d_dF, const double* d_dX,
                     int32_t depth, const int32_t* cols, int32_t ncols, const double* gamma, double beta,
                     uintptr_t stream, dse_err* err) {
    ok(err);
    mu::AaCols c;
    int rc = aa_cols(S, depth, cols, ncols, c, err);
    if (rc) return rc;
    if (n_ext < 1 || !d_x || !d_f || (ncols > 0 && (!d_dF || !d_dX || !gamma))) return fail(err, DSE_EPARAM, "bad argument");
    for (int q = 0; q < S; ++q)
        for (int k = 0; k < ncols; ++k)
            c.gamma[q][k] = make_double2(gamma[2 * ((size_t)q * ncols + k)], gamma[2 * ((size_t)q * ncols + k) + 1]);
    int cap = 0;
    rc = aa_device(d_x, &cap, err);
    if (rc) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const long long total = (long long)S * 3 * n_ext;
    const int blocks = (int)std::min<long long>((total + 255) / 256, cap);
    mu::aa_update_kernel<<<blocks, 256, 0, st>>>(S, n_ext, (double2*)d_x, (const double2*)d_f, (const double2*)d_dF,
                                                 (const double2*)d_dX, depth, beta, c);
    CUDA_TRY(cudaGetLastError());
    g_launches.fetch_add(1);
    return DSE_OK;
}

}  // extern "C"
