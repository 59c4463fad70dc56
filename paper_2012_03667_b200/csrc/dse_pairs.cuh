// dse_pairs.cuh -- "pairs" arithmetic (DSE_ARITH_PAIRS): the fast sweep with
// the angular sum of every (row, node) pair factored into five moments that
// are accumulated point by point, then contracted once per pair.  Included
// by dse_b200.cu after the moment kernel (it reuses SweepArgs, the node
// prologue, make_fastj_direct, the history/stop protocol).
//
// Per (row i, node j) the fast summands are e w/kappa (U(r) + V(r)/kappa)
// (A) and e w/kappa (W(r) + X(kq)/kappa) (B) with coefficients constant over
// the angular nodes (make_fastj_direct), kq = q2 - r, kp = r - p2 and
// kappa = p2 + q2 - 2r.  So with rho = 1/kappa
//     S0 = sum ew rho, S1 = sum ew rho r, T0 = sum ew rho^2, T1 = sum ew rho^2 r,
//     T2 = sum ew rho^2 r^2
// the moment-arithmetic contraction (dse_moment_kernel) applies with
// M0 = S0, M1 = S1, M2 = sum ew rho^2 kq kp = -T2 + psum T1 - p2 q2 T0,
// M3 = T1, M4 = T0, M5 = q2 T0 - T1.  Every integrand point is evaluated every
// iteration (one exp, one reciprocal, 23 FP64 instructions); a numpy model of
// exactly this order agrees with the reference's golden sweeps to <= 7.8e-14
// (hybrid), the fast-arithmetic tolerance is 1e-12.
//
// Work: item t = (owned row r, group g of 32 consecutive nodes, chunk c of
// the angles), one WARP per item (lane = node, the lane runs the chunk's
// angles; C = 1 chunk unless the problem has too few (row, group) items to
// fill the GPU -- C depends on N, M, K only, so every GPU and every row
// sharding uses the same partition; the contraction is linear in the
// moments, so each chunk contracts its own), items dealt by atomic
// ticket in decreasing order of evaluated nodes (host table) so warps never
// wait on each other inside an iteration and the tail is cheap items.  Nodes
// outside the row's exact-zero window (the sweep kernel's rule)
// are not evaluated unless a dressing value is non-finite (then NaN reaches
// the sum as in the reference).  A group's partial is the lane xor tree; the
// warp finishing a row's last group sums the G partials in order g = 0..G-1
// and finalises the row (partials in order (g, c)).  Results are bitwise independent of the grid size,
// the schedule and the row sharding.

// One CTA of 20 warps per SM (<= 102 registers, 5 warps per scheduler) with
// the angular loop unrolled 4x: 0.330 ms at config 2 against 0.342 for two
// CTAs of 8 warps unrolled 8x (118 registers).  Warps per SM that are not a
// multiple of 4 load the schedulers unevenly (18: 0.347-0.361, 22: 0.342-0.352);
// 24 warps at 80 registers 0.340; 16 warps in one CTA 0.338 (round 2, fourth
// session; scripts/r02vc.sh, r02vd.sh).
#ifndef DSE_PAIRS_THREADS
#define DSE_PAIRS_THREADS 640
#endif
constexpr int kPairsThreads = DSE_PAIRS_THREADS;
#ifndef DSE_PAIRS_MINB
#define DSE_PAIRS_MINB 1  // (256 threads: 2 CTAs 0.342, 3 (80 regs) 0.359, 4 (64 regs) 0.367 ms)
#endif
#ifndef DSE_PAIRS_UNROLL
#define DSE_PAIRS_UNROLL 4  // 20 warps as 2 x 320: 2 -> 0.360, 3 -> 0.349, 4 -> 0.336; as 1 x 640: 4 -> 0.330, 8 -> 0.335 ms
#endif
constexpr int kPairsUnroll = DSE_PAIRS_UNROLL;
// (sharing one exp between the symmetric angles z, -z -- exp(-kappa(-z)/w2)
// = exp(-2 psum/w2) / exp(-kappa(z)/w2) -- ran 0.338 vs 0.342 ms and moved
// one golden sweep past 1e-12: rejected)
// (an int2 (row, group) item table instead of one int and a division ran
// 0.350 vs 0.342 ms)
// (requesting the next ticket while an item computes ran 0.353 vs 0.341 ms:
// a busy warp then holds an item idle warps could run, the tail grows -- and
// still 0.349 vs 0.341 ms in round 2 with the prefetch stopped 1, 2 or 4
// grid-warps of items before the end; a multiply-high item -> row split
// instead of the division measured no different, 0.342 ms; angle
// chunks C = 2 / 4 at config 2 ran 0.362 / 0.410 ms: per-item overhead;
// round 2, third session: the next ticket requested only after the angular
// loop, its round trip overlapping the reduction and completion fences, ran
// 0.347 vs 0.341 ms, bitwise equal)
// (two accumulator sets for even/odd angles ran 0.344 vs 0.339 ms: the loop
// is FP64-pipe bound, not add-chain bound)
// (an 11-bit exp table with a degree-3 polynomial ran 0.333 ms but put a
// config-2 random-state sweep at 1.1e-12 of the oracle: kept at 8 bits, degree 4)
// (mirror pairs, round 2: the angular nodes are symmetric to ~3e-16, so
// nodes k and K-1-k could share one rz from the positive node (kappa's
// cancelling side stays exact) and the moments fold to (t0+ -/+ t0-) etc.:
// 21 instead of 23 FP64 per point, 0.341 -> 0.319 ms -- but the borrowed rz
// perturbs every negative-side kappa by the SAME node asymmetry in every
// row, a coherent bias that the B channel's cancelling sums amplify: a
// config-2 random-state sweep went from 4.3e-13 to 8.3e-13 of the oracle,
// past the 5e-13 bar.  Not kept.)
// (fewer accumulators: with r = (psum - kappa)/2 and rho kappa = 1, T1 =
// (psum T0 - S0)/2, T2 = (psum T1 - S1)/2, even S1 = (psum S0 - sum ew)/2 --
// 3 to 4 FP64 instructions fewer per point, but a numpy model against long
// double puts the A channel 5-20x further from the exact sums (1.6e-11 to
// 6e-11 vs 3e-12 at config 0): the subtraction reintroduces the cancellation
// that accumulating r-weighted moments avoids.  Not built.)

// Where the time goes (ncu source page, round 2, profiles/r02/SUMMARY.md): 83%
// of the warp samples sit in the angular loop, where the FP64 pipe runs at
// ~87% (stalls: pipe throttle 30%, not selected 27%, fixed-latency wait 21%);
// the other 17% are per-item work (ticket and the dependent loads 6.6%, fence
// 1.7%, row constants / coefficients / reduction ~6%) and the wait at the grid
// barrier (2.6%), and with 5 warps per scheduler every warp outside the loop
// costs pipe time.  Per launch 0.2246 ms is the pipe's floor (23.42 FP64
// instructions per point).  The loop's schedule is sensitive to the code
// around it: builds whose loop differs only in register allocation run
// 0.330-0.344 ms (the fixed-latency wait goes 21% -> 32%), so A/B differences
// under ~4% between structurally different builds are not evidence.  (The same
// operations in two other source orders: 0.338, 0.339 ms; a register cap of 80
// through a larger launch bound: 0.347 ms -- this build's schedule is a good one.)
// Measured and not kept in that session (all bitwise or within the parity
// bars, all slower than 0.330 ms at 640 x 1, unroll 4):
//  - static schedule: every warp an equal contiguous share of the (row, group,
//    chunk) sequence, no tickets, row constants once per row: 0.346-0.354 ms
//    -- warps of one scheduler do not progress alike, the early finishers
//    leave the pipe under-filled;
//  - guided self-scheduling (a batch = 1/(2 warps) of the units left, down to
//    single chunks): 0.340-0.346 ms at best, 0.36+ with 2-4 chunks per group
//    (each extra item costs ~1.5 us of warp time, more than the level finish
//    returns);
//  - a quarter of the rows cut into 4 angle chunks scheduled last: +3 to +10%;
//  - the finishing warp loading the row's partials side by side: 0.341 ms;
//    items only for the groups inside the window (the finishing warp
//    evaluating the outside ones in the non-finite case): 0.342 ms;
//  - the angular loop as a __noinline__ function (a schedule independent of
//    the surrounding code): 0.344 ms.
//  - warp specialisation: 16 (or 20) compute warps that only run the angular
//    loop, fed item descriptors through shared memory by a service warpgroup
//    whose lanes take the tickets, load the rows and do the completion
//    protocol (setmaxnreg moving the service warps' registers to the compute
//    warps, 112 per thread, loop unrolled 8x): bitwise equal, 0.349 ms with 16
//    compute warps, 0.360 with 20 (80 registers) -- warps in the loop full
//    time do not beat 20 warps that each spend a sixth of it on bookkeeping.
__global__ void __launch_bounds__(kPairsThreads, DSE_PAIRS_MINB) dse_pairs_kernel(SweepArgs a) {
    if (a.stop && *a.stop) return;  // sharded solve already stopped (uniform over the grid)
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    double* q2 = sm;
    double* sq = q2 + a.M;
    double* meas = sq + a.M;
    double* aqs = meas + a.M;
    double* bqs = aqs + a.M;
    double* dens = bqs + a.M;
    double2* zz = reinterpret_cast<double2*>(dens + a.M);
    double* etbl = reinterpret_cast<double*>(zz + a.K);
    __shared__ double red[2 * (kPairsThreads / 32)];
    __shared__ int s_bad;
    const int tid = threadIdx.x, lane = tid & 31;
    for (int j = tid; j < a.M; j += blockDim.x) {
        q2[j] = __ldg(a.q2 + j);
        sq[j] = __ldg(a.sq + j);
        meas[j] = __ldg(a.meas + j);
    }
    for (int k = tid; k < a.K; k += blockDim.x) zz[k] = make_double2(__ldg(a.z + k), __ldg(a.zw + k));
    for (int i = tid; i < (1 << kExpTableBits); i += blockDim.x) etbl[i] = __ldg(a.exp_tbl + i);
    __syncthreads();
    const unsigned tbl = smem_addr(etbl);
    const ExpK ek{a.exp_c1, a.nrw2};
    if (a.it_begin == 0 && a.hist && blockIdx.x == 0 && tid == 0)
        write_history(a, 0, __longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll),
                      a.X, a.X + a.N);
    const int C = a.pr_C, G = a.pr_G, GC = G * C;
    const int kc = (a.K + C - 1) / C;  // angles per chunk
    const int n_items = a.n_mrows * GC;
    for (int it = a.it_begin; it < a.it_end; ++it) {
        const int cur = it & 1, nxt = cur ^ 1;
        const double* Ac = a.X + (size_t)(2 * cur) * a.N;
        const double* Bc = Ac + a.N;
        double* An = a.X + (size_t)(2 * nxt) * a.N;
        double* Bn = An + a.N;
        double* dr = a.drow + (size_t)(2 * cur) * a.N;
        if (tid == 0) s_bad = 0;
        __syncthreads();
        int bad = 0;
        for (int j = tid; j < a.M; j += blockDim.x) {  // a_q, b_q, den at the internal nodes (F9)
            const double qq = q2[j];
            const double aq = a.aq_in ? __ldg(a.aq_in + j) : interp_internal(a, Ac, j, qq);
            const double bq = a.bq_in ? __ldg(a.bq_in + j) : interp_internal(a, Bc, j, qq);
            aqs[j] = aq;
            bqs[j] = bq;
            const double den = add(mul(mul(qq, aq), aq), mul(bq, bq));
            dens[j] = den;
            bad |= !isfinite(aq) || !isfinite(bq) || !isfinite(den);
        }
        if (bad) atomicOr(&s_bad, 1);
        __syncthreads();
        const bool any_bad = s_bad != 0;
        // ---- items: one warp each, by ticket
        for (;;) {
            int t = 0;
            if (lane == 0) t = (int)atomicAdd(a.ctr + cur, 1u);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= n_items) break;
            t = __ldg(a.pr_items + t);  // longest first: the iteration's tail is empty groups
            const int r = t / GC, gc = t - r * GC, g = gc / C, c = gc - g * C;
            const int k0 = c * kc, k1 = min(a.K, k0 + kc);
            const int i = a.mrow[r];
            const double p2 = __ldg(a.p2 + i), rp2 = 1.0 / p2, sqp = sqrt(p2);
            const double a_p = __ldcg(Ac + i), b_p = __ldcg(Bc + i);
            const int2 win = __ldg(a.pr_win + r);
            const int j = 32 * g + lane;
            DCHECK(r >= 0 && r < a.n_mrows && g >= 0 && g < G && c >= 0 && c < C && k0 >= 0 && k1 <= a.K, 20);
            DCHECK(i >= 0 && i < a.N && win.x >= 0 && win.y <= a.M, 21);
            const bool all = any_bad || !isfinite(a_p) || !isfinite(b_p);
            const bool active = j < a.M && (all || (j >= win.x && j < win.y));
            double sa = 0.0, sb = 0.0;
            if (active) {
                const double qq = q2[j];
                const double psum = p2 + qq;
                const double sqj = sq[j];
                double S0 = 0.0, S1 = 0.0, T0 = 0.0, T1 = 0.0, T2 = 0.0;
#pragma unroll kPairsUnroll
                for (int k = k0; k < k1; ++k) {
                    const double2 zk = zz[k];
                    // rz in the reference's rounding (kernels.py:189: sqrt(p2) * (sqrt(q2) z)):
                    // kappa = psum - 2 rz cancels near p2 = q2, z = 1, so rz must round as there
                    const double rr = sqp * (sqj * zk.x);
                    const double kap = fma(-2.0, rr, psum);
                    const double ew = zk.y * exp_neg_k2(kap, ek, tbl);
                    const double rho = rcp_nr(kap);
                    const double t0 = ew * rho;
                    S0 += t0;
                    S1 = fma(t0, rr, S1);
                    const double t4 = t0 * rho;
                    T0 += t4;
                    const double t5 = t4 * rr;
                    T1 += t5;
                    T2 = fma(t5, rr, T2);
                }
                const double M2 = fma(psum, T1, -T2) - (p2 * qq) * T0;
                const double M5 = fma(qq, T0, -T1);
                const FastJ f = make_fastj_direct(p2, a_p, b_p, qq, sq[j], meas[j], aqs[j], bqs[j], dens[j], a.coeff,
                                                  rp2);
                sa = fma(f.uA0, S0, fma(f.uA1, S1, fma(f.c2A2, M2, f.vA * T1)));
                sb = fma(f.wB0, S0, fma(f.wB1, S1, fma(f.xB0, T0, f.xB1 * M5)));
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                sa += __shfl_xor_sync(0xffffffffu, sa, o);
                sb += __shfl_xor_sync(0xffffffffu, sb, o);
            }
            if (lane == 0) {
                a.pr_part[(size_t)r * GC + gc] = make_double2(sa, sb);
                // (an acq_rel atomic_ref RMW instead of the two fences measured
                // slower, 0.342 -> 0.347 ms)
                __threadfence();
                const unsigned done = atomicAdd(a.pr_cnt + r, 1u);
                if (done == (unsigned)GC - 1) {  // last item of the row: sum the partials in order
                    __threadfence();
                    const double2* pp = a.pr_part + (size_t)r * GC;
                    double ta = 0.0, tb = 0.0;
                    for (int q = 0; q < GC; ++q) {
                        const double2 v = __ldcg(pp + q);
                        ta += v.x;
                        tb += v.y;
                    }
                    a.pr_cnt[r] = 0u;
                    double an = add(a.z1, ta), bn = add(a.m0z1, tb);
                    if (!(isfinite(an) && isfinite(bn))) atomicMin(a.err_row + cur, (unsigned long long)i);
                    if (a.relax != 1.0) {
                        an = add(mul(a.relax, an), mul(sub(1.0, a.relax), a_p));
                        bn = add(mul(a.relax, bn), mul(sub(1.0, a.relax), b_p));
                    }
                    An[i] = an;
                    Bn[i] = bn;
                    // fused all-gather: this row goes to every rank's receive
                    // buffer now, overlapping the rest of the sweep
                    for (int q = 0; q < a.pr_world; ++q) {
                        double* dst = a.pr_peer[q] + (size_t)a.pr_rank * 2 * a.pr_per;
                        dst[r] = an;
                        dst[a.pr_per + r] = bn;
                    }
                    dr[i] = fabs(sub(an, a_p));
                    dr[a.N + i] = fabs(sub(bn, b_p));
                }
            }
        }
        if (blockIdx.x == 0 && tid == 0) {
            a.err_row[nxt] = kNoRow;
            a.ctr[nxt] = 0u;
        }
        grid.sync();
        double da = 0.0, db = 0.0;  // the sweep kernel's stop rule (iteration.py:34-39)
        for (int q = tid; q < a.n_mrows; q += blockDim.x) {
            const int i = a.mrow[q];
            da = nanmax(da, __ldcg(dr + i));
            db = nanmax(db, __ldcg(dr + a.N + i));
        }
        block_max2(da, db, red);
        const unsigned long long er = *(volatile unsigned long long*)(a.err_row + cur);
        const bool failed = er != kNoRow;
        const bool conv = !failed && (da < a.xi) && (db < a.xi);
        if (blockIdx.x == 0 && tid == 0) {
            if (!failed) {
                if (a.hist) write_history(a, it + 1, da, db, An, Bn);  // (the pre-bracketed form cost the
                                                                          // sweep 1.8%: 0.341 -> 0.347 ms)
                a.status[0] = it + 1;
                a.status[1] = conv ? 1 : 0;
                a.status[3] = nxt;
            } else {
                a.status[2] = it + 1;
            }
        }
        if (failed || conv) break;
    }
}
