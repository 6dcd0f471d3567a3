// admm_onchip.cuh -- cluster-row persistent ADMM kernel: the on-chip engine
// for PHEV-sized problems (BASELINE.json configs[0], [1]; Appendix A,
// Eq. (6a)-(6i), residuals :464-479, adaptive rho :318-324).
//
// Scenario row j = one thread-block cluster of T CTAs; tile 0 holds steps
// [0, TC0), tile r >= 1 holds [TC0 + (r-1) TC, ...).  Coefficients (prepared:
// a2/q, a1/q, b2, b1, b = 1.5 b1/b2, 1/b2^2), bounds, demand, x and v = s - mu
// stay in shared memory for the whole call.  Each bulk thread owns (usually)
// one cell, so an iteration is one Gauss-Seidel cell + one reduction + one
// cluster barrier + the scalar row update.
//
//  * capacity coupling (6b)/(6g)/(6d)/(6i): the row sum sum_k (b2 x^2 + b1 x)
//    is accumulated in 64-bit fixed point (per-source scale 2^E chosen at
//    set_problem so that n * max|b2 x^2 + b1 x| over the box < 2^62): a warp
//    sums with three redux.sync over 21-bit limbs, lane t < T adds the warp
//    sum into cluster-mate t's accumulator (DSMEM atomic), one cluster.sync,
//    and every CTA of the row performs the identical row update.  Integer
//    addition is associative, so the sum is exact up to the per-term rounding
//    (<= n 2^-63 of the bound) and independent of order: deterministic;
//  * consensus (6c)/(6h), the only cross-scenario coupling, touches only the
//    k = 0 cell.  Tile-0 CTAs carry one extra "consensus warp": at the start
//    of iteration t it reads the q contributions of iteration t-1 (one L2
//    round trip: epoch slots that hold a sentinel until written, polled with
//    relaxed loads + one acquire fence), applies (6h), resets its own slot of
//    the buffer iteration t+1 publishes into, computes the k = 0 cell and
//    publishes x_1 - nu (fence + relaxed stores).  No CTA waits on a counter
//    for the consensus; four rotating buffers make the reset race-free: when
//    a consensus warp has observed every contribution of iteration t-1, every
//    CTA has passed the row barrier of t-2, so nobody still reads the buffer
//    of t-3 = t+1 (mod 4).  Tile 0 gets fewer cells (TC0 < TC)
//    so the k = 0 chain is not starved of issue slots by its bulk warps;
//  * residual checks (every check_every): every term is a max (or min),
//    combined with order-independent atomics on order-preserving integer keys
//    (DSMEM for the row terms, global for the grid terms), one counter
//    barrier, one round trip to read the combined slots; every CTA takes the
//    same termination / rho decision.
#pragma once
#include <cooperative_groups.h>

#include "admm_kernels.cuh"

namespace admm_dev {

constexpr unsigned long long PUB_EMPTY = 0xFFF4DEADBEEF0001ull;  // sNaN payload: never computed
constexpr int PUB_BUFS = 4;
constexpr int ONCHIP_MAX_WARPS = 16;     // 15 bulk warps + 1 consensus warp (128 regs)
constexpr int ONCHIP_MAX_T = 16;         // tiles (CTAs) per cluster
constexpr int CHK_SLOTS = 6 + 2 * MAXM;  // r1 r2 r3 s1 s2 s3 | max_j x_1 [MAXM] | min_j x_1 [MAXM]

#ifdef ADMM_PHASE_PROF  // development build only: per-phase clock64() totals of CTA 0
__device__ unsigned long long g_phase[3][8];
#define PHASE(k)                                  \
    if (prof_on) {                                \
        const unsigned long long _c = clock64();  \
        ph_acc[k] += _c - ph_last;                \
        ph_last = _c;                             \
    }
#else
#define PHASE(k)
#endif

__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_count(const unsigned long long* p, unsigned long long target) {
    while (ld_acquire(p) < target) {
    }
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const void* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(void* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// okey / okey_inv / warp_sum_u64: admm_kernels.cuh

// (6c) x1^{(i)} = (1/q_total) sum_j c^{(i,j)} over one publication buffer
// [M][q] (reading G1: the mean).  Warp-collective; every lane returns the same
// x1, and every warp that reads the same buffer gets the same bits
// (lane-strided partial sums in j order, then a fixed butterfly).
template <int M>
__device__ __forceinline__ void read_consensus(const double* buf, long long q, double qtot, double* x1) {
    const int lane = threadIdx.x & 31;
    double s[M];
#pragma unroll
    for (int i = 0; i < M; ++i) s[i] = 0.0;
    constexpr int U = 4;  // slots per lane per pass: q <= 128 in one round trip
    for (long long base = 0; base < q; base += 32 * U) {
        double v[U][M];
        bool ok;
        do {
            ok = true;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long jj = base + u * 32 + lane;
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    if (jj < q) {
                        const unsigned long long b = ld_relaxed_u64(buf + (long long)i * q + jj);
                        v[u][i] = __longlong_as_double((long long)b);
                        ok = ok && (b != PUB_EMPTY);
                    } else {
                        v[u][i] = 0.0;
                    }
                }
            }
        } while (!__all_sync(0xffffffffu, ok));
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < M; ++i) s[i] += v[u][i];
    }
    fence_acq_rel_gpu();  // acquire side of the publishers' fence + relaxed stores
#pragma unroll
    for (int i = 0; i < M; ++i) x1[i] = warp_sum(s[i]) / qtot;
}

struct CArgs {
    int TC0, TC, T, G;
    double fx_scale[MAXM], fx_inv[MAXM];  // fixed-point scale 2^E_i of the row sums
    // prepared per-element constants [m][q][n_pad]: b = 1.5 b1/b2, 1/b2^2 (0 if b2 = 0)
    const double *bq, *ib2s;
    double *pub;                // [PUB_BUFS][m][q] consensus contributions x_1 - nu (epoch slots)
    unsigned long long *chk;    // [3][CHK_SLOTS] check maxima (ordered keys), rotating sets
    unsigned long long *cnt;    // [16] check-barrier arrivals (zeroed per launch)
};

// before each launch: every publication slot = sentinel, check sets = identities
__global__ void onchip_reset_kernel(double* pub, long long nslots, unsigned long long* chk) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nslots;
         t += (long long)gridDim.x * blockDim.x)
        pub[t] = __longlong_as_double((long long)PUB_EMPTY);
    if (blockIdx.x == 0)
        for (int t = threadIdx.x; t < 3 * CHK_SLOTS; t += blockDim.x)
            chk[t] = (t % CHK_SLOTS) >= 6 + MAXM ? ~0ull : 0ull;
}

// prepared constants (once per problem): b = 1.5 b1/b2, 1/b2^2
__global__ void prep_kernel(long long NE, const double* b2, const double* b1, double* bq, double* ib2s) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NE;
         t += (long long)gridDim.x * blockDim.x) {
        const double v2 = b2[t];
        bq[t] = v2 != 0.0 ? 1.5 * b1[t] / v2 : 0.0;
        ib2s[t] = v2 != 0.0 ? 1.0 / (v2 * v2) : 0.0;
    }
}

template <int M, int MODE>
__global__ void __launch_bounds__(ONCHIP_MAX_WARPS * 32) persist_cluster_kernel(KArgs a, CArgs p) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double sm[];
    const int TCM = max(p.TC0, p.TC);  // shared-memory row stride
    double* s_a2q = sm;
    double* s_a1q = s_a2q + M * TCM;
    double* s_b2 = s_a1q + M * TCM;
    double* s_b1 = s_b2 + M * TCM;
    double* s_bq = s_b1 + M * TCM;
    double* s_ib = s_bq + M * TCM;
    double* s_lo = s_ib + M * TCM;
    double* s_hi = s_lo + M * TCM;
    double* s_x = s_hi + M * TCM;
    double* s_y = s_x + M * TCM;
    double* s_v = s_y + TCM;

    __shared__ unsigned long long s_acc[2][M];       // fixed-point row sums, added by mates
    __shared__ double s_dgp[ONCHIP_MAX_T][2 * M];    // per-tile max / min of dg (checks), by mates
    __shared__ double s_wred[ONCHIP_MAX_WARPS][2 * M + 2];  // per-warp check maxima
    __shared__ double s_zl[M], s_x1[M], s_rho[4], s_R[4], s_kap, s_f[4], s_t[2];
    __shared__ int s_flag[2];

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int nbw = nw - 1;  // bulk warps; warp nbw = consensus warp (active in tile 0 only)
    const int nbt = nbw * 32;
    const bool cons_warp = (wid == nbw);
    const int T = p.T;
    const long long j = blockIdx.x / T;
    const int tile = (int)cluster.block_rank();
    const int k0 = tile == 0 ? 0 : p.TC0 + (tile - 1) * p.TC;
    const int ncell = min(tile == 0 ? p.TC0 : p.TC, a.n - k0);
    const long long qn = a.q * (long long)a.n_pad;
    const long long qq = a.q;
    const DParams& P = *a.prm;
    const double nd = a.nd;
    const double qtot = (double)a.q_total;
    const bool single = (a.q_total == 1);  // q = 1: x1 = own contribution, no exchange

    const long long it0 = *(volatile long long*)a.iter;
    const Ctrl& cin = a.ctrl[it0 & 1];
    if (cin.done || it0 >= P.iter_limit) return;  // uniform over the grid

    const double iq = a.inv_q;
    for (int t = tid; t < M * TCM; t += blockDim.x) {
        const int i = t / TCM, c = t - i * TCM;
        const bool ok = c < ncell;
        const long long e = (long long)i * qn + j * a.n_pad + k0 + c;
        const long long bk = (long long)i * a.n_pad + k0 + c;
        s_a2q[t] = ok ? a.a2[e] * iq : 0.0;
        s_a1q[t] = ok ? a.a1[e] * iq : 0.0;
        s_b2[t] = ok ? a.b2[e] : 0.0;
        s_b1[t] = ok ? a.b1[e] : 0.0;
        s_bq[t] = ok ? p.bq[e] : 0.0;
        s_ib[t] = ok ? p.ib2s[e] : 0.0;
        s_lo[t] = ok ? a.lo[bk] : 0.0;
        s_hi[t] = ok ? a.hi[bk] : 0.0;
        s_x[t] = ok ? a.x[e] : 0.0;
    }
    for (int c = tid; c < TCM; c += blockDim.x) {
        const bool ok = c < ncell;
        const double vv = ok ? a.v[j * a.n_pad + k0 + c] : 0.0;
        s_y[c] = ok ? a.y[j * a.n_pad + k0 + c] : 0.0;
        s_v[c] = vv < 0.0 ? vv * cin.f[2] : vv;
    }
    // row scalars of source i live in thread i (< M) of every CTA of the row
    double r_lam = 0.0, r_p = 0.0, r_h = 0.0, r_zeta = 0.0, r_c = 0.0, r_sb0 = 0.0;
    double r_r2 = 0.0, r_r3 = 0.0, r_s1 = 0.0, r_s2 = 0.0;
    if (tid < M) {
        const long long rix = (long long)tid * qq + j;
        r_lam = a.lam[rix] * cin.f[0];
        r_p = a.p[rix] * cin.f[1];
        r_h = a.h[rix];
        r_zeta = a.zeta[rix];
        r_c = a.c[tid];
        r_sb0 = a.sb0[rix];
        s_zl[tid] = r_zeta + r_lam;
        s_x1[tid] = cin.x1[tid];
        s_acc[0][tid] = 0ull;
        s_acc[1][tid] = 0ull;
    }
    // consensus warp (tile 0), lane i < M: nu, x1, x_1 and the last contribution of source i
    double c_nu = 0.0, c_x1 = 0.0, c_x0 = 0.0, c_pub = 0.0, c_fnu = 1.0;
    if (cons_warp && tile == 0 && lane < M) {
        const long long rix = (long long)lane * qq + j;
        double nu = a.nu[rix];
        if (cin.nu_pending) nu = nu + cin.x1[lane] - a.x[(long long)lane * qn + j * a.n_pad];
        c_nu = nu * cin.f[3];
        c_x1 = cin.x1[lane];
    }
    if (tid == 0) {
        for (int l = 0; l < 4; ++l) {
            s_rho[l] = cin.rho[l];
            s_f[l] = 1.0;
        }
        s_R[0] = cin.rho[0];
        s_R[1] = cin.rho[2];
        s_R[2] = cin.rho[3];
        s_R[3] = 1.0 / cin.rho[0];
        s_kap = cin.rho[1] / (cin.rho[0] + nd * cin.rho[1]);
    }
    double fxs[M], fxi[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        fxs[i] = p.fx_scale[i];
        fxi[i] = p.fx_inv[i];
    }
    double l_r = cin.r, l_sigma = cin.sigma;
    int l_status = cin.status, l_checks = cin.checks, l_err = cin.err, l_done = 0;
    const int ce = P.check_every;
    unsigned long long nchk = 0;
    bool x1_known = true;  // consensus warp: c_x1 holds x1 of the previous iteration
    __syncthreads();
    cluster.sync();  // mates' shared memory is live before any DSMEM access
#ifdef ADMM_PHASE_PROF
    const bool prof_on = (blockIdx.x == 0 && (tid == 0 || tid == nbt)) || (blockIdx.x == 1 && tid == 0);
    unsigned long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ph_last = clock64();
#endif

    // DSMEM address of cluster-mate `lane`'s row accumulators (lanes < T), mapped once
    unsigned long long* mate_acc =
        lane < T ? cluster.map_shared_rank(&s_acc[0][0], lane) : &s_acc[0][0];
    const long long lim = P.iter_limit;
    int until_chk = ce > 0 ? (int)(ce - 1 - it0 % ce) : -1;  // iterations until the next check
    long long it = it0;
    for (; it < lim; ++it) {
        const int par = (int)(it & 1);
        const bool is_check = (until_chk == 0);
        until_chk = is_check ? ce - 1 : until_chk - 1;
        double R[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) R[l] = s_R[l];
        double zl[M];
#pragma unroll
        for (int i = 0; i < M; ++i) zl[i] = s_zl[i];

        double dgx[M], dgn[M];
        long long fx[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            fx[i] = 0;
            dgx[i] = -INFINITY;
            dgn[i] = INFINITY;
        }
        double my_r1 = 0.0, my_s3 = 0.0;
        if (!cons_warp) {
            // ---- bulk cells: every cell of the tile except the consensus cell k = 0.
            // Pairs (cc, cc + nbt) go through the interleaved two-cell chain.
            for (int cc = tid; cc < ncell; cc += 2 * nbt) {
                const int c2 = cc + nbt;
                const bool two = (c2 < ncell) && (k0 + cc != 0);
                if (two) {
                    const int cs2[2] = {cc, c2};
                    double xo[M][2], xn[M][2], yy[2], vv[2], se[2], me[2];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
#pragma unroll
                        for (int i = 0; i < M; ++i) xo[i][u] = s_x[i * TCM + cs2[u]];
                        vv[u] = s_v[cs2[u]];
                        yy[u] = s_y[cs2[u]];
                        se[u] = fmax(vv[u], 0.0);
                        me[u] = vv[u] < 0.0 ? -vv[u] : 0.0;
                    }
                    gs_cell2_smem<M, MODE>(s_a2q, s_a1q, s_b2, s_b1, s_bq, s_ib, s_lo, s_hi, TCM, cs2,
                                           xo, xn, yy, se, me, zl, R);
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int c = cs2[u];
                        double txo[M], txn[M];
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            txo[i] = xo[i][u];
                            txn[i] = xn[i][u];
                        }
                        s_v[c] = cell_tail<M>(txo, txn, yy[u], vv[u], 1.0, is_check, my_r1, my_s3);
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            const double b2 = s_b2[i * TCM + c], b1 = s_b1[i * TCM + c];
                            s_x[i * TCM + c] = txn[i];
                            if ((a.gfree >> i) & 1u) continue;  // g = 0: no row sum, dg = 0
                            fx[i] += __double2ll_rn(fma(b2, txn[i], b1) * txn[i] * fxs[i]);
                            if (is_check) {
                                const double dg = (txn[i] - txo[i]) * fma(b2, txn[i] + txo[i], b1);
                                dgx[i] = fmax(dgx[i], dg);
                                dgn[i] = fmin(dgn[i], dg);
                            }
                        }
                    }
                    continue;
                }
#pragma unroll 1
                for (int c = cc; c < ncell && c <= cc + nbt; c += nbt) {
                    if (k0 + c == 0) continue;
                    double a2q[M], a1q[M], cb2[M], cb1[M], bq[M], ib[M], clo[M], chi[M], xo[M], xn[M],
                        dummy[M];
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        const int e = i * TCM + c;
                        a2q[i] = s_a2q[e]; a1q[i] = s_a1q[e]; cb2[i] = s_b2[e]; cb1[i] = s_b1[e];
                        bq[i] = s_bq[e]; ib[i] = s_ib[e]; clo[i] = s_lo[e]; chi[i] = s_hi[e];
                        xo[i] = s_x[e];
                        dummy[i] = 0.0;
                    }
                    const double vv = s_v[c];
                    const double yy = s_y[c];
                    gs_cell_prep<M, MODE>(a2q, a1q, cb2, cb1, bq, ib, clo, chi, xo, xn, yy, fmax(vv, 0.0),
                                          vv < 0.0 ? -vv : 0.0, zl, R, false, dummy);
                    s_v[c] = cell_tail<M>(xo, xn, yy, vv, 1.0, is_check, my_r1, my_s3);
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        s_x[i * TCM + c] = xn[i];
                        if ((a.gfree >> i) & 1u) continue;
                        fx[i] += __double2ll_rn(fma(cb2[i], xn[i], cb1[i]) * xn[i] * fxs[i]);
                        if (is_check) {
                            const double dg = (xn[i] - xo[i]) * fma(cb2[i], xn[i] + xo[i], cb1[i]);
                            dgx[i] = fmax(dgx[i], dg);
                            dgn[i] = fmin(dgn[i], dg);
                        }
                    }
                }
            }
        } else if (tile == 0) {
            // ---- consensus warp: x1 of iteration it-1 and (6h), then the k = 0 cell
            if (!x1_known) {
                double x1v[M];
                if (single) {
#pragma unroll
                    for (int i = 0; i < M; ++i) x1v[i] = __shfl_sync(0xffffffffu, c_pub, i);
                } else {
                    read_consensus<M>(p.pub + (size_t)((it - 1) & (PUB_BUFS - 1)) * a.m * qq, qq, qtot,
                                      x1v);
                }
#pragma unroll
                for (int i = 0; i < M; ++i)
                    if (lane == i) c_x1 = x1v[i];
                if (lane < M) {
                    c_nu = (c_nu + c_x1 - c_x0) * c_fnu;  // (6h) of iteration it-1
                    c_fnu = 1.0;
                }
            }
            x1_known = false;
            PHASE(2)
            // reset this row's slots of the buffer iteration it+1 publishes into
            if (lane == 0)
#pragma unroll
                for (int i = 0; i < M; ++i)
                    st_relaxed_u64(p.pub + ((size_t)((it + 1) & (PUB_BUFS - 1)) * a.m + i) * qq + j,
                                   PUB_EMPTY);
            double x1nu[M], cnu[M];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                cnu[i] = __shfl_sync(0xffffffffu, c_nu, i);
                x1nu[i] = __shfl_sync(0xffffffffu, c_x1, i) + cnu[i];
            }
            double xk0[M];
#pragma unroll
            for (int i = 0; i < M; ++i) xk0[i] = 0.0;
            if (lane == 0) {
                double a2q[M], a1q[M], cb2[M], cb1[M], bq[M], ib[M], clo[M], chi[M], xo[M];
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const int e = i * TCM;
                    a2q[i] = s_a2q[e]; a1q[i] = s_a1q[e]; cb2[i] = s_b2[e]; cb1[i] = s_b1[e];
                    bq[i] = s_bq[e]; ib[i] = s_ib[e]; clo[i] = s_lo[e]; chi[i] = s_hi[e];
                    xo[i] = s_x[e];
                }
                const double vv = s_v[0];
                const double yy = s_y[0];
                gs_cell_prep<M, MODE>(a2q, a1q, cb2, cb1, bq, ib, clo, chi, xo, xk0, yy, fmax(vv, 0.0),
                                      vv < 0.0 ? -vv : 0.0, zl, R, true, x1nu);
                // (6c)'s contribution x_1 - nu (nu before (6h)): published first
                if (!single || is_check) {  // q = 1: only the residual check reads it
                    fence_acq_rel_gpu();
#pragma unroll
                    for (int i = 0; i < M; ++i)
                        st_relaxed_u64(p.pub + ((size_t)(it & (PUB_BUFS - 1)) * a.m + i) * qq + j,
                                       (unsigned long long)__double_as_longlong(xk0[i] - cnu[i]));
                }
                PHASE(3)
                s_v[0] = cell_tail<M>(xo, xk0, yy, vv, 1.0, is_check, my_r1, my_s3);
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    s_x[i * TCM] = xk0[i];
                    fx[i] += __double2ll_rn(fma(cb2[i], xk0[i], cb1[i]) * xk0[i] * fxs[i]);
                    if (is_check) {
                        const double dg = (xk0[i] - xo[i]) * fma(cb2[i], xk0[i] + xo[i], cb1[i]);
                        dgx[i] = fmax(dgx[i], dg);
                        dgn[i] = fmin(dgn[i], dg);
                        // max/min over j of x_1 for the consensus residual
                        unsigned long long* cs = p.chk + (size_t)(nchk % 3) * CHK_SLOTS;
                        atomicMax(cs + 6 + i, okey(xk0[i]));
                        atomicMin(cs + 6 + MAXM + i, okey(xk0[i]));
                    }
                }
            }
            // lanes i < M keep x_1 and the contribution for (6h) / the q = 1 path
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const double x0 = __shfl_sync(0xffffffffu, xk0[i], 0);
                if (lane == i) {
                    c_x0 = x0;
                    c_pub = x0 - cnu[i];
                }
            }
        }
        PHASE(0)
        // ---- row partials: exact fixed-point warp sums, DSMEM adds into every mate
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const unsigned long long ws = warp_sum_u64((unsigned long long)fx[i]);
            if (lane < T && ws != 0ull) atomicAdd(mate_acc + par * M + i, ws);
        }
        double cta_r1 = 0.0, cta_s3 = 0.0;
        if (is_check) {
            // (checks only) tile maxima/minima of dg and CTA maxima of r1, s3: warp
            // reductions, one CTA reduction in warp 0, DSMEM stores into every mate
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const double mx = warp_max(dgx[i]), mn = warp_min(dgn[i]);
                if (lane == 0) {
                    s_wred[wid][i] = mx;
                    s_wred[wid][M + i] = mn;
                }
            }
            const double r1 = warp_max(my_r1), s3 = warp_max(my_s3);
            if (lane == 0) {
                s_wred[wid][2 * M] = r1;
                s_wred[wid][2 * M + 1] = s3;
            }
            __syncthreads();
            if (wid == 0) {
                double v[2 * M];
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    v[i] = warp_max(lane < nw ? s_wred[lane][i] : -INFINITY);
                    v[M + i] = warp_min(lane < nw ? s_wred[lane][M + i] : INFINITY);
                }
                cta_r1 = warp_max(lane < nw ? s_wred[lane][2 * M] : 0.0);
                cta_s3 = warp_max(lane < nw ? s_wred[lane][2 * M + 1] : 0.0);
                if (lane < T) {
                    double* dst = cluster.map_shared_rank(&s_dgp[tile][0], lane);
#pragma unroll
                    for (int u = 0; u < 2 * M; ++u) dst[u] = v[u];
                }
            }
        }
        PHASE(1)
        cluster.sync();  // all partials of row j are in every CTA's s_acc[par] (and s_dgp)
        PHASE(4)

        // ---- row update (6b),(6g),(6d),(6i) via identity I1, identical in every CTA:
        //   W = sum_k g - n lam, t = h + p - W, lam' = kappa t, zeta' = lam' - lam,
        //   1'z' = W + n lam', h' = min(c, 1'z' - p), p' = p + h' - 1'z'
        if (tid < M) {
            const double sg = (double)(long long)s_acc[par][tid] * fxi[tid];
            s_acc[par][tid] = 0ull;  // mates add into this buffer again after the next barrier
            double mx = -INFINITY, mn = INFINITY;
            if (is_check)  // s_dgp is rewritten only at the next check, 2+ barriers later
                for (int t = 0; t < T; ++t) {
                    mx = fmax(mx, s_dgp[t][tid]);
                    mn = fmin(mn, s_dgp[t][M + tid]);
                }
            if ((a.gfree >> tid) & 1u) mx = mn = 0.0;  // g-free source: dg = 0 for every k
            const double W = (sg + r_sb0) - nd * r_lam;
            const double t = (r_h + r_p) - W;
            const double lam = s_kap * t;
            const double zeta = lam - r_lam;
            const double oneTz = W + nd * lam;
            const double h = fmin(r_c, oneTz - r_p);
            const double pn = (r_p + h) - oneTz;
            if (is_check) {
                const double dz = zeta - r_zeta;
                r_r2 = fabs(zeta);
                r_r3 = fabs(h - oneTz);
                r_s1 = fmax(mx + dz, -(mn + dz));
                r_s2 = fabs(h - r_h);
            }
            r_lam = lam;
            r_zeta = zeta;
            r_h = h;
            r_p = pn;
            s_zl[tid] = zeta + lam;
        }
        PHASE(5)

        if (is_check) {
            unsigned long long* cs = p.chk + (size_t)(nchk % 3) * CHK_SLOTS;
            if (tile == 0 && tid < M) {
                atomicMax(cs + 1, okey(r_r2));
                atomicMax(cs + 2, okey(r_r3));
                atomicMax(cs + 3, okey(r_s1));
                atomicMax(cs + 4, okey(r_s2));
            }
            if (tid == 0) {
                atomicMax(cs + 0, okey(cta_r1));
                atomicMax(cs + 5, okey(cta_s3));
            }
            __syncthreads();
            ++nchk;
            if (tid == 0) {
                __threadfence();
                red_release_add(p.cnt, 1ull);
                wait_count(p.cnt, nchk * (unsigned long long)p.G);
            }
            __syncthreads();
            if (wid == 0) {
                // x1 of this iteration (same reduction as the consensus warps)
                double x1v[M];
                read_consensus<M>(p.pub + (size_t)(it & (PUB_BUFS - 1)) * a.m * qq, qq, qtot, x1v);
                const unsigned long long kv = lane < CHK_SLOTS ? ld_relaxed_u64(cs + lane) : 0ull;
                double v[CHK_SLOTS];
#pragma unroll
                for (int s = 0; s < CHK_SLOTS; ++s) v[s] = okey_inv(__shfl_sync(0xffffffffu, kv, s));
                if (lane == 0) {
                    // max_j |x_1^{(i,j)} - x1| = max(max_j x_1 - x1, x1 - min_j x_1) exactly
                    double t3 = 0.0;
                    for (int i = 0; i < M; ++i) {
                        t3 = fmax(t3, fmax(v[6 + i] - x1v[i], x1v[i] - v[6 + MAXM + i]));
                        s_x1[i] = x1v[i];
                    }
                    double tt[7] = {v[0], v[1], v[2], t3, v[3], v[4], v[5]};
                    double rho[4], rn[4], fl[4], r, sg, fac, s123[3];
                    for (int l = 0; l < 4; ++l) rho[l] = s_rho[l];
                    const int conv = check_decide(P, rho, tt, rn, fl, &r, &sg, &fac, s123);
                    if (blockIdx.x == 0 && a.hist && a.hist_cap > 0)
                        write_hist(a.hist + (size_t)(l_checks % a.hist_cap) * HCOLS, it + 1, r, sg,
                                   rho, tt, s123, conv, fac);
                    for (int l = 0; l < 4; ++l) {
                        s_rho[l] = rn[l];
                        s_f[l] = fl[l];
                    }
                    s_R[0] = rn[0];
                    s_R[1] = rn[2];
                    s_R[2] = rn[3];
                    s_R[3] = 1.0 / rn[0];
                    s_kap = rn[1] / (rn[0] + nd * rn[1]);
                    s_t[0] = r;
                    s_t[1] = sg;
                    s_flag[0] = conv;
                    s_flag[1] = (!isfinite(r) || !isfinite(sg)) ? 1 : 0;
                }
                // CTA 0 resets the set the check after next combines into: its readers
                // (check nchk-2) are done, its writers start after the next barrier
                if (blockIdx.x == 0 && lane < CHK_SLOTS)
                    st_relaxed_u64(p.chk + (size_t)((nchk + 1) % 3) * CHK_SLOTS + lane,
                                   lane >= 6 + MAXM ? ~0ull : 0ull);
            }
            __syncthreads();
            l_r = s_t[0];
            l_sigma = s_t[1];
            l_status = s_flag[0];
            l_checks += 1;
            if (s_flag[1]) l_err = 1;
            // dual rescale (reading G11): lam<->rho1, p<->rho2, mu<->rho3, nu<->rho4; the
            // consensus warp applies (6h) with the x1 just computed, then f3
            if (tid < M) {
                r_lam *= s_f[0];
                r_p *= s_f[1];
                s_zl[tid] = r_zeta + r_lam;
            }
            if (cons_warp && tile == 0 && lane < M) {
                c_x1 = s_x1[lane];
                c_nu = (c_nu + c_x1 - c_x0) * s_f[3];
                c_fnu = 1.0;
            }
            if (cons_warp && tile == 0) x1_known = true;
            const double f2 = s_f[2];
            if (f2 != 1.0)
                for (int c = tid; c < ncell; c += blockDim.x)
                    if (s_v[c] < 0.0) s_v[c] *= f2;
            if (l_err || (l_status && P.stop_on_conv)) l_done = 1;
            __syncthreads();
            if (tid < 4) s_f[tid] = 1.0;
        }
        PHASE(6)
        __syncthreads();
        PHASE(7)
        if (l_done) {
            ++it;
            break;
        }
    }
#ifdef ADMM_PHASE_PROF
    if (prof_on)
        for (int k = 0; k < 8; ++k) g_phase[blockIdx.x == 1 ? 2 : (tid == 0 ? 0 : 1)][k] = ph_acc[k];
#endif
    // ---- (6h) of the last iteration if it was not a check, then write back
    if (cons_warp && tile == 0 && !x1_known) {
        double x1v[M];
        if (single) {
#pragma unroll
            for (int i = 0; i < M; ++i) x1v[i] = __shfl_sync(0xffffffffu, c_pub, i);
        } else {
            read_consensus<M>(p.pub + (size_t)((it - 1) & (PUB_BUFS - 1)) * a.m * qq, qq, qtot, x1v);
        }
#pragma unroll
        for (int i = 0; i < M; ++i)
            if (lane == i) c_x1 = x1v[i];
        if (lane < M) c_nu = (c_nu + c_x1 - c_x0) * c_fnu;
    }
    if (cons_warp && tile == 0 && lane < M) s_x1[lane] = c_x1;
    __syncthreads();
    for (int t = tid; t < M * TCM; t += blockDim.x) {
        const int i = t / TCM, c = t - i * TCM;
        if (c < ncell) a.x[(long long)i * qn + j * a.n_pad + k0 + c] = s_x[t];
    }
    for (int c = tid; c < ncell; c += blockDim.x) a.v[j * a.n_pad + k0 + c] = s_v[c];
    if (tile == 0 && tid < M) {
        const long long rix = (long long)tid * qq + j;
        a.lam[rix] = r_lam;
        a.zeta[rix] = r_zeta;
        a.h[rix] = r_h;
        a.p[rix] = r_p;
    }
    if (cons_warp && tile == 0 && lane < M) a.nu[(long long)lane * qq + j] = c_nu;
    if (blockIdx.x == 0 && tid == 0) {
        Ctrl& co = a.ctrl[it & 1];
        for (int l = 0; l < 4; ++l) {
            co.rho[l] = s_rho[l];
            co.f[l] = 1.0;
        }
        for (int i = 0; i < MAXM; ++i) co.x1[i] = i < M ? s_x1[i] : 0.0;
        co.r = l_r;
        co.sigma = l_sigma;
        co.nu_pending = 0;
        co.done = l_done;
        co.status = l_status;
        co.checks = l_checks;
        co.err = l_err;
        __threadfence();
        *(volatile long long*)a.iter = it;
    }
    cluster.sync();  // no CTA exits while a mate may still touch its shared memory
}

}  // namespace admm_dev
