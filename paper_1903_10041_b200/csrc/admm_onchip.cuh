// admm_onchip.cuh -- cluster-row persistent ADMM kernel: the on-chip engine
// for PHEV-sized problems (BASELINE.json configs[0], [1]; Appendix A,
// Eq. (6a)-(6i), residuals :464-479, adaptive rho :318-324).
//
// Scenario row j = one thread-block cluster of T CTAs (tile r holds steps
// [r*TC, r*TC + ncell)); coefficients, bounds, demand, x and v = s - mu stay
// in shared memory for the whole call.  Each bulk thread owns (usually) one
// cell, so the critical path of an iteration is one Gauss-Seidel cell + one
// block reduction + one cluster barrier + the scalar row update.
//
//  * capacity coupling (6b)/(6g)/(6d)/(6i): warp 0 of every CTA stores its
//    tile partials straight into every cluster-mate's shared memory (DSMEM),
//    one cluster.sync(), then every CTA of the row performs the identical row
//    update from the T partials (fixed order => identical values);
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
//    of t-3 = t+1 (mod 4);
//  * residual checks (every check_every): one counter barrier over all CTAs
//    (release add / acquire poll), after which every CTA reduces the same
//    published maxima and takes the same termination / rho decision.
#pragma once
#include <cooperative_groups.h>

#include "admm_kernels.cuh"

namespace admm_dev {

constexpr unsigned long long PUB_EMPTY = 0xFFF4DEADBEEF0001ull;  // sNaN payload: never computed
constexpr int PUB_BUFS = 4;
constexpr int ONCHIP_MAX_WARPS = 17;  // 16 bulk warps + 1 consensus warp
constexpr int ONCHIP_MAX_T = 16;      // tiles (CTAs) per cluster

#ifdef ADMM_PHASE_PROF  // development build only: per-phase clock64() totals of CTA 0
__device__ unsigned long long g_phase[2][8];
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
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(double* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

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
    int TC, T, G;
    double *pub;                // [PUB_BUFS][m][q] consensus contributions x_1 - nu (epoch slots)
    double *xraw;               // [2][m][q]        x_1^{(i,j)} by iteration parity (checks)
    double *rpart;              // [2][G][2]        per-CTA r1, s3 maxima (check parity)
    double *rowchk;             // [2][m][q][4]     row check terms r2, r3, s1, s2 (check parity)
    unsigned long long *cnt;    // [16] check-barrier arrivals (zeroed per launch)
};

// fill every publication slot with the sentinel (before each launch)
__global__ void pub_reset_kernel(double* pub, long long nslots) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nslots;
         t += (long long)gridDim.x * blockDim.x)
        pub[t] = __longlong_as_double((long long)PUB_EMPTY);
}

template <int M, int MODE>
__global__ void __launch_bounds__(ONCHIP_MAX_WARPS * 32) persist_cluster_kernel(KArgs a, CArgs p) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double sm[];
    const int TC = p.TC;
    double* s_a2 = sm;
    double* s_a1 = s_a2 + M * TC;
    double* s_b2 = s_a1 + M * TC;
    double* s_b1 = s_b2 + M * TC;
    double* s_lo = s_b1 + M * TC;
    double* s_hi = s_lo + M * TC;
    double* s_x = s_hi + M * TC;
    double* s_y = s_x + M * TC;
    double* s_v = s_y + TC;

    __shared__ double red[ONCHIP_MAX_WARPS][3 * M + 2];
    __shared__ double s_part[2][ONCHIP_MAX_T][3 * M];  // [parity][tile], written by mates (DSMEM)
    __shared__ double s_zl[M], s_x1[M], s_rho[4], s_f[4], s_t[2];
    __shared__ int s_flag[2];

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int nbw = nw - 1;  // bulk warps; warp nbw = consensus warp (active in tile 0 only)
    const int nbt = nbw * 32;
    const bool cons_warp = (wid == nbw);
    const int T = p.T;
    const long long j = blockIdx.x / T;
    const int tile = (int)cluster.block_rank();
    const int k0 = tile * TC;
    const int ncell = min(TC, a.n - k0);
    const long long qn = a.q * (long long)a.n_pad;
    const long long qq = a.q;
    const DParams& P = *a.prm;
    const double nd = (double)a.n;
    const double qtot = (double)a.q_total;
    const bool single = (a.q_total == 1);  // q = 1: x1 = own contribution, no exchange

    const long long it0 = *(volatile long long*)a.iter;
    const Ctrl& cin = a.ctrl[it0 & 1];
    if (cin.done || it0 >= P.iter_limit) return;  // uniform over the grid

    for (int t = tid; t < M * TC; t += blockDim.x) {
        const int i = t / TC, c = t - i * TC;
        const bool ok = c < ncell;
        const long long e = (long long)i * qn + j * a.n_pad + k0 + c;
        const long long bk = (long long)i * a.n_pad + k0 + c;
        s_a2[t] = ok ? a.a2[e] : 0.0;
        s_a1[t] = ok ? a.a1[e] : 0.0;
        s_b2[t] = ok ? a.b2[e] : 0.0;
        s_b1[t] = ok ? a.b1[e] : 0.0;
        s_lo[t] = ok ? a.lo[bk] : 0.0;
        s_hi[t] = ok ? a.hi[bk] : 0.0;
        s_x[t] = ok ? a.x[e] : 0.0;
    }
    for (int c = tid; c < TC; c += blockDim.x) {
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
    if (tid < 4) {
        s_rho[tid] = cin.rho[tid];
        s_f[tid] = 1.0;
    }
    double l_r = cin.r, l_sigma = cin.sigma;
    int l_status = cin.status, l_checks = cin.checks, l_err = cin.err, l_done = 0;
    const double iq = a.inv_q;
    const int ce = P.check_every;
    unsigned long long nchk = 0;
    bool x1_known = true;  // consensus warp: c_x1 holds x1 of the previous iteration
    __syncthreads();
    cluster.sync();  // mates' shared memory is live before any DSMEM store
#ifdef ADMM_PHASE_PROF
    const bool prof_on = blockIdx.x == 0 && (tid == 0 || tid == nbt);
    unsigned long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ph_last = clock64();
#endif

    const long long lim = P.iter_limit;
    int until_chk = ce > 0 ? (int)(ce - 1 - it0 % ce) : -1;  // iterations until the next check
    long long it = it0;
    for (; it < lim; ++it) {
        const int par = (int)(it & 1);
        const bool is_check = (until_chk == 0);
        until_chk = is_check ? ce - 1 : until_chk - 1;
        double rho[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) rho[l] = s_rho[l];
        double zl[M];
#pragma unroll
        for (int i = 0; i < M; ++i) zl[i] = s_zl[i];

        double Sg[M], dgx[M], dgn[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            Sg[i] = 0.0;
            dgx[i] = -INFINITY;
            dgn[i] = INFINITY;
        }
        double my_r1 = 0.0, my_s3 = 0.0;
        if (!cons_warp) {
            // ---- bulk cells: every cell of the tile except the consensus cell k = 0
            for (int cc = tid; cc < ncell; cc += nbt) {
                if (k0 + cc == 0) continue;
                double ca2[M], ca1[M], cb2[M], cb1[M], clo[M], chi[M], xo[M], xn[M], dummy[M];
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    ca2[i] = s_a2[i * TC + cc]; ca1[i] = s_a1[i * TC + cc];
                    cb2[i] = s_b2[i * TC + cc]; cb1[i] = s_b1[i * TC + cc];
                    clo[i] = s_lo[i * TC + cc]; chi[i] = s_hi[i * TC + cc];
                    xo[i] = s_x[i * TC + cc];
                    dummy[i] = 0.0;
                }
                const double vv = s_v[cc];
                const double yy = s_y[cc];
                gs_cell<M, MODE>(ca2, ca1, cb2, cb1, clo, chi, xo, xn, yy, fmax(vv, 0.0),
                                 vv < 0.0 ? -vv : 0.0, zl, rho, iq, false, dummy);
                s_v[cc] = cell_tail<M>(xo, xn, yy, vv, 1.0, is_check, my_r1, my_s3);
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    s_x[i * TC + cc] = xn[i];
                    Sg[i] += fma(cb2[i], xn[i], cb1[i]) * xn[i];
                    const double dg = (xn[i] - xo[i]) * fma(cb2[i], xn[i] + xo[i], cb1[i]);
                    dgx[i] = fmax(dgx[i], dg);
                    dgn[i] = fmin(dgn[i], dg);
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
                    read_consensus<M>(p.pub + (size_t)((it - 1) & (PUB_BUFS - 1)) * a.m * qq, qq, qtot, x1v);
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
            // reset this row's slots of the buffer iteration it+1 publishes into
            if (lane == 0)
#pragma unroll
                for (int i = 0; i < M; ++i)
                    st_relaxed_u64(p.pub + ((size_t)((it + 1) & (PUB_BUFS - 1)) * a.m + i) * qq + j, PUB_EMPTY);
            double x1nu[M], cnu[M];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                cnu[i] = __shfl_sync(0xffffffffu, c_nu, i);
                x1nu[i] = __shfl_sync(0xffffffffu, c_x1, i) + cnu[i];
            }
            double xk0[M];
            if (lane == 0) {
                double ca2[M], ca1[M], cb2[M], cb1[M], clo[M], chi[M], xo[M];
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    ca2[i] = s_a2[i * TC]; ca1[i] = s_a1[i * TC];
                    cb2[i] = s_b2[i * TC]; cb1[i] = s_b1[i * TC];
                    clo[i] = s_lo[i * TC]; chi[i] = s_hi[i * TC];
                    xo[i] = s_x[i * TC];
                }
                const double vv = s_v[0];
                const double yy = s_y[0];
                gs_cell<M, MODE>(ca2, ca1, cb2, cb1, clo, chi, xo, xk0, yy, fmax(vv, 0.0),
                                 vv < 0.0 ? -vv : 0.0, zl, rho, iq, true, x1nu);
                s_v[0] = cell_tail<M>(xo, xk0, yy, vv, 1.0, is_check, my_r1, my_s3);
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    s_x[i * TC] = xk0[i];
                    Sg[i] += fma(cb2[i], xk0[i], cb1[i]) * xk0[i];
                    const double dg = (xk0[i] - xo[i]) * fma(cb2[i], xk0[i] + xo[i], cb1[i]);
                    dgx[i] = fmax(dgx[i], dg);
                    dgn[i] = fmin(dgn[i], dg);
                }
                // x_1 for the check; (6c)'s contribution x_1 - nu (nu before (6h))
#pragma unroll
                for (int i = 0; i < M; ++i) __stcg(p.xraw + ((size_t)par * a.m + i) * qq + j, xk0[i]);
                if (!single || is_check) {  // q = 1: only the residual check reads it
                    fence_acq_rel_gpu();
#pragma unroll
                    for (int i = 0; i < M; ++i)
                        st_relaxed_u64(p.pub + ((size_t)(it & (PUB_BUFS - 1)) * a.m + i) * qq + j,
                                       (unsigned long long)__double_as_longlong(xk0[i] - cnu[i]));
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
        // ---- block reduction (fixed tree) of the tile partials
#pragma unroll
        for (int i = 0; i < M; ++i) {
            Sg[i] = warp_sum(Sg[i]);
            if (is_check) {
                dgx[i] = warp_max(dgx[i]);
                dgn[i] = warp_min(dgn[i]);
            }
        }
        if (is_check) {
            my_r1 = warp_max(my_r1);
            my_s3 = warp_max(my_s3);
        }
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                red[wid][3 * i] = Sg[i];
                red[wid][3 * i + 1] = dgx[i];
                red[wid][3 * i + 2] = dgn[i];
            }
            red[wid][3 * M] = my_r1;
            red[wid][3 * M + 1] = my_s3;
        }
        PHASE(1)
        __syncthreads();
        PHASE(2)
        double cta_r1 = 0.0, cta_s3 = 0.0;
        if (wid == 0) {
            double val[3 * M];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                val[3 * i] = warp_sum(lane < nw ? red[lane][3 * i] : 0.0);
                val[3 * i + 1] = is_check ? warp_max(lane < nw ? red[lane][3 * i + 1] : -INFINITY) : 0.0;
                val[3 * i + 2] = is_check ? warp_min(lane < nw ? red[lane][3 * i + 2] : INFINITY) : 0.0;
            }
            if (is_check) {
                cta_r1 = warp_max(lane < nw ? red[lane][3 * M] : 0.0);
                cta_s3 = warp_max(lane < nw ? red[lane][3 * M + 1] : 0.0);
            }
            if (lane < T) {  // DSMEM: this tile's partials into mate `lane`
                double* dst = cluster.map_shared_rank(&s_part[par][tile][0], lane);
#pragma unroll
                for (int v = 0; v < 3 * M; ++v) dst[v] = val[v];
            }
        }
        PHASE(3)
        cluster.sync();  // all T partials of row j are in every CTA's s_part[par]
        PHASE(4)

        // ---- row update (6b),(6g),(6d),(6i): identical in every CTA of the cluster
        if (tid < M) {
            double sg = 0.0, mx = -INFINITY, mn = INFINITY;
            for (int t = 0; t < T; ++t) {
                sg += s_part[par][t][3 * tid];
                mx = fmax(mx, s_part[par][t][3 * tid + 1]);
                mn = fmin(mn, s_part[par][t][3 * tid + 2]);
            }
            const RowOut o = row_update(sg, r_sb0, r_lam, r_p, r_h, r_zeta, r_c, nd, rho, mx, mn);
            r_lam = o.lam;
            r_zeta = o.zeta;
            r_h = o.h;
            r_p = o.p;
            r_r2 = o.r2;
            r_r3 = o.r3;
            r_s1 = o.s1;
            r_s2 = o.s2;
            s_zl[tid] = r_zeta + r_lam;
        }

        PHASE(5)
        if (is_check) {
            const int cpar = (int)(nchk & 1);
            if (tile == 0 && tid < M) {
                double* rc = p.rowchk + (((size_t)cpar * a.m + tid) * qq + j) * 4;
                __stcg(rc, r_r2);
                __stcg(rc + 1, r_r3);
                __stcg(rc + 2, r_s1);
                __stcg(rc + 3, r_s2);
            }
            if (tid == 0) {
                __stcg(p.rpart + ((size_t)cpar * p.G + blockIdx.x) * 2, cta_r1);
                __stcg(p.rpart + ((size_t)cpar * p.G + blockIdx.x) * 2 + 1, cta_s3);
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
                // x1 of this iteration (same reduction as the consensus warps) and the maxima
                double x1v[M], xmx[M], xmn[M];
                read_consensus<M>(p.pub + (size_t)(it & (PUB_BUFS - 1)) * a.m * qq, qq, qtot, x1v);
                const double* xr = p.xraw + (size_t)par * a.m * qq;
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    double mx = -INFINITY, mn = INFINITY;
                    for (long long jj = lane; jj < qq; jj += 32) {
                        const double x0 = __ldcg(xr + (size_t)i * qq + jj);
                        mx = fmax(mx, x0);
                        mn = fmin(mn, x0);
                    }
                    xmx[i] = warp_max(mx);
                    xmn[i] = warp_min(mn);
                }
                double t0 = 0.0, t6 = 0.0, t1 = 0.0, t2 = 0.0, t4 = 0.0, t5 = 0.0;
                for (int g = lane; g < p.G; g += 32) {
                    t0 = fmax(t0, __ldcg(p.rpart + ((size_t)cpar * p.G + g) * 2));
                    t6 = fmax(t6, __ldcg(p.rpart + ((size_t)cpar * p.G + g) * 2 + 1));
                }
                const long long R = (long long)a.m * qq;
                for (long long r = lane; r < R; r += 32) {
                    const double* rc = p.rowchk + ((size_t)cpar * R + r) * 4;
                    t1 = fmax(t1, __ldcg(rc));
                    t2 = fmax(t2, __ldcg(rc + 1));
                    t4 = fmax(t4, __ldcg(rc + 2));
                    t5 = fmax(t5, __ldcg(rc + 3));
                }
                t0 = warp_max(t0); t1 = warp_max(t1); t2 = warp_max(t2);
                t4 = warp_max(t4); t5 = warp_max(t5); t6 = warp_max(t6);
                if (lane == 0) {
                    double t3 = 0.0;
                    for (int i = 0; i < M; ++i) {
                        // max_j |x_1^{(i,j)} - x1| = max(max_j x_1 - x1, x1 - min_j x_1) exactly
                        t3 = fmax(t3, fmax(xmx[i] - x1v[i], x1v[i] - xmn[i]));
                        s_x1[i] = x1v[i];
                    }
                    double t[7] = {t0, t1, t2, t3, t4, t5, t6};
                    double rn[4], fl[4], r, sg, fac, s123[3];
                    const int conv = check_decide(P, rho, t, rn, fl, &r, &sg, &fac, s123);
                    if (blockIdx.x == 0 && a.hist && a.hist_cap > 0)
                        write_hist(a.hist + (size_t)(l_checks % a.hist_cap) * HCOLS, it + 1, r, sg,
                                   rho, t, s123, conv, fac);
                    for (int l = 0; l < 4; ++l) {
                        s_rho[l] = rn[l];
                        s_f[l] = fl[l];
                    }
                    s_t[0] = r;
                    s_t[1] = sg;
                    s_flag[0] = conv;
                    s_flag[1] = (!isfinite(r) || !isfinite(sg)) ? 1 : 0;
                }
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
        for (int k = 0; k < 8; ++k) g_phase[tid == 0 ? 0 : 1][k] = ph_acc[k];
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
    for (int t = tid; t < M * TC; t += blockDim.x) {
        const int i = t / TC, c = t - i * TC;
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
    cluster.sync();  // no CTA exits while a mate may still write its shared memory
}

}  // namespace admm_dev
