// admm_persist.cuh -- persistent, on-chip ADMM solver kernel for problems whose
// whole state fits in the shared memory of the co-resident CTAs (the PHEV
// config q=50, the toy, the horizon sweep up to n ~ 1e5).
//
// One cooperative launch runs every iteration of a solve/iterate call:
//   * CTA b owns one tile (scenario j, TC consecutive steps k) and keeps its
//     coefficients, bounds, demand, x and v = s - mu in shared memory for the
//     whole call (HBM is touched once at entry and once at exit);
//   * per iteration: the same per-cell math as the streaming sweep (gs_cell,
//     cell_tail), a block reduction of the row partials, ONE grid barrier, and
//     then every CTA computes the row update of its own row and the consensus
//     x1 (6c) redundantly from the published partials -- identical code and
//     inputs give identical values in every CTA, so no second barrier and no
//     "last CTA" serial step are needed;
//   * at a residual check a second barrier publishes the row-level residual
//     terms; every CTA reduces them and takes the same rho decision.
// Partial buffers are double-buffered by iteration parity: a CTA can be at
// most one barrier ahead of another.
#pragma once
#include <cooperative_groups.h>

#include "admm_kernels.cuh"

namespace admm_dev {

struct PArgs {
    int TC, T, G;
    double *gpart;   // [2][m][q][T][3]  tile partials: sum_k (b2 x^2 + b1 x), max/min dg
    double *cpart;   // [2][m][q][2]     consensus contribution x_1 - nu, and x_1
    double *rpart;   // [2][G][2]        per-CTA r1, s3 maxima
    double *rowchk;  // [2][m][q][4]     row check terms r2, r3, s1, s2
    unsigned *bar;   // [0] arrival count, [32] generation (separate 128-byte lines)
};

__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned G, unsigned& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == G - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicExch(bar + 32, g + 1u);
        } else {
            while (*(volatile unsigned*)(bar + 32) == g) {
            }
        }
        __threadfence();
    }
    gen += 1u;
    __syncthreads();
}

template <int M, int MODE>
__global__ void __launch_bounds__(512) persist_kernel(KArgs a, PArgs p) {
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

    __shared__ double red[16][3 * M + 2];
    __shared__ double rowres[3 * M];
    __shared__ double s_zl[M], s_x1nu[M], s_x1[M], s_x0mx[M], s_x0mn[M];
    __shared__ double s_rho[4], s_f[4], s_t[7];
    __shared__ int s_flag[2];  // [0] conv, [1] rho changed / error bits

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int T = p.T;
    const long long j = blockIdx.x / T;
    const int tile = blockIdx.x - (int)j * T;
    const int k0 = tile * TC;
    const int ncell = min(TC, a.n - k0);
    const long long qn = a.q * (long long)a.n_pad;
    const DParams& P = *a.prm;
    const double nd = a.nd;

    const long long it0 = *(volatile long long*)a.iter;
    const Ctrl& cin = a.ctrl[it0 & 1];
    if (cin.done || it0 >= P.iter_limit) return;
    unsigned gen = *(volatile unsigned*)(p.bar + 32);

    // ---- load the tile (coalesced); apply the pending rescale of mu to v
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
    // row scalars of source i live in thread i (< M), as effective values
    double r_lam = 0.0, r_p = 0.0, r_h = 0.0, r_zeta = 0.0, r_nu = 0.0, r_c = 0.0, r_sb0 = 0.0;
    double r_r2 = 0.0, r_r3 = 0.0, r_s1 = 0.0, r_s2 = 0.0;
    if (tid < M) {
        const long long rix = (long long)tid * a.q + j;
        r_lam = a.lam[rix] * cin.f[0];
        r_p = a.p[rix] * cin.f[1];
        r_h = a.h[rix];
        r_zeta = a.zeta[rix];
        r_c = a.c[tid];
        r_sb0 = a.sb0[rix];
        if (tile == 0) {
            double nu = a.nu[rix];
            if (cin.nu_pending) nu = nu + cin.x1[tid] - a.x[(long long)tid * qn + j * a.n_pad];
            r_nu = nu * cin.f[3];
        }
        s_zl[tid] = r_zeta + r_lam;
        s_x1[tid] = cin.x1[tid];
        s_x1nu[tid] = cin.x1[tid] + r_nu;
    }
    if (tid < 4) {
        s_rho[tid] = cin.rho[tid];
        s_f[tid] = 1.0;
    }
    double l_r = cin.r, l_sigma = cin.sigma;
    int l_status = cin.status, l_checks = cin.checks, l_err = cin.err, l_done = 0;
    const double iq = a.inv_q;
    const int ce = P.check_every;
    __syncthreads();

    long long it = it0;
    for (; it < P.iter_limit; ++it) {
        const int par = (int)(it & 1);
        const bool is_check = ce > 0 && ((it + 1) % ce) == 0;
        double rho[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) rho[l] = s_rho[l];
        double zl[M], x1nu[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            zl[i] = s_zl[i];
            x1nu[i] = s_x1nu[i];
        }
        // ---- (6a) + (6e)/(6f) on this thread's 2 cells
        double Sg[M], dgx[M], dgn[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            Sg[i] = 0.0;
            dgx[i] = -INFINITY;
            dgn[i] = INFINITY;
        }
        double my_r1 = 0.0, my_s3 = 0.0;
        const int cl = CPT * tid;
        if (cl < TC) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int cc = cl + c;
                const bool valid = cc < ncell;
                double ca2[M], ca1[M], cb2[M], cb1[M], clo[M], chi[M], xo[M], xn[M];
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    ca2[i] = s_a2[i * TC + cc]; ca1[i] = s_a1[i * TC + cc];
                    cb2[i] = s_b2[i * TC + cc]; cb1[i] = s_b1[i * TC + cc];
                    clo[i] = s_lo[i * TC + cc]; chi[i] = s_hi[i * TC + cc];
                    xo[i] = s_x[i * TC + cc];
                }
                const double vv = s_v[cc];
                const double yy = s_y[cc];
                gs_cell<M, MODE>(ca2, ca1, cb2, cb1, clo, chi, xo, xn, yy, fmax(vv, 0.0),
                                 vv < 0.0 ? -vv : 0.0, zl, rho, iq, k0 + cc == 0, x1nu);
                const double vnew = cell_tail<M>(xo, xn, yy, vv, 1.0, is_check && valid, my_r1, my_s3);
                if (valid) {
                    s_v[cc] = vnew;
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        s_x[i * TC + cc] = xn[i];
                        Sg[i] += fma(cb2[i], xn[i], cb1[i]) * xn[i];
                        const double dg = (xn[i] - xo[i]) * fma(cb2[i], xn[i] + xo[i], cb1[i]);
                        dgx[i] = fmax(dgx[i], dg);
                        dgn[i] = fmin(dgn[i], dg);
                    }
                }
            }
        }
        // ---- block reduction (fixed tree) of the row partials
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
        __syncthreads();
        if (wid == 0) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                double s = lane < nw ? red[lane][3 * i] : 0.0;
                double mx = lane < nw ? red[lane][3 * i + 1] : -INFINITY;
                double mn = lane < nw ? red[lane][3 * i + 2] : INFINITY;
                s = warp_sum(s);
                mx = warp_max(mx);
                mn = warp_min(mn);
                if (lane == 0) {
                    double* gp = p.gpart + ((((long long)par * a.m + i) * a.q + j) * T + tile) * 3;
                    __stcg(gp, s);
                    __stcg(gp + 1, mx);
                    __stcg(gp + 2, mn);
                }
            }
            if (is_check) {
                double r1 = lane < nw ? red[lane][3 * M] : 0.0;
                double s3 = lane < nw ? red[lane][3 * M + 1] : 0.0;
                r1 = warp_max(r1);
                s3 = warp_max(s3);
                if (lane == 0) {
                    __stcg(p.rpart + ((long long)par * p.G + blockIdx.x) * 2, r1);
                    __stcg(p.rpart + ((long long)par * p.G + blockIdx.x) * 2 + 1, s3);
                }
            }
        }
        if (tile == 0 && tid < M) {
            const double x0 = s_x[tid * TC];
            double* cp = p.cpart + (((long long)par * a.m + tid) * a.q + j) * 2;
            __stcg(cp, x0 - r_nu);  // (6c) contribution with nu before (6h)
            __stcg(cp + 1, x0);
        }
        grid_sync(p.bar, p.G, gen);

        // ---- row update of own row (6b),(6g),(6d),(6i), identical in every tile CTA
        // tile partials: lane-strided loads (all in flight at once), fixed-order
        // per-lane sums, then a butterfly -- identical in every CTA of the row
        double row_sg = 0.0, row_mx = -INFINITY, row_mn = INFINITY;
        if (wid == 0) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const double* gp = p.gpart + (((long long)par * a.m + i) * a.q + j) * T * 3;
                double sg = 0.0, mx = -INFINITY, mn = INFINITY;
                for (int t = lane; t < T; t += 32) {
                    sg += __ldcg(gp + 3 * t);
                    mx = fmax(mx, __ldcg(gp + 3 * t + 1));
                    mn = fmin(mn, __ldcg(gp + 3 * t + 2));
                }
                sg = warp_sum(sg);
                mx = warp_max(mx);
                mn = warp_min(mn);
                if (lane == i) {
                    row_sg = sg;
                    row_mx = mx;
                    row_mn = mn;
                }
            }
        }
        if (tid < M) {
            const RowOut o = row_update(row_sg, r_sb0, r_lam, r_p, r_h, r_zeta, r_c, nd, rho, row_mx,
                                        row_mn);
            r_lam = o.lam;
            r_zeta = o.zeta;
            r_h = o.h;
            r_p = o.p;
            r_r2 = o.r2;
            r_r3 = o.r3;
            r_s1 = o.s1;
            r_s2 = o.s2;
        }
        // ---- (6c) consensus x1 = (1/q) sum_j (x_1 - nu), same fixed order in every CTA
        if (wid == 0) {
            for (int i = 0; i < M; ++i) {
                const double* cp = p.cpart + ((long long)par * a.m + i) * a.q * 2;
                double s = 0.0, mx = -INFINITY, mn = INFINITY;
                for (long long jj = lane; jj < a.q; jj += 32) {
                    s += __ldcg(cp + 2 * jj);
                    if (is_check) {
                        const double x0 = __ldcg(cp + 2 * jj + 1);
                        mx = fmax(mx, x0);
                        mn = fmin(mn, x0);
                    }
                }
                s = warp_sum(s);
                if (is_check) {
                    mx = warp_max(mx);
                    mn = warp_min(mn);
                }
                if (lane == 0) {
                    s_x1[i] = s / (double)a.q_total;
                    s_x0mx[i] = mx;
                    s_x0mn[i] = mn;
                }
            }
        }
        __syncthreads();
        // (6h) nu += x1 - x_1^{(i,j)}  (tile 0 holds nu)
        if (tid < M && tile == 0) r_nu = r_nu + s_x1[tid] - s_x[tid * TC];

        if (is_check) {
            if (tid < M && tile == 0) {
                double* rc = p.rowchk + (((long long)par * a.m + tid) * a.q + j) * 4;
                __stcg(rc, r_r2);
                __stcg(rc + 1, r_r3);
                __stcg(rc + 2, r_s1);
                __stcg(rc + 3, r_s2);
            }
            grid_sync(p.bar, p.G, gen);
            // every CTA: the same maxima (max is order independent)
            if (wid == 0) {
                double t0 = 0.0, t6 = 0.0, t1 = 0.0, t2 = 0.0, t4 = 0.0, t5 = 0.0;
                for (int g = lane; g < p.G; g += 32) {
                    t0 = fmax(t0, __ldcg(p.rpart + ((long long)par * p.G + g) * 2));
                    t6 = fmax(t6, __ldcg(p.rpart + ((long long)par * p.G + g) * 2 + 1));
                }
                const long long R = (long long)a.m * a.q;
                for (long long r = lane; r < R; r += 32) {
                    const double* rc = p.rowchk + ((long long)par * R + r) * 4;
                    t1 = fmax(t1, __ldcg(rc));
                    t2 = fmax(t2, __ldcg(rc + 1));
                    t4 = fmax(t4, __ldcg(rc + 2));
                    t5 = fmax(t5, __ldcg(rc + 3));
                }
                t0 = warp_max(t0); t1 = warp_max(t1); t2 = warp_max(t2);
                t4 = warp_max(t4); t5 = warp_max(t5); t6 = warp_max(t6);
                if (lane == 0) {
                    double t3 = 0.0;
                    for (int i = 0; i < M; ++i)
                        t3 = fmax(t3, fmax(s_x0mx[i] - s_x1[i], s_x1[i] - s_x0mn[i]));
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
            // dual rescale (reading G11): lam<->rho1, p<->rho2, mu<->rho3, nu<->rho4
            if (s_f[0] != 1.0 || s_f[1] != 1.0 || s_f[2] != 1.0 || s_f[3] != 1.0) {
                if (tid < M) {
                    r_lam *= s_f[0];
                    r_p *= s_f[1];
                    r_nu *= s_f[3];
                }
                const double f2 = s_f[2];
                for (int c = tid; c < ncell; c += blockDim.x)
                    if (s_v[c] < 0.0) s_v[c] *= f2;
            }
            if (l_err || (l_status && P.stop_on_conv)) l_done = 1;
        }
        if (tid < M) {
            s_zl[tid] = r_zeta + r_lam;
            s_x1nu[tid] = s_x1[tid] + r_nu;
        }
        __syncthreads();
        if (tid < 4) s_f[tid] = 1.0;
        if (l_done) {
            ++it;
            break;
        }
    }

    // ---- write back (effective state: nothing pending)
    for (int t = tid; t < M * TC; t += blockDim.x) {
        const int i = t / TC, c = t - i * TC;
        if (c < ncell) a.x[(long long)i * qn + j * a.n_pad + k0 + c] = s_x[t];
    }
    for (int c = tid; c < ncell; c += blockDim.x) a.v[j * a.n_pad + k0 + c] = s_v[c];
    if (tile == 0 && tid < M) {
        const long long rix = (long long)tid * a.q + j;
        a.lam[rix] = r_lam;
        a.zeta[rix] = r_zeta;
        a.h[rix] = r_h;
        a.p[rix] = r_p;
        a.nu[rix] = r_nu;
    }
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
}





}  // namespace admm_dev
