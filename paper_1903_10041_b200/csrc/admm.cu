// admm.cu -- libadmm_b200.so: host runtime behind include/admm.h plus the
// non-hot kernels (validation, initialisation, objective, state transfer)
// and the quartic microbench kernel.  Hot path: admm_kernels.cuh.
//
// Execution model:
//   * one CUDA graph per context: a conditional WHILE node whose body is
//     check_every sweep launches; the last CTA of each sweep sets the
//     condition (not done and iteration limit not reached), so a whole solve
//     runs with zero host round trips;
//   * multi-GPU (an admm_dist given, any world size): the body is check_every x
//     [sweep -> ncclAllGather(per-rank aggregates, 32 doubles) -> finalize_kernel]
//     (scenario sharding) or [sweep -> ncclAllReduce(row sums, dg extrema) ->
//     ncclAllGather -> hz_rows_kernel] (horizon blocks), driven by a host loop
//     that polls the done flag once per body.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "admm.h"
#include "admm_kernels.cuh"
#include "admm_persist.cuh"
#include "admm_onchip.cuh"
#include "admm_sweep2.cuh"
#include "admm_onchip2.cuh"

namespace admm_dev {
const void* cluster2_pick(int m, int mode);  // onchip2.cu
}

using namespace admm_dev;

namespace {

constexpr int HIST_CAP = 8192;
constexpr int MAX_WORLD = 64;

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Layout {
    size_t a2, a1, a0, b2, b1, b0, lo, hi, y, c, sb0, x, v, lam, zeta, h, p, nu, cta_part,
        row_part, obj_rows, xsend, xall, hist, row_cnt, glob_cnt, ctrl, iter, prm, vflag, pg, pc, pr,
        prc, pbar, pub, pub2, chkv2, chkx2, cnt2, xraw, bq, ib2s, chk, gbound, rowacc, rowdg, rowcnt, cf, hzdg, hzrow, total;
};

// streaming sweep block size: 2 cells per thread, at most ADMM_SWEEP_BS (default
// 512: one row per item; 256 splits rows over two CTAs and measured 30 % vs 44 %)
// cpt = cells per thread (2, or 4 with 256-thread CTAs: same 1024-cell tile)
int pick_bs(long long n, int cpt = CPT) {
    long long cap = cpt == 4 ? 256 : 512;
    if (const char* e = getenv("ADMM_SWEEP_BS")) cap = std::max(32LL, std::min(cap, atoll(e)));
    long long need = (n + cpt - 1) / cpt;
    long long bs = ((need + 31) / 32) * 32;
    return (int)std::max(32LL, std::min(cap, bs));
}

constexpr size_t ONCHIP_PREP_MAX_ELEMS = (size_t)1 << 23;  // m*q*n_pad of the largest on-chip problem

Layout make_layout(int m, long long n, long long q, int sms) {
    Layout L{};
    const long long n_pad = align_up((size_t)n, 4);
    const int bs = pick_bs(n);
    const long long tile = (long long)bs * CPT;
    const long long T = (n + tile - 1) / tile;
    const size_t E = (size_t)m * q * n_pad * 8, Cc = (size_t)q * n_pad * 8, R = (size_t)m * q * 8;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t r = o;
        o = align_up(o + std::max<size_t>(bytes, 8), 256);
        return r;
    };
    // a2, a1, b2, b1 at one stride (the TMA sweep fetches the four with one 4-D tensor
    // copy), lo/hi and y/v adjacent likewise
    L.a2 = take(E); L.a1 = take(E); L.b2 = take(E); L.b1 = take(E); L.a0 = take(E); L.b0 = take(E);
    L.lo = take((size_t)m * n_pad * 8); L.hi = take((size_t)m * n_pad * 8);
    L.y = take(Cc); L.v = take(Cc); L.c = take((size_t)m * 8); L.sb0 = take(R);
    L.x = take(E);
    L.lam = take(R); L.zeta = take(R); L.h = take(R); L.p = take(R); L.nu = take(R);
    L.cta_part = take((size_t)32 * sms * XB * 8);
    L.row_part = take(T > 1 ? (size_t)m * q * T * 3 * 8 : 8);
    L.obj_rows = take(R);
    L.xsend = take(XB * 8); L.xall = take((size_t)MAX_WORLD * XB * 8);
    L.hist = take((size_t)HIST_CAP * HCOLS * 8);
    L.row_cnt = take((size_t)q * 4); L.glob_cnt = take(4);
    L.ctrl = take(2 * sizeof(Ctrl)); L.iter = take(8); L.prm = take(sizeof(DParams));
    L.vflag = take(8);
    // persistent-kernel scratch (used only when q*T <= 32*sms CTAs)
    const size_t GP = (size_t)32 * sms;
    L.pg = take(2 * (size_t)m * GP * 3 * 8);
    L.pc = take(2 * (size_t)m * std::min<size_t>(q, GP) * 2 * 8);
    L.pr = take(2 * GP * 2 * 8);
    L.prc = take(2 * (size_t)m * std::min<size_t>(q, GP) * 4 * 8);
    L.pbar = take(64 * 4);
    L.pub = take((size_t)PUB_BUFS * m * std::min<size_t>(q, GP) * 8);
    // message-passing cluster engine: LL publication buffers (16 B per value)
    L.pub2 = take((size_t)OC2_BUFS * m * std::min<size_t>(q, GP) * 16);
    L.chkv2 = take((size_t)OC2_BUFS * OC2_CHKV * std::min<size_t>(q, GP) * 16);
    L.chkx2 = take((size_t)OC2_BUFS * m * std::min<size_t>(q, GP) * 16);
    L.cnt2 = take(16);
    L.xraw = take(2 * (size_t)m * std::min<size_t>(q, GP) * 8);
    // prepared constants for the on-chip engine (only for problems that can be on chip)
    const bool onchip_sized = (size_t)m * q * n_pad <= ONCHIP_PREP_MAX_ELEMS;
    L.bq = take(onchip_sized ? E : 8);
    L.ib2s = take(onchip_sized ? E : 8);
    L.chk = take(3 * CHK_SLOTS * 8);
    L.gbound = take(MAXM * 8);
    L.rowacc = take((size_t)q * MAXM * 8);
    L.rowdg = take((size_t)q * 2 * MAXM * 8);
    L.rowcnt = take((size_t)q * MAXM * 4);
    L.cf = take(2 * E);  // F2: fp32 a2, a1, b2, b1 [4][m][q][n_pad] (16 B per element)
    L.hzdg = take((size_t)q * 2 * MAXM * 8);  // horizon blocks: dg extrema keys per row
    L.hzrow = take((size_t)2 * m * q * 8);     // initial row sums (all-reduced over horizon blocks)
    L.total = o;
    return L;
}

// lo/hi of row rix = i*q + j at step k
__device__ __forceinline__ double lo_of(const KArgs& a, long long rix, long long k) {
    return a.lo[(rix / a.q) * a.n_pad + k];
}
__device__ __forceinline__ double hi_of(const KArgs& a, long long rix, long long k) {
    return a.hi[(rix / a.q) * a.n_pad + k];
}

// ------------------------------------------------------------ small kernels
__global__ void validate_kernel(int m, long long q, long long n, long long n_pad,
                                const double* a2, const double* a1, const double* a0,
                                const double* b2, const double* b1, const double* b0,
                                const double* lo, const double* hi, const double* y,
                                const double* c, unsigned long long* flag) {
    // code = kind << 56 | linear index; the smallest code is reported
    const long long NE = (long long)m * q * n;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NE; t += stride) {
        const long long k = t % n, ij = t / n;
        const long long e = ij * n_pad + k;
        unsigned long long code = ~0ull;
        if (!(isfinite(a2[e]) && isfinite(a1[e]) && isfinite(a0[e]) && isfinite(b2[e]) &&
              isfinite(b1[e]) && isfinite(b0[e])))
            code = (1ull << 56) | (unsigned long long)t;
        else if (a2[e] < 0.0) code = (2ull << 56) | (unsigned long long)t;
        else if (b2[e] < 0.0) code = (3ull << 56) | (unsigned long long)t;
        if (code != ~0ull) atomicMin(flag, code);
    }
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * n;
         t += stride) {
        const long long i = t / n, k = t % n;
        const double l = lo[i * n_pad + k], h = hi[i * n_pad + k];
        if (!(l <= h) || isnan(l) || isnan(h)) atomicMin(flag, (4ull << 56) | (unsigned long long)t);
    }
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < q * n; t += stride) {
        const long long j = t / n, k = t % n;
        if (!isfinite(y[j * n_pad + k])) atomicMin(flag, (5ull << 56) | (unsigned long long)t);
    }
    if (blockIdx.x == 0 && threadIdx.x < m && isnan(c[threadIdx.x]))
        atomicMin(flag, (6ull << 56) | (unsigned long long)threadIdx.x);
}

// per source i: max over (j,k) of |b2 x^2 + b1 x| over the box (x in [lo, hi]),
// as order-preserving keys (fixed-point scale of the on-chip row sums)
__global__ void gbound_kernel(int m, long long q, long long n, long long n_pad, const double* b2,
                              const double* b1, const double* lo, const double* hi,
                              unsigned long long* out) {
    const long long NE = (long long)m * q * n;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t0 = blockIdx.x * (long long)blockDim.x; t0 < NE; t0 += stride) {
        const long long t = t0 + threadIdx.x;
        double g = 0.0;
        int i = (int)(t0 / (q * n));
        if (t < NE) {
            const long long k = t % n, ij = t / n;
            i = (int)(ij / q);
            const long long e = ij * n_pad + k;
            const double X = fmax(fabs(lo[i * n_pad + k]), fabs(hi[i * n_pad + k]));
            g = fma(b2[e] * X, X, fabs(b1[e]) * X);
            if (isnan(g)) g = INFINITY;
        }
        // warps are source-uniform except at source boundaries: per-lane atomics there
        const int i0 = __shfl_sync(0xffffffffu, i, 0);
        if (__all_sync(0xffffffffu, i == i0)) {
            g = warp_max(g);
            if ((threadIdx.x & 31) == 0) atomicMax(out + i0, okey(g));
        } else if (t < NE) {
            atomicMax(out + i, okey(g));
        }
    }
}

// row dg extrema accumulators of the streaming engine: identities (max 0, min ~0)
__global__ void rowdg_init_kernel(unsigned long long* rowdg, long long q) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < q * 2 * MAXM;
         t += (long long)gridDim.x * blockDim.x)
        rowdg[t] = (t % (2 * MAXM)) >= MAXM ? ~0ull : 0ull;
}

// init (reading G19): x = clamp(midpoint) or clamp(0); v = s = max(0, sum_i x - y)
__global__ void init_cells_kernel(KArgs a) {
    const long long N = a.q * (long long)a.n_pad;
    const long long qn = a.q * (long long)a.n_pad;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N;
         t += (long long)gridDim.x * blockDim.x) {
        const long long j = t / a.n_pad, k = t % a.n_pad;
        if (k >= a.n) {
            a.v[t] = 0.0;
            for (int i = 0; i < a.m; ++i) a.x[i * qn + t] = 0.0;
            continue;
        }
        double sx = 0.0;
        for (int i = 0; i < a.m; ++i) {
            const double l = a.lo[i * a.n_pad + k], h = a.hi[i * a.n_pad + k];
            const double mid = (isfinite(l) && isfinite(h)) ? 0.5 * (l + h) : 0.0;
            const double xv = clampd(mid, l, h);
            a.x[i * qn + t] = xv;
            sx += xv;
        }
        a.v[t] = fmax(0.0, sx - a.y[j * a.n_pad + k]);
    }
    (void)0;
}

// block-wide fixed-order sum (blockDim.x == 256)
__device__ double block_sum_256(double v, double* sh) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = threadIdx.x < 8 ? sh[threadIdx.x] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;  // valid in threads < 32
}

// per row (i,j): this rank's sum_k g(x) and sum_k b0 (all-reduced over horizon blocks),
// then sb0 = sum_k b0; h = min(c, sum_k g(x)); lam = zeta = p = nu = 0
__global__ void __launch_bounds__(256) init_rows_kernel(KArgs a, double* rs) {
    __shared__ double sh[8];
    const long long rix = blockIdx.x;  // i * q + j
    const int i = (int)(rix / a.q);
    const double* b2 = a.b2 + rix * a.n_pad;
    const double* b1 = a.b1 + rix * a.n_pad;
    const double* b0 = a.b0 + rix * a.n_pad;
    const double* x = a.x + rix * a.n_pad;
    double sg = 0.0, s0 = 0.0;
    for (long long k = threadIdx.x; k < a.n; k += 256) {
        const double xv = x[k];
        sg += b2[k] * xv * xv + b1[k] * xv + b0[k];
        s0 += b0[k];
    }
    sg = block_sum_256(sg, sh);
    s0 = block_sum_256(s0, sh);
    if (threadIdx.x == 0) {
        rs[rix] = sg;
        rs[(long long)a.m * a.q + rix] = s0;
    }
    (void)i;
}

__global__ void init_rows_fin_kernel(KArgs a, const double* rs) {
    const long long R = (long long)a.m * a.q;
    for (long long rix = blockIdx.x * (long long)blockDim.x + threadIdx.x; rix < R;
         rix += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(rix / a.q);
        ((double*)a.sb0)[rix] = rs[R + rix];
        a.h[rix] = fmin(a.c[i], rs[rix]);
        a.lam[rix] = 0.0;
        a.zeta[rix] = 0.0;
        a.p[rix] = 0.0;
        a.nu[rix] = 0.0;
    }
}

// consensus partial sums sum_j x_1^{(i,j)} - nu (fixed order) -> xsend; zero on a rank
// without the k = 1 cell (horizon blocks)
__global__ void cons_partial_kernel(KArgs a, int with_nu) {
    if (threadIdx.x >= 32) return;
    for (int i = 0; i < a.m; ++i) {
        double s = 0.0;
        for (long long j = threadIdx.x; a.k0own && j < a.q; j += 32) {
            const long long rix = (long long)i * a.q + j;
            s += a.x[rix * a.n_pad] - (with_nu ? a.nu[rix] : 0.0);
        }
        s = warp_sum(s);
        if (threadIdx.x == 0) a.xsend[i] = s;
    }
}

__global__ void init_ctrl_kernel(KArgs a, const double* agg, int world, double r0, double r1,
                                 double r2, double r3) {
    if (threadIdx.x != 0) return;
    Ctrl& c = a.ctrl[0];
    const double rr[4] = {r0, r1, r2, r3};
    for (int l = 0; l < 4; ++l) {
        c.rho[l] = rr[l];
        c.f[l] = 1.0;
    }
    for (int i = 0; i < MAXM; ++i) {
        double s = 0.0;
        if (i < a.m)
            for (int r = 0; r < world; ++r) s += agg[r * XB + i];
        c.x1[i] = i < a.m ? s / (double)a.q_total : 0.0;
    }
    c.r = NAN;
    c.sigma = NAN;
    c.nu_pending = 0;
    c.done = 0;
    c.status = 0;
    c.checks = 0;
    c.err = 0;
    a.ctrl[1] = c;
    *a.iter = 0;
    *a.glob_cnt = 0;
}

// objective rows: sum_k f(x) per (i,j), fixed order
__global__ void __launch_bounds__(256) obj_rows_kernel(KArgs a, double* out) {
    __shared__ double sh[8];
    const long long rix = blockIdx.x;
    const double* a2 = a.a2 + rix * a.n_pad;
    const double* a1 = a.a1 + rix * a.n_pad;
    const double* a0 = a.a0 + rix * a.n_pad;
    const double* x = a.x + rix * a.n_pad;
    double s = 0.0;
    for (long long k = threadIdx.x; k < a.n; k += 256) {
        const double xv = x[k];
        s += a2[k] * xv * xv + a1[k] * xv + a0[k];
    }
    s = block_sum_256(s, sh);
    if (threadIdx.x == 0) out[rix] = s;
}

__global__ void obj_sum_kernel(long long R, const double* rows, double* out) {
    if (threadIdx.x >= 32) return;
    double s = 0.0;
    for (long long r = threadIdx.x; r < R; r += 32) s += rows[r];
    s = warp_sum(s);
    if (threadIdx.x == 0) out[0] = s;
}

// effective (materialised) state -> dense caller layout
__global__ void materialize_kernel(KArgs a, double* x, double* z, double* lam, double* s,
                                   double* mu, double* h, double* p, double* nu, double* x1) {
    const long long it = *a.iter;
    const Ctrl& cin = a.ctrl[it & 1];
    const long long n = a.n, q = a.q;
    const long long NE = (long long)a.m * q * n;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (long long t = t0; t < NE; t += stride) {
        const long long k = t % n, rix = t / n;
        const long long e = rix * a.n_pad + k;
        const double xv = a.x[e];
        if (x) x[t] = xv;
        if (z) z[t] = a.b2[e] * xv * xv + a.b1[e] * xv + a.b0[e] + a.zeta[rix];
        if (lam) lam[t] = a.lam[rix] * cin.f[0];
    }
    for (long long t = t0; t < q * n; t += stride) {
        const long long k = t % n, j = t / n;
        const double vv = a.v[j * a.n_pad + k];
        if (s) s[t] = fmax(vv, 0.0);
        if (mu) mu[t] = vv < 0.0 ? -vv * cin.f[2] : 0.0;
    }
    for (long long t = t0; t < (long long)a.m * q; t += stride) {
        const int i = (int)(t / q);
        if (h) h[t] = a.h[t];
        if (p) p[t] = a.p[t] * cin.f[1];
        if (nu) {
            double v = a.nu[t];
            if (cin.nu_pending) v = v + cin.x1[i] - a.x[t * a.n_pad];
            nu[t] = v * cin.f[3];
        }
    }
    if (x1 && t0 < a.m) x1[t0] = cin.x1[t0];
}

// warm start: literal arrays -> reduced representation (identities I1, I2)
__global__ void compress_kernel(KArgs a, const double* x, const double* z, const double* lam,
                                const double* s, const double* mu, const double* h,
                                const double* p, const double* nu, unsigned long long* flag) {
    const long long n = a.n, q = a.q;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long NE = (long long)a.m * q * n;
    for (long long t = t0; t < NE; t += stride) {
        const long long k = t % n, rix = t / n;
        const long long e = rix * a.n_pad + k;
        a.x[e] = x[t];
        const double l0 = lam[rix * n];
        const double g0 = a.b2[rix * a.n_pad] * x[rix * n] * x[rix * n] +
                          a.b1[rix * a.n_pad] * x[rix * n] + a.b0[rix * a.n_pad];
        const double ze0 = z[rix * n] - g0;
        const double gk = a.b2[e] * x[t] * x[t] + a.b1[e] * x[t] + a.b0[e];
        const double zek = z[t] - gk;
        if (fabs(lam[t] - l0) > 1e-12 * (1.0 + fabs(l0)))
            atomicMin(flag, (1ull << 56) | (unsigned long long)t);
        if (fabs(zek - ze0) > 1e-12 * (1.0 + fabs(z[t]) + fabs(gk)))
            atomicMin(flag, (2ull << 56) | (unsigned long long)t);
        const double l = lo_of(a, rix, k), hh = hi_of(a, rix, k);
        if (!(x[t] >= l && x[t] <= hh)) atomicMin(flag, (4ull << 56) | (unsigned long long)t);
        if (k == 0) {
            a.lam[rix] = l0;
            a.zeta[rix] = ze0;
        }
    }
    for (long long t = t0; t < q * n; t += stride) {
        const long long k = t % n, j = t / n;
        const double sv = s[t], mv = mu[t];
        if (sv < 0.0 || mv < 0.0 || fmin(sv, mv) > 1e-12 * (1.0 + fmax(sv, mv)))
            atomicMin(flag, (3ull << 56) | (unsigned long long)t);
        a.v[j * a.n_pad + k] = sv - mv;
    }
    for (long long t = t0; t < (long long)a.m * q; t += stride) {
        a.h[t] = h[t];
        a.p[t] = p[t];
        a.nu[t] = nu[t];
    }
}

__global__ void set_ctrl_kernel(KArgs a, const double* x1) {
    if (threadIdx.x != 0) return;
    const long long it = *a.iter;
    Ctrl& c = a.ctrl[it & 1];
    for (int l = 0; l < 4; ++l) c.f[l] = 1.0;
    for (int i = 0; i < a.m; ++i) c.x1[i] = x1[i];
    c.nu_pending = 0;
    c.done = 0;
}

__global__ void clear_done_kernel(KArgs a) {
    if (threadIdx.x != 0) return;
    const long long it = *a.iter;
    a.ctrl[it & 1].done = 0;
}

// ---------------------------------------------------------- microbench
template <int MODE>
__device__ __forceinline__ void qb_vec_body(const double* A, const double* B, const double* C, const double* D,
                                            const double* lo, const double* hi, double* x, long long N2) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N2; t += stride) {
        const double2 a = __ldcs(reinterpret_cast<const double2*>(A) + t);
        const double2 b = __ldcs(reinterpret_cast<const double2*>(B) + t);
        const double2 c = __ldcs(reinterpret_cast<const double2*>(C) + t);
        const double2 d = __ldcs(reinterpret_cast<const double2*>(D) + t);
        double2 l = make_double2(-INFINITY, -INFINITY), h = make_double2(INFINITY, INFINITY);
        if (lo) l = __ldcs(reinterpret_cast<const double2*>(lo) + t);
        if (hi) h = __ldcs(reinterpret_cast<const double2*>(hi) + t);
        double2 r;
        r.x = quartic_boxmin<MODE>(a.x, b.x, c.x, d.x, l.x, h.x);
        r.y = quartic_boxmin<MODE>(a.y, b.y, c.y, d.y, l.y, h.y);
        __stcs(reinterpret_cast<double2*>(x) + t, r);
    }
}

// flag (the sampled dispatch): run only when *flag == 0
template <int MODE>
__global__ void __launch_bounds__(256) quartic_batch_vec_kernel(const double* A, const double* B,
                                                                const double* C, const double* D,
                                                                const double* lo, const double* hi,
                                                                double* x, long long N2,
                                                                const int* flag = nullptr) {
    if (flag && *flag != 0) return;  // the warp-compacted kernel takes this batch
    qb_vec_body<MODE>(A, B, C, D, lo, hi, x, N2);
}

// Warp-compacted variant for mixed trigonometric / Cardano batches (PAPER.md:143-161:
// the two branches of Algorithm 1 have similar cost, so a warp whose lanes split between
// them pays both).  Each warp streams tiles of 64 quartics (a double2 per lane per
// stream), normalises and classifies both of each lane's quartics, solves the
// non-trigonometric ones in place, and appends the trigonometric ones (b, c, d, lo, hi,
// index) to a per-warp shared-memory queue that is drained 32 at a time with every lane
// on the trigonometric branch.  No block barrier: a warp's loads still overlap the other
// warps' fp64 work.  Uniform tiles (all one branch) take the per-lane path.  Every
// quartic goes through exactly quartic_boxmin's arithmetic: results are bit-identical to
// quartic_batch_vec_kernel.
constexpr int QWC_CAP = 96;  // queue slots per warp (<= 31 left + 64 appended per tile)

// quartic_boxmin's normalisation (A != 0) and the cubic's Q, R, Delta
__device__ __forceinline__ void qwc_norm(double A, double B, double C, double D, double& b, double& c,
                                         double& d, double& Q, double& R, double& De) {
    const double ia = 1.0 / A;
    b = 0.75 * B * ia;
    c = 0.5 * C * ia;
    d = 0.25 * D * ia;
    cubic_qrd(b, c, d, Q, R, De);
}

constexpr int QWC_NW = 8;  // warps per CTA of the warp-compacted kernel

// flag (the sampled dispatch): run only when *flag == 1
template <int MODE>
__global__ void __launch_bounds__(QWC_NW * 32) quartic_batch_wc_kernel(const double* A, const double* B,
                                                                      const double* C, const double* D,
                                                                      const double* lo, const double* hi,
                                                                      double* x, long long N2,
                                                                      const int* flag = nullptr) {
    if (flag && *flag != 1) return;  // the per-lane kernel takes this batch
    __shared__ double qf[QWC_NW][5][QWC_CAP];  // trigonometric queue: [warp][b c d lo hi][slot]
    __shared__ long long qi[QWC_NW][QWC_CAP];  // [warp][slot] quartic index
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    int qn = 0;  // queued trigonometric quartics (warp-uniform)
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long base = ((long long)blockIdx.x * (blockDim.x >> 5) + wid) * 32; base < N2; base += nw * 32) {
        const long long t = base + lane;
        const bool in = t < N2;
        double2 a = make_double2(1.0, 1.0), b = make_double2(0.0, 0.0), c = b, d = b;
        double2 l = make_double2(-INFINITY, -INFINITY), h = make_double2(INFINITY, INFINITY);
        if (in) {
            a = __ldcs(reinterpret_cast<const double2*>(A) + t);
            b = __ldcs(reinterpret_cast<const double2*>(B) + t);
            c = __ldcs(reinterpret_cast<const double2*>(C) + t);
            d = __ldcs(reinterpret_cast<const double2*>(D) + t);
            if (lo) l = __ldcs(reinterpret_cast<const double2*>(lo) + t);
            if (hi) h = __ldcs(reinterpret_cast<const double2*>(hi) + t);
        }
        const double Av[2] = {a.x, a.y}, Bv[2] = {b.x, b.y}, Cv[2] = {c.x, c.y}, Dv[2] = {d.x, d.y};
        const double lv[2] = {l.x, l.y}, hv[2] = {h.x, h.y};
        double bn[2], cn[2], dn[2], Q[2], R[2], De[2];
        bool tr[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            bn[u] = cn[u] = dn[u] = Q[u] = R[u] = De[u] = 0.0;
            tr[u] = false;
            if (Av[u] != 0.0) {
                qwc_norm(Av[u], Bv[u], Cv[u], Dv[u], bn[u], cn[u], dn[u], Q[u], R[u], De[u]);
                tr[u] = in && isfinite(De[u]) && !(De[u] > 0.0) && !(Q[u] == 0.0 && R[u] == 0.0);
            }
        }
        const unsigned m0 = __ballot_sync(0xffffffffu, tr[0]), m1 = __ballot_sync(0xffffffffu, tr[1]);
        const unsigned act = __ballot_sync(0xffffffffu, in);
        if ((m0 | m1) == 0u || (m0 == act && m1 == act)) {  // uniform tile: per-lane path
            if (in) {
                double2 r;
                r.x = Av[0] != 0.0 ? quartic_core_qrd<MODE>(bn[0], cn[0], dn[0], Q[0], R[0], De[0], Cv[0], Dv[0], lv[0], hv[0])
                                   : clampd(-Dv[0] * rcp_nr(2.0 * Cv[0]), lv[0], hv[0]);
                r.y = Av[1] != 0.0 ? quartic_core_qrd<MODE>(bn[1], cn[1], dn[1], Q[1], R[1], De[1], Cv[1], Dv[1], lv[1], hv[1])
                                   : clampd(-Dv[1] * rcp_nr(2.0 * Cv[1]), lv[1], hv[1]);
                __stcs(reinterpret_cast<double2*>(x) + t, r);
            }
            continue;
        }
        // append the trigonometric quartics, solve the others in place
        const int n0 = __popc(m0), n1 = __popc(m1);
        const int pos[2] = {qn + __popc(m0 & lt), qn + n0 + __popc(m1 & lt)};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (tr[u]) {
                qf[wid][0][pos[u]] = bn[u];
                qf[wid][1][pos[u]] = cn[u];
                qf[wid][2][pos[u]] = dn[u];
                qf[wid][3][pos[u]] = lv[u];
                qf[wid][4][pos[u]] = hv[u];
                qi[wid][pos[u]] = 2 * t + u;
            } else if (in) {
                x[2 * t + u] = Av[u] != 0.0 ? quartic_core_qrd<MODE>(bn[u], cn[u], dn[u], Q[u], R[u], De[u], Cv[u], Dv[u], lv[u], hv[u])
                                            : clampd(-Dv[u] * rcp_nr(2.0 * Cv[u]), lv[u], hv[u]);
            }
        }
        qn += n0 + n1;
        __syncwarp();
        while (qn >= 32) {  // one full pass on the trigonometric branch
            const int k = qn - 32 + lane;
            const double qb = qf[wid][0][k], qc = qf[wid][1][k], qd = qf[wid][2][k];
            double QQ, RR, DD;
            cubic_qrd(qb, qc, qd, QQ, RR, DD);
            __stcs(x + qi[wid][k], trig_pick<MODE>(qb, qc, qd, QQ, RR, DD, qf[wid][3][k], qf[wid][4][k]));
            qn -= 32;
            __syncwarp();
        }
    }
    if (lane < qn) {  // the warp's last partial pass
        const int k = lane;
        const double qb = qf[wid][0][k], qc = qf[wid][1][k], qd = qf[wid][2][k];
        double QQ, RR, DD;
        cubic_qrd(qb, qc, qd, QQ, RR, DD);
        __stcs(x + qi[wid][k], trig_pick<MODE>(qb, qc, qd, QQ, RR, DD, qf[wid][3][k], qf[wid][4][k]));
    }
}


// Dispatch between the two batch kernels from a strided sample of the batch: one CTA
// classifies 4096 quartics (every (N/4096)-th) and sets flag = 1 when both branches are
// common (trigonometric share in [1/64, 63/64]); the per-lane kernel runs when flag == 0
// and the warp-compacted one when flag == 1 (the other returns at once), so the choice
// needs no host round trip.
__global__ void __launch_bounds__(512) quartic_sample_kernel(const double* A, const double* B, const double* C,
                                                             const double* D, long long N, int* flag) {
    // 512 threads x 8 samples, every load issued before any arithmetic (one memory round trip)
    constexpr int PER = 8, NS = 512 * PER;
    __shared__ int cnt[2];
    if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
    __syncthreads();
    const long long step = N >= NS ? N / NS : 1;
    double a[PER], b[PER], c[PER], d[PER];
    bool ok[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const long long i = (long long)(u * 512 + threadIdx.x) * step;
        ok[u] = i < N;
        a[u] = ok[u] ? __ldg(A + i) : 0.0;
        b[u] = ok[u] ? __ldg(B + i) : 0.0;
        c[u] = ok[u] ? __ldg(C + i) : 0.0;
        d[u] = ok[u] ? __ldg(D + i) : 0.0;
    }
    int nt = 0, nall = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        if (!ok[u]) continue;
        ++nall;
        if (a[u] != 0.0) {
            double bn, cn, dn, Q, R, De;
            const double ia = 1.0 / a[u];
            bn = 0.75 * b[u] * ia;
            cn = 0.5 * c[u] * ia;
            dn = 0.25 * d[u] * ia;
            cubic_qrd(bn, cn, dn, Q, R, De);
            nt += (isfinite(De) && !(De > 0.0) && !(Q == 0.0 && R == 0.0)) ? 1 : 0;
        }
    }
    nt = __reduce_add_sync(0xffffffffu, nt);
    nall = __reduce_add_sync(0xffffffffu, nall);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&cnt[0], nt);
        atomicAdd(&cnt[1], nall);
    }
    __syncthreads();
    if (threadIdx.x == 0) *flag = (64 * cnt[0] >= cnt[1] && 64 * cnt[0] <= 63 * cnt[1]) ? 1 : 0;
}

template <int MODE>
__global__ void __launch_bounds__(256) quartic_batch_kernel(const double* A, const double* B,
                                                            const double* C, const double* D,
                                                            const double* lo, const double* hi,
                                                            double* x, long long N) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < N; t += stride) {
        const double l = lo ? lo[t] : -INFINITY, h = hi ? hi[t] : INFINITY;
        x[t] = quartic_boxmin<MODE>(A[t], B[t], C[t], D[t], l, h);
    }
}

}  // namespace


// ======================================================================
// host runtime
// ======================================================================
struct admm_ctx {
    int m = 0;
    long long n = 0, n_pad = 0, q = 0, q_total = 0, j0 = 0;
    int device = 0, sms = 148;
    cudaStream_t stream = nullptr;      // caller's stream: all work is ordered on it
    cudaStream_t cap_stream = nullptr;  // private stream used only to capture the graph
    int world = 1, rank = 0;
    bool dist = false;            // collective path (admm_dist given, any world size)
    bool hz = false;              // horizon-block sharding (ADMM_SHARD_HORIZON)
    long long n_total = 0, k_begin = 0;  // whole horizon, this rank's first step (hz)
    ncclComm_t comm = nullptr;
    bool owns_ws = false;
    char* ws = nullptr;
    size_t ws_bytes = 0;
    Layout L{};
    KArgs ka{};
    unsigned long long* vflag = nullptr;
    double* obj_rows = nullptr;
    admm_params params{};
    bool has_problem = false;
    int bs = 32, T = 1, tile = 64, G = 1;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    int graph_mode = -1;  // box mode the graph was built for
    std::string err;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    double t_call_ms = 0.0, t_sweep_ms = 0.0;
    long long iter_host = 0;
    Ctrl* h_ctrl = nullptr;       // pinned
    long long* h_iter = nullptr;  // pinned
    unsigned long long cond = 0;  // cudaGraphConditionalHandle
    bool no_graph = false;        // ADMM_NO_GRAPH=1: plain launches (for ncu)
    int last_engine = 0;          // ADMM_ENGINE_* of the last iterate/solve
    DParams dparams{};            // parameters of the current call (host copy of the device block)
    long long launches = 0;       // kernels launched by this context since create
    bool prep_ok = false;         // bq / ib2s valid (on-chip-sized problems)
    bool fx_ok = false;           // fixed-point scales of the row sums valid (finite bounds)
    double fx_scale[MAXM] = {}, fx_inv[MAXM] = {};
    bool use_tma = false;         // streaming engine: the TMA sweep (sweep2_kernel) runs
    const void* s2_fn = nullptr;  // sweep2_kernel instantiation of the current plan
    S2Maps s2maps{};              // its TMA tensor maps
    size_t s2_smem = 0;           // its dynamic shared memory (the stage ring)
    int coeff_bits = 64;          // F2: storage precision of a2, a1, b2, b1 (64 or 32)
    int cpt = 2;                  // streaming sweep: cells per thread (2, or 4 for m <= 2)
    int rl = 0;                   // streaming sweep: row loop, CTA size (0 = off, 128 or 64)
    bool graph_dirty = true;      // problem changed since the graph was captured
    S2Args s2{};
};

namespace {

admm_status fail(admm_ctx* c, admm_status s, const std::string& msg) {
    if (c) c->err = msg;
    return s;
}

#define CKC(call)                                                                       \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess)                                                          \
            return fail(ctx, ADMM_ERR_CUDA,                                             \
                        std::string(#call) + ": " + cudaGetErrorString(_e));            \
    } while (0)

#define CKN(call)                                                                       \
    do {                                                                                \
        ncclResult_t _r = (call);                                                       \
        if (_r != ncclSuccess)                                                          \
            return fail(ctx, ADMM_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(_r)); \
    } while (0)

int grid_for(long long work, int bs, int sms) {
    long long g = (work + bs - 1) / bs;
    return (int)std::max(1LL, std::min(g, (long long)sms * 8));
}

void upload_params(admm_ctx* ctx, long long iter_limit, int stop_on_conv) {
    DParams d{};
    d.tau = ctx->params.tau;
    d.hi_ratio = ctx->params.hi_ratio;
    d.lo_ratio = ctx->params.lo_ratio;
    d.r_bar = ctx->params.r_bar;
    d.sigma_bar = ctx->params.sigma_bar;
    d.iter_limit = iter_limit;
    d.check_every = ctx->params.check_every;
    d.adapt = ctx->params.adapt_rho;
    d.rescale = ctx->params.rescale_duals;
    d.box_mode = ctx->params.box_mode;
    d.stop_on_conv = stop_on_conv;
    ctx->dparams = d;
    cudaMemcpyAsync(ctx->ws + ctx->L.prm, &ctx->dparams, sizeof(d), cudaMemcpyHostToDevice, ctx->stream);
}

// F2: round a2, a1, b2, b1 to fp32 (round to nearest even, the cast), keep the
// rounded values in the fp64 arrays (all engines see one problem) and the fp32 copies
__global__ void round_coeff_kernel(long long NE, double* a2, double* a1, double* b2, double* b1,
                                   float* fa2, float* fa1, float* fb2, float* fb1) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < NE; t += stride) {
        const float u2 = __double2float_rn(a2[t]), u1 = __double2float_rn(a1[t]);
        const float w2 = __double2float_rn(b2[t]), w1 = __double2float_rn(b1[t]);
        fa2[t] = u2; fa1[t] = u1; fb2[t] = w2; fb1[t] = w1;
        a2[t] = u2; a1[t] = u1; b2[t] = w2; b1[t] = w1;
    }
}

typedef void (*sweep_fn)(KArgs);

// Barrier-free (fixed-point, last-warp-finalises) sweep for rows spanning several
// tiles (horizon n = 1e6: 26 -> 34 % of HBM peak); the barrier variant stays for
// one-tile rows, where it measured faster (44 vs 38 % at q = 1e4, profiles/README.md).
bool use_pf_sweep(const admm_ctx* ctx) {
    const char* e = getenv("ADMM_SWEEP_PF");
    if (!(e && (e[0] == '1' || e[0] == '2'))) return false;  // opt-in while measured
    return ctx->fx_ok && ctx->T == 1 && ctx->m <= 2 && ctx->cpt == 2;
}

size_t pf_smem_bytes(const admm_ctx* ctx) {
    if (ctx->cpt == 4)  // staged 4-cell sweep: the per-thread slab
        return (size_t)(ctx->m == 1 ? Slab4<1>::NF : Slab4<2>::NF) * ctx->bs * 4 * 8;
    if (!use_pf_sweep(ctx)) return 0;
    const size_t per = ctx->coeff_bits == 32 ? (size_t)PFCfg<2, float>::PER_THREAD
                                             : (size_t)PFCfg<2, double>::PER_THREAD;
    const size_t per1 = ctx->coeff_bits == 32 ? (size_t)PFCfg<1, float>::PER_THREAD
                                              : (size_t)PFCfg<1, double>::PER_THREAD;
    return 2 * (size_t)ctx->bs * (ctx->m == 1 ? per1 : per);
}

bool use_fx_sweep(const admm_ctx* ctx) {
    if (use_pf_sweep(ctx)) {  // ADMM_SWEEP_PF=1: with the fixed-point slots, =2: with block barriers
        const char* e = getenv("ADMM_SWEEP_PF");
        return !(e && e[0] == '2');
    }
    const char* e = getenv("ADMM_SWEEP_FX");
    if (e && e[0] == '0') return false;
    if (e && e[0] == '1') return ctx->fx_ok;
    return ctx->fx_ok && ctx->T > 1;
}

template <typename CT>
sweep_fn pick_sweep_t(int m, int mode, bool fx, bool pf, int cpt, int rl) {
#define S(MM, UU)                                                                              \
    if (m == MM) {                                                                             \
        if (fx) return mode == BOX_EXACT ? sweep_kernel<MM, BOX_EXACT, true, CT, false, UU, 0> \
                                         : sweep_kernel<MM, BOX_PROJECT, true, CT, false, UU, 0>; \
        return mode == BOX_EXACT ? sweep_kernel<MM, BOX_EXACT, false, CT, false, UU, 0>    \
                                 : sweep_kernel<MM, BOX_PROJECT, false, CT, false, UU, 0>; \
    }
#define SR(MM, TT)                                                                             \
    if (m == MM) return mode == BOX_EXACT ? sweep_kernel<MM, BOX_EXACT, false, CT, false, 2, TT> \
                                          : sweep_kernel<MM, BOX_PROJECT, false, CT, false, 2, TT>;
    if (rl == 128) {  // row loop: 128-thread CTAs own whole rows
        SR(1, 128) SR(2, 128)
        return nullptr;
    }
    if (rl == 64) {
        SR(1, 64) SR(2, 64)
        return nullptr;
    }
#define SP(MM)                                                                                 \
    if (m == MM && pf) {                                                                       \
        if (fx) return mode == BOX_EXACT ? sweep_kernel<MM, BOX_EXACT, true, CT, true, 2, 0> \
                                         : sweep_kernel<MM, BOX_PROJECT, true, CT, true, 2, 0>; \
        return mode == BOX_EXACT ? sweep_kernel<MM, BOX_EXACT, false, CT, true, 2, 0>      \
                                 : sweep_kernel<MM, BOX_PROJECT, false, CT, true, 2, 0>;   \
    }
    if (cpt == 4) {
        S(1, 4) S(2, 4)
        return nullptr;
    }
    SP(1) SP(2)
    S(1, 2) S(2, 2) S(3, 2) S(4, 2)
#undef S
#undef SP
#undef SR
    return nullptr;
}

// f32: F2 mixed-precision sweep (coefficients read from their fp32 copies); pf: the
// cp.async-prefetching sweep (one-tile rows, m <= 2; use_pf_sweep); cpt: cells per thread
sweep_fn pick_sweep(int m, int mode, bool fx, bool f32, bool pf, int cpt, int rl) {
    return f32 ? pick_sweep_t<float>(m, mode, fx, pf, cpt, rl) : pick_sweep_t<double>(m, mode, fx, pf, cpt, rl);
}

// The prefetching sweep: rows of one tile (n <= 2 * block size), m <= 2, fixed-point
// row sums (finite boxes).  ADMM_SWEEP_PF=0 turns it off.
bool use_pf_sweep(const admm_ctx* ctx);
size_t pf_smem_bytes(const admm_ctx* ctx);

// TMA tensor maps (driver entry point cuTensorMapEncodeTiled, no libcuda link needed)
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

bool tmap(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base, const cuuint64_t* dims,
          const cuuint64_t* strides, const cuuint32_t* box) {
    auto fn = tmap_encoder();
    if (!fn) return false;
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    // L2 promotion 64 B: with 256 B a q = 1e5 sweep launch read 10.85 GB from DRAM against the
    // 9.63 GB algorithmic (the promoted blocks straddle the 64-B-aligned row segments), with
    // 64 B it reads 9.63 GB and is 1.8 % faster (profiles/r02i/promo_*); experiments:
    // ADMM_TMA_PROMO = 0 none / 64 / 128 / 256 bytes
    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    if (const char* e = getenv("ADMM_TMA_PROMO")) {
        const int v = atoi(e);
        promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
              : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
              : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }
    return fn(m, dt, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the four maps of the TMA sweep for chunks of tl cells (admm_sweep2.cuh S2Maps)
bool build_s2_maps(admm_ctx* ctx, int tl) {
    const KArgs& a = ctx->ka;
    const Layout& L = ctx->L;
    const cuuint64_t np = (cuuint64_t)ctx->n_pad, q = (cuuint64_t)ctx->q, m = (cuuint64_t)ctx->m;
    const cuuint32_t T = (cuuint32_t)tl, M = (cuuint32_t)ctx->m;
    S2Maps& t = ctx->s2maps;
    {
        const cuuint64_t dims[3] = {np, q, m}, str[2] = {np * 8, q * np * 8};
        const cuuint32_t box[3] = {T, 1, M};
        if (!tmap(&t.x, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a.x, dims, str, box)) return false;
    }
    {
        const bool f32 = ctx->coeff_bits == 32;
        const cuuint64_t es = f32 ? 4 : 8;
        const cuuint64_t cstr = f32 ? m * q * np * 4 : (cuuint64_t)(L.a1 - L.a2);
        if (!f32 && ((cuuint64_t)(L.b2 - L.a1) != cstr || (cuuint64_t)(L.b1 - L.b2) != cstr)) return false;
        const cuuint64_t dims[4] = {np, q, m, 4}, str[3] = {np * es, q * np * es, cstr};
        const cuuint32_t box[4] = {T, 1, M, 4};
        const void* base = f32 ? (const void*)a.fa2 : (const void*)a.a2;
        if (!tmap(&t.c, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims,
                  str, box))
            return false;
    }
    {
        const cuuint64_t dims[3] = {np, q, 2}, str[2] = {np * 8, (cuuint64_t)(L.v - L.y)};
        const cuuint32_t box[3] = {T, 1, 2};
        if (!tmap(&t.yv, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a.y, dims, str, box)) return false;
    }
    {
        const cuuint64_t dims[3] = {np, m, 2}, str[2] = {np * 8, (cuuint64_t)(L.hi - L.lo)};
        const cuuint32_t box[3] = {T, M, 2};
        if (!tmap(&t.box, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a.lo, dims, str, box)) return false;
    }
    return true;
}

// streaming engine: the TMA sweep (admm_sweep2.cuh) whenever the fixed-point row
// scales exist (finite boxes) and m <= 4; ADMM_SWEEP2=0 selects the register-fed
// sweep_kernel (kept for infinite bounds and as a measured alternative)
admm_status plan_stream(admm_ctx* ctx) {
    ctx->use_tma = false;
    const char* opt = getenv("ADMM_SWEEP2");
    if (opt && opt[0] == '0') return ADMM_OK;
    if (!ctx->fx_ok || ctx->m > 4) return ADMM_OK;
    int ns = 0, tl = 0;
    size_t smem = 0;
    const void* fn = sweep2_pick(ctx->m, ctx->params.box_mode, ctx->coeff_bits / 8, ctx->q, &ns, &smem, &tl);
    if (!fn) return ADMM_OK;
    CKC(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CKC(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, S2_NT, smem));
    if (occ < 1) return ADMM_OK;
    occ = std::min(occ, 32);
    if (!build_s2_maps(ctx, tl)) return ADMM_OK;  // no tensor maps: the register-fed sweep
    ctx->s2 = sweep2_plan(ctx->q, ctx->n_pad, tl, occ * ctx->sms);
    ctx->s2_fn = fn;
    ctx->s2_smem = smem;
    ctx->use_tma = true;
    if (const char* dbg = getenv("ADMM_DEBUG")) {
        if (dbg[0] == '1') {
            cudaFuncAttributes fa;
            if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess)
                fprintf(stderr, "[admm] sweep2: chunk %d regs %d local %zu smem %zu+%zu occ %d G %d S %d TPS %d TPR %d\n",
                        tl, fa.numRegs, fa.localSizeBytes, fa.sharedSizeBytes, smem, occ, ctx->s2.G, ctx->s2.S,
                        ctx->s2.TPS, ctx->s2.TPR);
        }
    }
    return ADMM_OK;
}

// body of one while-loop pass: check_every iterations
admm_status record_body(admm_ctx* ctx, sweep_fn fn, cudaStream_t st) {
    const int K = std::max(1, ctx->params.check_every);
    for (int r = 0; r < K; ++r) {
        if (ctx->use_tma) {
            void* args[] = {(void*)&ctx->ka, (void*)&ctx->s2, (void*)&ctx->s2maps};
            CKC(cudaLaunchKernel(ctx->s2_fn, dim3((unsigned)ctx->s2.G), dim3(S2_NT), args, ctx->s2_smem, st));
        } else
            fn<<<ctx->G, ctx->bs, pf_smem_bytes(ctx), st>>>(ctx->ka);
        CKC(cudaGetLastError());
        if (ctx->dist) {
            if (ctx->hz) {  // row sums over k and their dg extrema, every rank's rows
                CKN(ncclAllReduce(ctx->ka.rowacc, ctx->ka.rowacc, (size_t)ctx->q * MAXM, ncclUint64, ncclSum,
                                  ctx->comm, st));
                CKN(ncclAllReduce(ctx->ka.hzdg, ctx->ka.hzdg, (size_t)ctx->q * 2 * MAXM, ncclUint64, ncclMax,
                                  ctx->comm, st));
            }
            CKN(ncclAllGather(ctx->ka.xsend, ctx->ka.xall, XB, ncclDouble, ctx->comm, st));
            if (ctx->hz)
                hz_rows_kernel<<<1, 256, 0, st>>>(ctx->ka);
            else
                finalize_kernel<<<1, 32, 0, st>>>(ctx->ka);
            CKC(cudaGetLastError());
        }
    }
    return ADMM_OK;
}

__global__ void set_cond_kernel(KArgs a, cudaGraphConditionalHandle h) {
    const long long it = *(volatile long long*)a.iter;
    const Ctrl& c = a.ctrl[it & 1];
    const bool go = !c.done && it < a.prm->iter_limit;
    cudaGraphSetConditional(h, go ? 1u : 0u);
}

admm_status build_graph(admm_ctx* ctx) {
    if (ctx->gexec && ctx->graph_mode == ctx->params.box_mode && !ctx->graph_dirty) return ADMM_OK;
    if (ctx->gexec) {
        cudaGraphExecDestroy(ctx->gexec);
        ctx->gexec = nullptr;
    }
    if (ctx->graph) {
        cudaGraphDestroy(ctx->graph);
        ctx->graph = nullptr;
    }
    sweep_fn fn = pick_sweep(ctx->m, ctx->params.box_mode, use_fx_sweep(ctx), ctx->coeff_bits == 32, use_pf_sweep(ctx), ctx->cpt, ctx->rl);
    if (!fn) return fail(ctx, ADMM_ERR_INVALID, "m must be in 1..4");
    int occ = 0;
    const size_t dsm = pf_smem_bytes(ctx);
    if (dsm > 0)
        CKC(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
    CKC(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, ctx->bs, dsm));
    occ = std::max(1, std::min(occ, 32));
    const long long items = ctx->rl ? ctx->q : ctx->q * ctx->T;
    ctx->G = (int)std::max(1LL, std::min(items, (long long)occ * ctx->sms));
    ctx->ka.G = ctx->G;
    {
        admm_status ps = plan_stream(ctx);
        if (ps != ADMM_OK) return ps;
    }
    if (!ctx->dist) {
        CKC(cudaGraphCreate(&ctx->graph, 0));
        cudaGraphConditionalHandle h;
        CKC(cudaGraphConditionalHandleCreate(&h, ctx->graph, 1, cudaGraphCondAssignDefault));
        ctx->cond = h;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CKC(cudaGraphAddNode(&node, ctx->graph, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CKC(cudaStreamBeginCaptureToGraph(ctx->cap_stream, body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
        admm_status st = record_body(ctx, fn, ctx->cap_stream);
        set_cond_kernel<<<1, 1, 0, ctx->cap_stream>>>(ctx->ka, h);
        cudaGraph_t out = nullptr;
        cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &out);
        if (st != ADMM_OK) return st;
        CKC(ce);
    } else {
        CKC(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
        admm_status st = record_body(ctx, fn, ctx->cap_stream);
        cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &ctx->graph);
        if (st != ADMM_OK) return st;
        CKC(ce);
    }
    CKC(cudaGraphInstantiate(&ctx->gexec, ctx->graph, 0));
    ctx->graph_mode = ctx->params.box_mode;
    ctx->graph_dirty = false;
    return ADMM_OK;
}

admm_status read_ctrl(admm_ctx* ctx) {
    CKC(cudaMemcpyAsync(ctx->h_iter, ctx->ka.iter, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CKC(cudaStreamSynchronize(ctx->stream));
    ctx->iter_host = *ctx->h_iter;
    CKC(cudaMemcpyAsync(ctx->h_ctrl, ctx->ka.ctrl + (ctx->iter_host & 1), sizeof(Ctrl),
                        cudaMemcpyDeviceToHost, ctx->stream));
    CKC(cudaStreamSynchronize(ctx->stream));
    return ADMM_OK;
}

typedef void (*persist_fn)(KArgs, PArgs);

persist_fn pick_persist(int m, int mode) {
#define S(MM)                                                                                  \
    if (m == MM) return mode == BOX_EXACT ? persist_kernel<MM, BOX_EXACT> : persist_kernel<MM, BOX_PROJECT>;
    S(1) S(2) S(3) S(4)
#undef S
    return nullptr;
}

struct PPlan {
    bool ok = false;
    int TC = 0, T = 0, G = 0, BS = 0, TC0 = 0;
    size_t smem = 0;
};

// tile the (j, k) plane so that every SM gets about one CTA and each CTA's
// state fits in shared memory; all CTAs must be co-resident
PPlan plan_persist(admm_ctx* ctx, persist_fn fn) {
    PPlan pl;
    if (ctx->dist || !fn) return pl;
    const long long n = ctx->n, q = ctx->q;
    const int sms = ctx->sms;
    long long T = std::max<long long>((n + 1023) / 1024, q <= sms ? sms / q : 1);
    T = std::min<long long>(T, (n + 63) / 64);
    T = std::max<long long>(T, 1);
    long long TC = 0;
    size_t smem = 0;
    for (int guard = 0; guard < 4096; ++guard) {
        const long long per = (n + T - 1) / T;
        TC = 64 * ((per + 63) / 64);
        T = (n + TC - 1) / TC;
        smem = (size_t)(7 * ctx->m + 2) * TC * 8;
        if (smem <= 200 * 1024) break;
        ++T;
    }
    const long long G = q * T;
    if (G > 32LL * sms) return pl;
    if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return pl;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, (int)(TC / 2), smem) !=
        cudaSuccess) {
        cudaGetLastError();
        return pl;
    }
    if ((long long)occ * sms < G) return pl;
    pl.ok = true;
    pl.TC = (int)TC;
    pl.T = (int)T;
    pl.G = (int)G;
    pl.BS = (int)(TC / 2);
    pl.smem = smem;
    return pl;
}

admm_status launch_persist(admm_ctx* ctx, persist_fn fn, const PPlan& pl) {
    PArgs pa;
    pa.TC = pl.TC;
    pa.T = pl.T;
    pa.G = pl.G;
    pa.gpart = (double*)(ctx->ws + ctx->L.pg);
    pa.cpart = (double*)(ctx->ws + ctx->L.pc);
    pa.rpart = (double*)(ctx->ws + ctx->L.pr);
    pa.rowchk = (double*)(ctx->ws + ctx->L.prc);
    pa.bar = (unsigned*)(ctx->ws + ctx->L.pbar);
    KArgs ka = ctx->ka;
    void* args[] = {&ka, &pa};
    CKC(cudaLaunchCooperativeKernel((const void*)fn, pl.G, pl.BS, args, pl.smem, ctx->stream));
    ctx->launches += 1;
    return ADMM_OK;
}

typedef void (*cluster_fn)(KArgs, CArgs);

cluster_fn pick_cluster(int m, int mode) {
#define S(MM)                                                                                  \
    if (m == MM) return mode == BOX_EXACT ? persist_cluster_kernel<MM, BOX_EXACT>              \
                                          : persist_cluster_kernel<MM, BOX_PROJECT>;
    S(1) S(2) S(3) S(4)
#undef S
    return nullptr;
}

// rows inside clusters of T <= 16 CTAs (see admm_onchip.cuh): one CTA per SM,
// at most 16 bulk warps (usually one cell per thread) + the consensus warp.
// Tile 0 (which also runs the consensus chain) gets TC0 ~ frac * n/T cells.
// Candidate tile counts: the one that spreads the rows over the SMs, then
// fewer (when q*T CTAs do not fit, e.g. 3 x 50 > 148), then more (when a
// long row does not fit the shared memory of T CTAs).
PPlan plan_cluster(admm_ctx* ctx, cluster_fn fn) {
    PPlan pl;
    if (ctx->dist || !fn || !ctx->prep_ok || !ctx->fx_ok) return pl;
    const long long n = ctx->n, q = ctx->q;
    const int sms = ctx->sms;
    if (q > 32LL * sms) return pl;
    if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
        cudaSuccess)
        cudaGetLastError();
    double frac = 0.4;  // measured best for PHEV q=50 (profiles/README.md)
    if (const char* e = getenv("ADMM_TILE0_FRAC")) frac = atof(e);
    long long T0 = std::max<long long>(1, std::min<long long>(ONCHIP_MAX_T, (sms + q - 1) / q));
    T0 = std::min<long long>(T0, std::max<long long>(1, n / 32));
    std::vector<long long> cand;
    for (long long T = T0; T >= 1; --T) cand.push_back(T);
    for (long long T = T0 + 1; T <= ONCHIP_MAX_T; ++T) cand.push_back(T);
    // experiments: ADMM_CLUSTER_T forces the tiles per row, ADMM_CLUSTER_WARPS caps the
    // bulk warps per CTA (more cells per thread, smaller CTAs, more CTAs per SM)
    if (const char* e = getenv("ADMM_CLUSTER_T")) cand.assign(1, std::max(1LL, atoll(e)));
    int wcap = ONCHIP_MAX_WARPS - 1;
    if (const char* e = getenv("ADMM_CLUSTER_WARPS")) wcap = std::max(1, std::min(wcap, atoi(e)));
    for (long long T : cand) {
        long long TC0 = n, TC = n;
        if (T > 1) {
            TC0 = std::max<long long>(1, std::min<long long>(n - (T - 1), (long long)std::llround(frac * n / T)));
            TC = (n - TC0 + T - 2) / (T - 1);
            if (TC0 + (T - 2) * TC >= n) continue;  // last tile would be empty
        }
        const long long TCM = std::max(TC0, TC);
        const size_t smem = (size_t)(9 * ctx->m + 2) * TCM * 8;
        if (smem > 200 * 1024 || TCM > 4 * 512) continue;
        const long long G = q * T;
        if (G > 32LL * sms) continue;
        const int nbw = (int)std::min<long long>(wcap, (TCM + 31) / 32);
        const int BS = (nbw + 1) * 32;
        if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)G);
        cfg.blockDim = dim3((unsigned)BS);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)T;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)fn, &cfg) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if ((long long)nclusters < q) continue;  // all CTAs must be co-resident
        pl.ok = true;
        pl.TC0 = (int)TC0;
        pl.TC = (int)TC;
        pl.T = (int)T;
        pl.G = (int)G;
        pl.BS = BS;
        pl.smem = smem;
        return pl;
    }
    return pl;
}

admm_status launch_cluster(admm_ctx* ctx, cluster_fn fn, const PPlan& pl) {
    CArgs ca;
    ca.TC0 = pl.TC0;
    ca.TC = pl.TC;
    ca.T = pl.T;
    ca.G = pl.G;
    for (int i = 0; i < MAXM; ++i) {
        ca.fx_scale[i] = ctx->fx_scale[i];
        ca.fx_inv[i] = ctx->fx_inv[i];
    }
    ca.bq = (const double*)(ctx->ws + ctx->L.bq);
    ca.ib2s = (const double*)(ctx->ws + ctx->L.ib2s);
    ca.pub = (double*)(ctx->ws + ctx->L.pub);
    ca.chk = (unsigned long long*)(ctx->ws + ctx->L.chk);
    ca.cnt = (unsigned long long*)(ctx->ws + ctx->L.pbar);
    CKC(cudaMemsetAsync(ca.cnt, 0, 256, ctx->stream));
    const long long nslots = (long long)PUB_BUFS * ctx->m * ctx->q;
    onchip_reset_kernel<<<(unsigned)std::min<long long>(64, (nslots + 255) / 256), 256, 0,
                          ctx->stream>>>(ca.pub, nslots, ca.chk);
    CKC(cudaGetLastError());
    if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pl.smem) != cudaSuccess)
        return fail(ctx, ADMM_ERR_CUDA, "cluster kernel: shared memory attribute");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)pl.G);
    cfg.blockDim = dim3((unsigned)pl.BS);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)pl.T;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CKC(cudaLaunchKernelEx(&cfg, fn, ctx->ka, ca));
    ctx->launches += 2;  // onchip_reset_kernel + the cluster kernel
    return ADMM_OK;
}

// Message-passing cluster engine (admm_onchip2.cuh): rows in clusters of T CTAs of nw
// warps (tile 0: nw-1 bulk warps + the consensus warp).  The plan minimises a model of
// the iteration time over (T, nw) among the shapes whose q*T CTAs are all co-resident:
//   cells per thread k_t = ceil(cells of tile t / bulk threads of tile t) -> latency
//   L * max_t k_t of the dependent Algorithm-1 chains, and fp64 throughput
//   W * (CTAs per SM) * (cells per CTA) when an SM holds several CTAs,
// plus a per-message cost of the row exchange (T * nw slots summed by the row warp).
// L = 2800 and W = 6.9 cycles are the PHEV q = 50 per-cell latency and per-SM
// throughput of profiles/r02b/cluster_phase.txt.  ADMM_CLUSTER_T / ADMM_CLUSTER_WARPS
// force a shape (experiments).
struct C2Plan {
    bool ok = false;
    int T = 0, NW = 0, TC0 = 0, TC = 0, G = 0;
    int k = 0;  // cells per bulk thread (the most loaded tile)
    size_t smem = 0;
};

size_t oc2_smem(int m, long long TCM, int T, int nw) {
    return ((((size_t)(9 * m + 2) * TCM + 1) & ~(size_t)1) * 8) + oc2_msg_bytes(m, T, nw);
}

C2Plan plan_cluster2(admm_ctx* ctx, const void* fn) {
    C2Plan pl;
    if (ctx->dist || !fn || !ctx->prep_ok || !ctx->fx_ok) return pl;
    const long long n = ctx->n, q = ctx->q;
    const int sms = ctx->sms, m = ctx->m;
    if (q > 32LL * sms) return pl;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        cudaGetLastError();
    int forceT = 0, forceW = 0;
    if (const char* e = getenv("ADMM_CLUSTER_T")) forceT = atoi(e);
    if (const char* e = getenv("ADMM_CLUSTER_WARPS")) forceW = atoi(e);
    struct Cand {
        double cost;
        int T, NW;
        long long TC0, TC;
    };
    std::vector<Cand> cand;
    for (int T = 1; T <= OC2_MAX_T; ++T) {
        if (forceT && T != forceT) continue;
        if (T > 1 && n < 2LL * T) break;
        for (int NW = 2; NW <= OC2_MAX_W; ++NW) {
            if (forceW && NW != forceW) continue;
            const long long b0 = 32LL * (NW - 1), b1 = 32LL * NW;  // bulk threads of tile 0 / others
            long long TC0 = n, TC = n;
            if (T > 1) {
                // cells in proportion to the bulk threads (tile 0 also runs the consensus chain)
                TC0 = std::max<long long>(1, std::min<long long>(n - (T - 1), (long long)((double)n * b0 / (b0 + (T - 1) * b1))));
                if (const char* e = getenv("ADMM_TILE0_FRAC"))
                    TC0 = std::max<long long>(1, std::min<long long>(n - (T - 1), std::llround(atof(e) * n / T)));
                TC = (n - TC0 + T - 2) / (T - 1);
                if (TC0 + (T - 2) * TC >= n) continue;  // last tile would be empty
            }
            const long long TCM = std::max(TC0, TC);
            if (oc2_smem(m, TCM, T, NW) > 200 * 1024) continue;
            const long long G = q * T;
            const long long k = std::max((TC0 + b0 - 1) / b0, (TC + b1 - 1) / b1);  // cells per thread
            // CTAs per SM: register file (128 regs x 32 lanes per warp) and shared memory
            const long long by_regs = 65536LL / (32LL * NW * OC2_REGS), by_smem = (228 * 1024) / (long long)(oc2_smem(m, TCM, T, NW) + 1024);
            const long long per_sm_cap = std::max(1LL, std::min(by_regs, by_smem));
            const long long cps = (G + sms - 1) / sms;
            if (cps > per_sm_cap) continue;
            const double L = 2800.0 * m / 2.0, W = 6.9 * m / 2.0;
            const double cost = std::max(L * (double)k, W * (double)(cps * TCM)) + 30.0 * ((T * NW + 31) / 32) +
                                40.0 * T;
            cand.push_back({cost, T, NW, TC0, TC});
        }
    }
    std::sort(cand.begin(), cand.end(), [](const Cand& x, const Cand& y) {
        return x.cost < y.cost || (x.cost == y.cost && (x.T < y.T || (x.T == y.T && x.NW < y.NW)));
    });
    for (const Cand& c : cand) {
        const long long TCM = std::max(c.TC0, c.TC);
        const size_t smem = oc2_smem(m, TCM, c.T, c.NW);
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(q * c.T));
        cfg.blockDim = dim3((unsigned)(32 * c.NW));
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)c.T;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if ((long long)nclusters < q) continue;  // all CTAs must be co-resident
        if (getenv("ADMM_DEBUG_PLAN"))
            fprintf(stderr, "[admm] cluster2 plan: T=%d NW=%d TC0=%lld TC=%lld G=%lld smem=%zu cost=%.0f clusters=%d\n",
                    c.T, c.NW, c.TC0, c.TC, q * c.T, smem, c.cost, nclusters);
        pl.ok = true;
        pl.T = c.T;
        pl.NW = c.NW;
        pl.TC0 = (int)c.TC0;
        pl.TC = (int)c.TC;
        pl.G = (int)(q * c.T);
        pl.k = (int)std::max((c.TC0 + 32LL * (c.NW - 1) - 1) / (32LL * (c.NW - 1)), (c.TC + 32LL * c.NW - 1) / (32LL * c.NW));
        pl.smem = smem;
        return pl;
    }
    return pl;
}

admm_status launch_cluster2(admm_ctx* ctx, const void* fn, const C2Plan& pl) {
    C2Args ca;
    ca.TC0 = pl.TC0;
    ca.TC = pl.TC;
    ca.T = pl.T;
    ca.G = pl.G;
    for (int i = 0; i < MAXM; ++i) {
        ca.fx_scale[i] = ctx->fx_scale[i];
        ca.fx_inv[i] = ctx->fx_inv[i];
    }
    ca.bq = (const double*)(ctx->ws + ctx->L.bq);
    ca.ib2s = (const double*)(ctx->ws + ctx->L.ib2s);
    ca.pub = (unsigned long long*)(ctx->ws + ctx->L.pub2);
    ca.chkv = (unsigned long long*)(ctx->ws + ctx->L.chkv2);
    ca.chkx = (unsigned long long*)(ctx->ws + ctx->L.chkx2);
    ca.cnt = (unsigned long long*)(ctx->ws + ctx->L.cnt2);
    ca.prm = ctx->dparams;
    // epochs are 32-bit iteration / check counts of the call: at most 2^31 iterations per
    // launch (run_loop relaunches)
    if (ca.prm.iter_limit - ctx->iter_host > (1LL << 31)) ca.prm.iter_limit = ctx->iter_host + (1LL << 31);
    // the same expressions as check_decide (admm_kernels.cuh), evaluated once
    ca.thr_hi = ctx->params.hi_ratio * ctx->params.r_bar / ctx->params.sigma_bar;
    ca.thr_lo = ctx->params.lo_ratio * ctx->params.r_bar / ctx->params.sigma_bar;
    // epochs and check counts restart every call: clear the publication buffers, key
    // sets and counter (contiguous in the workspace)
    CKC(cudaMemsetAsync(ctx->ws + ctx->L.pub2, 0, ctx->L.cnt2 + 16 - ctx->L.pub2, ctx->stream));
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem) != cudaSuccess)
        return fail(ctx, ADMM_ERR_CUDA, "cluster kernel: shared memory attribute");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)pl.G);
    cfg.blockDim = dim3((unsigned)(32 * pl.NW));
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)pl.T;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    void* args[2] = {(void*)&ctx->ka, (void*)&ca};
    CKC(cudaLaunchKernelExC(&cfg, fn, args));
    ctx->launches += 1;  // the cluster kernel (the memset is not a kernel of ours)
    return ADMM_OK;
}

// run until done or iter_limit, through the graph
admm_status run_loop(admm_ctx* ctx, long long iter_limit, int stop_on_conv) {
    if (!ctx->has_problem) return fail(ctx, ADMM_ERR_STATE, "set_problem must be called first");
    admm_status st = ADMM_OK;
    PPlan pl, cpl;
    C2Plan c2pl;
    persist_fn pfn = nullptr;
    cluster_fn cfn = nullptr;
    const void* c2fn = nullptr;
    if (ctx->params.exec_mode != ADMM_EXEC_STREAMING) {
        const char* gm = getenv("ADMM_PERSIST_GRID");  // force the grid-barrier variant
        if (!(gm && gm[0] == '1')) {
            // default: the message-passing cluster engine (admm_onchip2.cuh);
            // ADMM_CLUSTER_V=1: the barrier-based one (admm_onchip.cuh)
            // default: the message-passing engine when its plan gives every bulk thread one
            // cell (PHEV q <= ~75, toy); with several cells per thread the barrier engine
            // measured faster (PHEV q = 100: 5.95 vs 7.18 us per iteration, profiles/r02g) and
            // is taken when it fits.  ADMM_CLUSTER_V=1 / 2 (or a forced shape) pick one.
            const char* cv = getenv("ADMM_CLUSTER_V");
            const bool force1 = cv && cv[0] == '1';
            const bool force2 = (cv && cv[0] == '2') || getenv("ADMM_CLUSTER_T") || getenv("ADMM_CLUSTER_WARPS");
            if (!force1) {
                c2fn = cluster2_pick(ctx->m, ctx->params.box_mode);
                c2pl = plan_cluster2(ctx, c2fn);
            }
            if (force1 || (!force2 && (!c2pl.ok || c2pl.k >= 2))) {
                cfn = pick_cluster(ctx->m, ctx->params.box_mode);
                cpl = plan_cluster(ctx, cfn);
                if (cpl.ok) c2pl.ok = false;
            }
        }
        if (!cpl.ok && !c2pl.ok) {
            pfn = pick_persist(ctx->m, ctx->params.box_mode);
            pl = plan_persist(ctx, pfn);
        }
        if (!pl.ok && !cpl.ok && !c2pl.ok && ctx->params.exec_mode == ADMM_EXEC_PERSISTENT)
            return fail(ctx, ADMM_ERR_INVALID, "problem does not fit the persistent engine");
    }
    if (!pl.ok && !cpl.ok && !c2pl.ok) {
        st = build_graph(ctx);
        if (st != ADMM_OK) return st;
        if (ctx->hz && !ctx->use_tma)
            return fail(ctx, ADMM_ERR_INVALID,
                        "horizon blocks need the TMA sweep: finite boxes and m <= 4");
    }
    ctx->last_engine = c2pl.ok ? ADMM_ENGINE_CLUSTER_MSG : cpl.ok ? ADMM_ENGINE_CLUSTER
                              : (pl.ok ? ADMM_ENGINE_GRID
                                       : (ctx->use_tma ? ADMM_ENGINE_STREAM_TMA : ADMM_ENGINE_STREAM));
    upload_params(ctx, iter_limit, stop_on_conv);
    clear_done_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ka);
    ctx->launches += 1;
    const long long start = ctx->iter_host;
    long long graph_bodies = 0;
    CKC(cudaEventRecord(ctx->e0, ctx->stream));
    if (c2pl.ok) {
        st = launch_cluster2(ctx, c2fn, c2pl);
        if (st != ADMM_OK) return st;
        while (iter_limit - ctx->iter_host > (1LL << 31)) {  // more than one launch's epochs
            st = read_ctrl(ctx);
            if (st != ADMM_OK) return st;
            if (ctx->h_ctrl->done || ctx->iter_host >= iter_limit) break;
            st = launch_cluster2(ctx, c2fn, c2pl);
            if (st != ADMM_OK) return st;
        }
    } else if (cpl.ok) {
        st = launch_cluster(ctx, cfn, cpl);
        if (st != ADMM_OK) return st;
    } else if (pl.ok) {
        st = launch_persist(ctx, pfn, pl);
        if (st != ADMM_OK) return st;
    } else if (ctx->no_graph) {
        // profiling mode (ADMM_NO_GRAPH=1): plain launches, host polls per body
        sweep_fn fn = pick_sweep(ctx->m, ctx->params.box_mode, use_fx_sweep(ctx), ctx->coeff_bits == 32, use_pf_sweep(ctx), ctx->cpt, ctx->rl);
        while (true) {
            st = record_body(ctx, fn, ctx->stream);
            if (st != ADMM_OK) return st;
            ctx->launches += (long long)std::max(1, ctx->params.check_every) * (ctx->dist ? 2 : 1);
            st = read_ctrl(ctx);
            if (st != ADMM_OK) return st;
            if (ctx->h_ctrl->done || ctx->iter_host >= iter_limit) break;
        }
    } else if (!ctx->dist) {
        CKC(cudaGraphLaunch(ctx->gexec, ctx->stream));
        graph_bodies = -1;  // counted after the call from the iterations done
    } else {
        const int K = std::max(1, ctx->params.check_every);
        while (true) {
            CKC(cudaGraphLaunch(ctx->gexec, ctx->stream));
            ++graph_bodies;
            st = read_ctrl(ctx);
            if (st != ADMM_OK) return st;
            if (ctx->h_ctrl->done || ctx->iter_host >= iter_limit) break;
            (void)K;
        }
    }
    CKC(cudaEventRecord(ctx->e1, ctx->stream));
    st = read_ctrl(ctx);
    if (st != ADMM_OK) return st;
    float ms = 0.f;
    CKC(cudaEventElapsedTime(&ms, ctx->e0, ctx->e1));
    ctx->t_call_ms = ms;
    const long long did = ctx->iter_host - start;
    ctx->t_sweep_ms = did > 0 ? ms / (double)did : 0.0;
    {
        const long long K = std::max(1, ctx->params.check_every);
        if (graph_bodies < 0) graph_bodies = std::max(1LL, (did + K - 1) / K);  // while-node passes
        ctx->launches += graph_bodies * (K * (ctx->dist ? 2 : 1) + (ctx->dist ? 0 : 1));
    }
    if (ctx->h_ctrl->err) return fail(ctx, ADMM_ERR_NUMERICAL, "NaN/Inf in residuals");
    return ADMM_OK;
}

void fill_info(admm_ctx* ctx, admm_info* info) {
    if (!info) return;
    info->iterations = ctx->iter_host;
    info->r = ctx->h_ctrl->r;
    info->sigma = ctx->h_ctrl->sigma;
    for (int l = 0; l < 4; ++l) info->rho[l] = ctx->h_ctrl->rho[l];
    info->status = ctx->h_ctrl->status ? ADMM_OK : ADMM_NOT_CONVERGED;
    info->checks = ctx->h_ctrl->checks;
}

admm_status compute_objective(admm_ctx* ctx, double* out) {
    const long long R = (long long)ctx->m * ctx->q;
    obj_rows_kernel<<<(unsigned)R, 256, 0, ctx->stream>>>(ctx->ka, ctx->obj_rows);
    obj_sum_kernel<<<1, 32, 0, ctx->stream>>>(R, ctx->obj_rows, ctx->ka.xsend);
    ctx->launches += 2;
    CKC(cudaGetLastError());
    double tot = 0.0;
    if (ctx->dist) {
        CKN(ncclAllGather(ctx->ka.xsend, ctx->ka.xall, XB, ncclDouble, ctx->comm, ctx->stream));
        std::vector<double> all((size_t)ctx->world * XB);
        CKC(cudaMemcpyAsync(all.data(), ctx->ka.xall, all.size() * 8, cudaMemcpyDeviceToHost,
                            ctx->stream));
        CKC(cudaStreamSynchronize(ctx->stream));
        for (int r = 0; r < ctx->world; ++r) tot += all[(size_t)r * XB];
    } else {
        CKC(cudaMemcpyAsync(&tot, ctx->ka.xsend, 8, cudaMemcpyDeviceToHost, ctx->stream));
        CKC(cudaStreamSynchronize(ctx->stream));
    }
    *out = tot / (double)ctx->q_total;
    return ADMM_OK;
}

// copy a dense [rows][n] block (host or device) into a padded [rows][n_pad] array
admm_status put_rows(admm_ctx* ctx, double* dst, const double* src, long long rows) {
    if (rows == 0) return ADMM_OK;
    CKC(cudaMemcpy2DAsync(dst, ctx->n_pad * 8, src, ctx->n * 8, ctx->n * 8, rows, cudaMemcpyDefault,
                          ctx->stream));
    return ADMM_OK;
}

const char* kind_msg(int kind) {
    switch (kind) {
        case 1: return "non-finite coefficient";
        case 2: return "nonconvex cost (a2 < 0)";
        case 3: return "nonconvex loss (b2 < 0)";
        case 4: return "inverted or NaN bounds";
        case 5: return "non-finite demand y";
        case 6: return "NaN capacity c";
    }
    return "invalid";
}

// initial state from the current problem (reading G19)
admm_status init_state(admm_ctx* ctx) {
    KArgs& a = ctx->ka;
    const long long R = (long long)ctx->m * ctx->q;
    init_cells_kernel<<<grid_for(ctx->q * ctx->n_pad, 256, ctx->sms), 256, 0, ctx->stream>>>(a);
    double* rs = (double*)(ctx->ws + ctx->L.hzrow);  // [2][m][q]: sum_k g(x), sum_k b0
    init_rows_kernel<<<(unsigned)R, 256, 0, ctx->stream>>>(a, rs);
    CKC(cudaGetLastError());
    if (ctx->hz) CKN(ncclAllReduce(rs, rs, (size_t)2 * R, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    init_rows_fin_kernel<<<grid_for(R, 256, ctx->sms), 256, 0, ctx->stream>>>(a, rs);
    cons_partial_kernel<<<1, 32, 0, ctx->stream>>>(a, 0);
    CKC(cudaGetLastError());
    const double* agg = a.xsend;
    if (ctx->dist) {
        CKN(ncclAllGather(a.xsend, a.xall, XB, ncclDouble, ctx->comm, ctx->stream));
        agg = a.xall;
    }
    ctx->launches += 5;  // init_cells, init_rows, init_rows_fin, cons_partial, init_ctrl
    init_ctrl_kernel<<<1, 32, 0, ctx->stream>>>(a, agg, ctx->world, ctx->params.rho[0],
                                                 ctx->params.rho[1], ctx->params.rho[2],
                                                 ctx->params.rho[3]);
    CKC(cudaMemsetAsync(a.row_cnt, 0, (size_t)ctx->q * 4, ctx->stream));
    CKC(cudaMemsetAsync(a.hist, 0, (size_t)HIST_CAP * HCOLS * 8, ctx->stream));
    CKC(cudaGetLastError());
    return ADMM_OK;
}

}  // namespace

extern "C" {

void admm_default_params(admm_params* out) {
    if (!out) return;
    // PAPER.md:317-324, :353
    out->rho[0] = 1e-4;
    out->rho[1] = 2e-6;
    out->rho[2] = 5e-6;
    out->rho[3] = 5e-6;
    out->tau = 1.1;
    out->hi_ratio = 1.2;
    out->lo_ratio = 0.8;
    out->r_bar = 1e-6;
    out->sigma_bar = 1e-2;
    out->check_every = 10;
    out->adapt_rho = 1;
    out->rescale_duals = 1;
    out->box_mode = ADMM_BOX_PROJECT;
    out->exec_mode = ADMM_EXEC_AUTO;
}

size_t admm_workspace_bytes(int32_t m, int64_t n, int64_t q_local, int32_t device) {
    if (m <= 0 || n <= 0 || q_local <= 0) return 0;
    int sms = 148;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
        cudaGetLastError();
        sms = 148;
    }
    return make_layout(m, n, q_local, sms).total;
}

admm_status admm_nccl_unique_id(unsigned char out[128]) {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return ADMM_ERR_NCCL;
    static_assert(sizeof(id.internal) == 128, "nccl id size");
    memcpy(out, id.internal, 128);
    return ADMM_OK;
}

admm_status admm_create(admm_ctx** out, int32_t m, int64_t n, int64_t q_total, const admm_dist* dist,
                        int32_t device, void* workspace, size_t workspace_bytes, void* cuda_stream) {
    if (!out) return ADMM_ERR_INVALID;
    *out = nullptr;
    if (m < 1 || m > 4 || n < 1 || q_total < 1) return ADMM_ERR_INVALID;
    admm_ctx* ctx = new admm_ctx();
    ctx->m = m;
    ctx->n = n;
    ctx->n_total = n;
    ctx->q_total = q_total;
    ctx->q = q_total;
    ctx->device = device;
    if (dist) {
        if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world || dist->world > MAX_WORLD ||
            dist->j_begin < 0 || dist->j_end <= dist->j_begin || dist->j_end > q_total ||
            (dist->mode != ADMM_SHARD_SCENARIOS && dist->mode != ADMM_SHARD_HORIZON)) {
            delete ctx;
            return ADMM_ERR_INVALID;
        }
        ctx->dist = true;
        ctx->world = dist->world;
        ctx->rank = dist->rank;
        ctx->j0 = dist->j_begin;
        ctx->q = dist->j_end - dist->j_begin;
        if (dist->mode == ADMM_SHARD_HORIZON) {
            // every scenario, steps [k_begin, k_end) of the horizon
            if (dist->j_begin != 0 || dist->j_end != q_total || dist->k_begin < 0 ||
                dist->k_end <= dist->k_begin || dist->k_end > n) {
                delete ctx;
                return ADMM_ERR_INVALID;
            }
            ctx->hz = true;
            ctx->k_begin = dist->k_begin;
            ctx->n = dist->k_end - dist->k_begin;
        }
    }
    ctx->n_pad = (long long)align_up((size_t)ctx->n, 4);
    n = ctx->n;  // local horizon from here on
    admm_status st = ADMM_OK;
    auto bail = [&](admm_status s) {
        *out = ctx;  // keep ctx so the caller can read admm_last_error, then destroy it
        return s;
    };
    if (cudaSetDevice(device) != cudaSuccess) return bail(fail(ctx, ADMM_ERR_CUDA, "cudaSetDevice"));
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
    ctx->stream = (cudaStream_t)cuda_stream;
    ctx->L = make_layout(m, n, ctx->q, ctx->sms);
    if (workspace) {
        if (workspace_bytes < ctx->L.total)
            return bail(fail(ctx, ADMM_ERR_INVALID, "workspace too small"));
        if (((uintptr_t)workspace) % 256 != 0)
            return bail(fail(ctx, ADMM_ERR_INVALID, "workspace must be 256-byte aligned"));
        ctx->ws = (char*)workspace;
    } else {
        if (cudaMalloc(&ctx->ws, ctx->L.total) != cudaSuccess)
            return bail(fail(ctx, ADMM_ERR_CUDA, "cudaMalloc workspace"));
        ctx->owns_ws = true;
    }
    ctx->ws_bytes = ctx->L.total;
    if (cudaMemsetAsync(ctx->ws, 0, ctx->L.total, ctx->stream) != cudaSuccess)
        return bail(fail(ctx, ADMM_ERR_CUDA, "memset workspace"));
    if (cudaMallocHost(&ctx->h_ctrl, sizeof(Ctrl)) != cudaSuccess ||
        cudaMallocHost(&ctx->h_iter, 8) != cudaSuccess)
        return bail(fail(ctx, ADMM_ERR_CUDA, "cudaMallocHost"));
    memset(ctx->h_ctrl, 0, sizeof(Ctrl));
    cudaEventCreate(&ctx->e0);
    cudaEventCreate(&ctx->e1);
    if (cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(ctx, ADMM_ERR_CUDA, "cudaStreamCreate"));
    admm_default_params(&ctx->params);
    {
        const char* ng = getenv("ADMM_NO_GRAPH");
        ctx->no_graph = ng && ng[0] == '1';
    }
    // kernel arguments
    const Layout& L = ctx->L;
    KArgs& a = ctx->ka;
    {
        // 4 cells per thread staged through shared memory (ADMM_SWEEP_CPT=4, m <= 2) is opt-in:
        // it beat the two-cell CTA at q = 1e5 (46 vs 43 %) but the row loop below supersedes it
        // for many rows, and at few rows the two-cell CTA is as fast (profiles/r01d, r01f)
        const char* e = getenv("ADMM_SWEEP_CPT");
        ctx->cpt = (e && e[0] == '4' && m <= 2) ? 4 : 2;
        // row loop (128-thread CTAs own whole rows; 4 per SM): the default for m <= 2 when
        // there are rows for every CTA (q >= 4 x SMs): q = 1e4 / 1e5 at 54 / 56 % of the
        // HBM peak vs 44 / 46 % (profiles/r01e).  ADMM_SWEEP_RL = 0 off, 1 force, 6 = 64 threads
        const char* r = getenv("ADMM_SWEEP_RL");
        if (r) ctx->rl = (m <= 2) ? (r[0] == '1' ? 128 : (r[0] == '6' ? 64 : 0)) : 0;
        else ctx->rl = (m <= 2 && ctx->q >= 4LL * ctx->sms) ? 128 : 0;
        if (ctx->rl) ctx->cpt = 2;
    }
    ctx->bs = ctx->rl ? (int)std::min<long long>(ctx->rl, ((n + 1) / 2 + 31) / 32 * 32) : pick_bs(n, ctx->cpt);
    ctx->tile = ctx->bs * ctx->cpt;
    ctx->T = (int)((n + ctx->tile - 1) / ctx->tile);
    a.m = m;
    a.n = (int)n;
    a.n_pad = (int)ctx->n_pad;
    a.T = ctx->T;
    a.tile = ctx->tile;
    a.G = 1;
    a.world = ctx->world;
    a.rank = ctx->rank;
    a.dist = ctx->dist ? 1 : 0;
    a.hz = ctx->hz ? 1 : 0;
    a.k0own = (!ctx->hz || ctx->k_begin == 0) ? 1 : 0;
    a.nd = (double)ctx->n_total;
    a.q = ctx->q;
    a.q_total = q_total;
    a.inv_q = 1.0 / (double)q_total;
    char* w = ctx->ws;
    a.a2 = (double*)(w + L.a2); a.a1 = (double*)(w + L.a1); a.a0 = (double*)(w + L.a0);
    a.b2 = (double*)(w + L.b2); a.b1 = (double*)(w + L.b1); a.b0 = (double*)(w + L.b0);
    a.lo = (double*)(w + L.lo); a.hi = (double*)(w + L.hi); a.y = (double*)(w + L.y);
    a.c = (double*)(w + L.c); a.sb0 = (double*)(w + L.sb0);
    a.x = (double*)(w + L.x); a.v = (double*)(w + L.v);
    a.lam = (double*)(w + L.lam); a.zeta = (double*)(w + L.zeta); a.h = (double*)(w + L.h);
    a.p = (double*)(w + L.p); a.nu = (double*)(w + L.nu);
    a.cta_part = (double*)(w + L.cta_part); a.row_part = (double*)(w + L.row_part);
    a.row_cnt = (int*)(w + L.row_cnt); a.glob_cnt = (int*)(w + L.glob_cnt);
    a.xsend = (double*)(w + L.xsend); a.xall = (double*)(w + L.xall);
    a.ctrl = (Ctrl*)(w + L.ctrl); a.iter = (long long*)(w + L.iter);
    a.prm = (const DParams*)(w + L.prm);
    a.hist = (double*)(w + L.hist); a.hist_cap = HIST_CAP;
    a.rowacc = (unsigned long long*)(w + L.rowacc);
    a.rowdg = (unsigned long long*)(w + L.rowdg);
    a.rowcnt = (unsigned*)(w + L.rowcnt);
    a.hzdg = (unsigned long long*)(w + L.hzdg);
    {
        const size_t NE = (size_t)m * ctx->q * ctx->n_pad;
        float* cf = (float*)(w + L.cf);
        a.fa2 = cf; a.fa1 = cf + NE; a.fb2 = cf + 2 * NE; a.fb1 = cf + 3 * NE;
    }
    ctx->vflag = (unsigned long long*)(w + L.vflag);
    ctx->obj_rows = (double*)(w + L.obj_rows);
    if (ctx->dist) {
        ncclUniqueId id;
        memcpy(id.internal, dist->nccl_id, 128);
        ncclResult_t r = ncclCommInitRank(&ctx->comm, ctx->world, id, ctx->rank);
        if (r != ncclSuccess)
            return bail(fail(ctx, ADMM_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)));
    }
    *out = ctx;
    return st;
}

admm_status admm_set_problem(admm_ctx* ctx, const double* f, const double* g, const double* lo,
                             const double* hi, const double* y, const double* c,
                             int32_t on_device) {
    if (!ctx) return ADMM_ERR_INVALID;
    if (!f || !g || !lo || !hi || !y || !c) return fail(ctx, ADMM_ERR_INVALID, "null argument");
    (void)on_device;  // cudaMemcpyDefault resolves host vs device pointers (UVA)
    CKC(cudaSetDevice(ctx->device));
    KArgs& a = ctx->ka;
    const long long R = (long long)ctx->m * ctx->q;
    const size_t blk = (size_t)R * ctx->n;
    double* fd[3] = {(double*)a.a2, (double*)a.a1, (double*)a.a0};
    double* gd[3] = {(double*)a.b2, (double*)a.b1, (double*)a.b0};
    admm_status st;
    for (int t = 0; t < 3; ++t) {
        if ((st = put_rows(ctx, fd[t], f + t * blk, R)) != ADMM_OK) return st;
        if ((st = put_rows(ctx, gd[t], g + t * blk, R)) != ADMM_OK) return st;
    }
    if ((st = put_rows(ctx, (double*)a.lo, lo, ctx->m)) != ADMM_OK) return st;
    if ((st = put_rows(ctx, (double*)a.hi, hi, ctx->m)) != ADMM_OK) return st;
    if ((st = put_rows(ctx, (double*)a.y, y, ctx->q)) != ADMM_OK) return st;
    CKC(cudaMemcpyAsync((double*)a.c, c, ctx->m * 8, cudaMemcpyDefault, ctx->stream));
    // validation (Assumption 1, bounds, finiteness)
    CKC(cudaMemsetAsync(ctx->vflag, 0xff, 8, ctx->stream));
    validate_kernel<<<grid_for(blk, 256, ctx->sms), 256, 0, ctx->stream>>>(
        ctx->m, ctx->q, ctx->n, ctx->n_pad, a.a2, a.a1, a.a0, a.b2, a.b1, a.b0, a.lo, a.hi, a.y,
        a.c, ctx->vflag);
    CKC(cudaGetLastError());
    unsigned long long code = 0;
    CKC(cudaMemcpyAsync(&code, ctx->vflag, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CKC(cudaStreamSynchronize(ctx->stream));
    if (code != ~0ull) {
        ctx->has_problem = false;
        const int kind = (int)(code >> 56);
        const long long t = (long long)(code & ((1ull << 56) - 1));
        char buf[160];
        if (kind <= 3) {
            const long long k = t % ctx->n, j = (t / ctx->n) % ctx->q, i = t / ctx->n / ctx->q;
            snprintf(buf, sizeof buf, "%s at (i=%lld,j=%lld,k=%lld)", kind_msg(kind), i, j + ctx->j0, k);
        } else if (kind == 4) {
            snprintf(buf, sizeof buf, "%s at (i=%lld,k=%lld)", kind_msg(kind), t / ctx->n, t % ctx->n);
        } else if (kind == 5) {
            snprintf(buf, sizeof buf, "%s at (j=%lld,k=%lld)", kind_msg(kind), t / ctx->n + ctx->j0, t % ctx->n);
        } else {
            snprintf(buf, sizeof buf, "%s at (i=%lld)", kind_msg(kind), t);
        }
        return fail(ctx, (kind == 2 || kind == 3) ? ADMM_ERR_NONCONVEX : ADMM_ERR_INVALID, buf);
    }
    // F2: coefficients stored in fp32 -- every engine then solves the problem whose
    // a2, a1, b2, b1 are the fp32-rounded inputs (double arrays rounded in place, fp32
    // copies for the streaming sweep); a0, b0, bounds, demand stay fp64
    if (ctx->coeff_bits == 32) {
        const long long NE = (long long)ctx->m * ctx->q * ctx->n_pad;
        round_coeff_kernel<<<grid_for(NE, 256, ctx->sms), 256, 0, ctx->stream>>>(
            NE, (double*)a.a2, (double*)a.a1, (double*)a.b2, (double*)a.b1, (float*)a.fa2,
            (float*)a.fa1, (float*)a.fb2, (float*)a.fb1);
        CKC(cudaGetLastError());
    }
    // fixed-point scales of the row sums (every engine), prepared constants (on-chip engine)
    ctx->prep_ok = false;
    ctx->fx_ok = false;
    ctx->graph_dirty = true;
    {
        unsigned long long* gb = (unsigned long long*)(ctx->ws + ctx->L.gbound);
        CKC(cudaMemsetAsync(gb, 0, MAXM * 8, ctx->stream));
        gbound_kernel<<<grid_for(blk, 256, ctx->sms), 256, 0, ctx->stream>>>(
            ctx->m, ctx->q, ctx->n, ctx->n_pad, a.b2, a.b1, a.lo, a.hi, gb);
        CKC(cudaGetLastError());
        // one fixed-point scale per source on every rank (horizon blocks: the bound of
        // the whole row; scenario shards: identical scales keep the sums exact alike)
        if (ctx->dist) CKN(ncclAllReduce(gb, gb, MAXM, ncclUint64, ncclMax, ctx->comm, ctx->stream));
        rowdg_init_kernel<<<grid_for(ctx->q * 2 * MAXM, 256, ctx->sms), 256, 0, ctx->stream>>>(
            (unsigned long long*)(ctx->ws + ctx->L.rowdg), ctx->q);
        CKC(cudaGetLastError());
        unsigned long long keys[MAXM];
        CKC(cudaMemcpyAsync(keys, gb, MAXM * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CKC(cudaStreamSynchronize(ctx->stream));
        bool ok = true;
        ctx->ka.gfree = 0u;
        for (int i = 0; i < ctx->m; ++i) {
            const unsigned long long k = keys[i];
            unsigned long long u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
            double gbv;
            std::memcpy(&gbv, &u, 8);
            const double G = (double)ctx->n_total * gbv;  // bound on |sum_k (b2 x^2 + b1 x)|
            if (!(G < 1e300)) {
                ok = false;
                break;
            }
            int E = 0;
            if (G > 0.0) E = 62 - (int)std::ceil(std::log2(G));
            else ctx->ka.gfree |= 1u << i;
            E = std::max(-1000, std::min(1000, E));
            ctx->fx_scale[i] = std::ldexp(1.0, E);
            ctx->fx_inv[i] = std::ldexp(1.0, -E);
        }
        ctx->fx_ok = ok;
        for (int i = 0; i < MAXM; ++i) {
            ctx->ka.fx_scale[i] = ok ? ctx->fx_scale[i] : 0.0;
            ctx->ka.fx_inv[i] = ok ? ctx->fx_inv[i] : 0.0;
        }
    }
    if (ctx->fx_ok && (size_t)ctx->m * ctx->q * ctx->n_pad <= ONCHIP_PREP_MAX_ELEMS) {
        const long long NE = (long long)ctx->m * ctx->q * ctx->n_pad;
        prep_kernel<<<grid_for(NE, 256, ctx->sms), 256, 0, ctx->stream>>>(
            NE, a.b2, a.b1, (double*)(ctx->ws + ctx->L.bq), (double*)(ctx->ws + ctx->L.ib2s));
        CKC(cudaGetLastError());
        ctx->prep_ok = true;
    }
    admm_status is = init_state(ctx);
    if (is != ADMM_OK) return is;
    ctx->has_problem = true;
    admm_status rs = read_ctrl(ctx);
    if (rs != ADMM_OK) return rs;
    ctx->err.clear();
    return ADMM_OK;
}

admm_status admm_reset(admm_ctx* ctx) {
    if (!ctx) return ADMM_ERR_INVALID;
    if (!ctx->has_problem) return fail(ctx, ADMM_ERR_STATE, "no problem set");
    CKC(cudaSetDevice(ctx->device));
    admm_status st = init_state(ctx);
    if (st != ADMM_OK) return st;
    return read_ctrl(ctx);
}

admm_status admm_set_params(admm_ctx* ctx, const admm_params* p) {
    if (!ctx || !p) return ADMM_ERR_INVALID;
    for (int l = 0; l < 4; ++l)
        if (!(p->rho[l] > 0.0)) return fail(ctx, ADMM_ERR_INVALID, "rho must be > 0");
    if (!(p->tau >= 1.0) || p->check_every < 1 || !(p->r_bar > 0) || !(p->sigma_bar > 0) ||
        (p->box_mode != 0 && p->box_mode != 1) || p->exec_mode < 0 || p->exec_mode > 2)
        return fail(ctx, ADMM_ERR_INVALID, "bad parameters");
    const bool rebuild = p->check_every != ctx->params.check_every;
    ctx->params = *p;
    if (rebuild && ctx->gexec) {
        cudaGraphExecDestroy(ctx->gexec);
        ctx->gexec = nullptr;
        ctx->graph_mode = -1;
    }
    if (ctx->has_problem) {
        // rho takes effect on the next iteration: write it into the current control block
        const long long it = ctx->iter_host;
        CKC(cudaMemcpyAsync((char*)(ctx->ka.ctrl + (it & 1)) + offsetof(Ctrl, rho), p->rho,
                            4 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CKC(cudaStreamSynchronize(ctx->stream));
    }
    return ADMM_OK;
}

admm_status admm_get_params(const admm_ctx* ctx, admm_params* out) {
    if (!ctx || !out) return ADMM_ERR_INVALID;
    *out = ctx->params;
    return ADMM_OK;
}

admm_status admm_iterate(admm_ctx* ctx, int64_t iters) {
    if (!ctx || iters < 0) return ADMM_ERR_INVALID;
    if (iters == 0) return ADMM_OK;
    CKC(cudaSetDevice(ctx->device));
    return run_loop(ctx, ctx->iter_host + iters, 0);
}

admm_status admm_solve(admm_ctx* ctx, double r_bar, double sigma_bar, int64_t max_iter,
                       admm_info* info) {
    if (!ctx || !(r_bar > 0) || !(sigma_bar > 0) || max_iter < 0) return ADMM_ERR_INVALID;
    CKC(cudaSetDevice(ctx->device));
    ctx->params.r_bar = r_bar;
    ctx->params.sigma_bar = sigma_bar;
    admm_status st = run_loop(ctx, ctx->iter_host + max_iter, 1);
    if (st != ADMM_OK) return st;
    fill_info(ctx, info);
    if (info) {
        st = compute_objective(ctx, &info->objective);
        if (st != ADMM_OK) return st;
    }
    return ctx->h_ctrl->status ? ADMM_OK : ADMM_NOT_CONVERGED;
}

admm_status admm_get_solution(admm_ctx* ctx, double* x, double* x1, admm_info* info,
                              int32_t on_device) {
    if (!ctx) return ADMM_ERR_INVALID;
    if (!ctx->has_problem) return fail(ctx, ADMM_ERR_STATE, "no problem set");
    (void)on_device;
    CKC(cudaSetDevice(ctx->device));
    if (x)
        CKC(cudaMemcpy2DAsync(x, ctx->n * 8, ctx->ka.x, ctx->n_pad * 8, ctx->n * 8,
                              (size_t)ctx->m * ctx->q, cudaMemcpyDefault, ctx->stream));
    admm_status st = read_ctrl(ctx);
    if (st != ADMM_OK) return st;
    if (x1) CKC(cudaMemcpyAsync(x1, ctx->h_ctrl->x1, ctx->m * 8, cudaMemcpyDefault, ctx->stream));
    if (info) {
        fill_info(ctx, info);
        st = compute_objective(ctx, &info->objective);
        if (st != ADMM_OK) return st;
    }
    CKC(cudaStreamSynchronize(ctx->stream));
    return ADMM_OK;
}

admm_status admm_get_state(admm_ctx* ctx, double* x, double* z, double* lam, double* s, double* mu,
                           double* h, double* p, double* nu, double* x1, int32_t on_device) {
    if (!ctx) return ADMM_ERR_INVALID;
    if (!ctx->has_problem) return fail(ctx, ADMM_ERR_STATE, "no problem set");
    CKC(cudaSetDevice(ctx->device));
    const size_t E = (size_t)ctx->m * ctx->q * ctx->n, Cn = (size_t)ctx->q * ctx->n,
                 R = (size_t)ctx->m * ctx->q;
    double* outs[9] = {x, z, lam, s, mu, h, p, nu, x1};
    const size_t sz[9] = {E, E, E, Cn, Cn, R, R, R, (size_t)ctx->m};
    double* dev[9] = {nullptr};
    size_t tot = 0;
    for (int t = 0; t < 9; ++t)
        if (outs[t] && !on_device) tot += sz[t];
    double* tmp = nullptr;
    if (tot) CKC(cudaMallocAsync(&tmp, tot * 8, ctx->stream));
    size_t o = 0;
    for (int t = 0; t < 9; ++t) {
        if (!outs[t]) continue;
        if (on_device) {
            dev[t] = outs[t];
        } else {
            dev[t] = tmp + o;
            o += sz[t];
        }
    }
    materialize_kernel<<<grid_for(E, 256, ctx->sms), 256, 0, ctx->stream>>>(
        ctx->ka, dev[0], dev[1], dev[2], dev[3], dev[4], dev[5], dev[6], dev[7], dev[8]);
    CKC(cudaGetLastError());
    if (!on_device)
        for (int t = 0; t < 9; ++t)
            if (outs[t])
                CKC(cudaMemcpyAsync(outs[t], dev[t], sz[t] * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (tmp) CKC(cudaFreeAsync(tmp, ctx->stream));
    CKC(cudaStreamSynchronize(ctx->stream));
    return ADMM_OK;
}

admm_status admm_set_state(admm_ctx* ctx, const double* x, const double* z, const double* lam,
                           const double* s, const double* mu, const double* h, const double* p,
                           const double* nu, const double* x1, int32_t on_device) {
    if (!ctx) return ADMM_ERR_INVALID;
    if (!ctx->has_problem) return fail(ctx, ADMM_ERR_STATE, "no problem set");
    if (!x || !z || !lam || !s || !mu || !h || !p || !nu || !x1)
        return fail(ctx, ADMM_ERR_INVALID, "null argument");
    CKC(cudaSetDevice(ctx->device));
    const size_t E = (size_t)ctx->m * ctx->q * ctx->n, Cn = (size_t)ctx->q * ctx->n,
                 R = (size_t)ctx->m * ctx->q;
    const double* ins[9] = {x, z, lam, s, mu, h, p, nu, x1};
    const size_t sz[9] = {E, E, E, Cn, Cn, R, R, R, (size_t)ctx->m};
    size_t tot = 0;
    for (int t = 0; t < 9; ++t) tot += sz[t];
    double* tmp = nullptr;
    CKC(cudaMallocAsync(&tmp, tot * 8, ctx->stream));
    const double* dev[9];
    size_t o = 0;
    for (int t = 0; t < 9; ++t) {
        CKC(cudaMemcpyAsync(tmp + o, ins[t], sz[t] * 8, cudaMemcpyDefault, ctx->stream));
        dev[t] = tmp + o;
        o += sz[t];
    }
    (void)on_device;
    CKC(cudaMemsetAsync(ctx->vflag, 0xff, 8, ctx->stream));
    compress_kernel<<<grid_for(E, 256, ctx->sms), 256, 0, ctx->stream>>>(
        ctx->ka, dev[0], dev[1], dev[2], dev[3], dev[4], dev[5], dev[6], dev[7], ctx->vflag);
    set_ctrl_kernel<<<1, 1, 0, ctx->stream>>>(ctx->ka, dev[8]);
    CKC(cudaGetLastError());
    unsigned long long code = 0;
    CKC(cudaMemcpyAsync(&code, ctx->vflag, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CKC(cudaFreeAsync(tmp, ctx->stream));
    CKC(cudaStreamSynchronize(ctx->stream));
    if (code != ~0ull) {
        const int kind = (int)(code >> 56);
        const char* what = kind == 1 ? "lambda varies over k" : kind == 2 ? "z - g(x) varies over k"
                         : kind == 3 ? "s * mu != 0 or negative" : "x outside its box";
        return fail(ctx, ADMM_ERR_STATE, std::string("state not representable: ") + what);
    }
    return read_ctrl(ctx);
}

int64_t admm_get_history(admm_ctx* ctx, double* out, int64_t max_rows) {
    if (!ctx || !out || max_rows <= 0 || !ctx->has_problem) return 0;
    if (read_ctrl(ctx) != ADMM_OK) return 0;
    const long long nrec = ctx->h_ctrl->checks;
    const long long avail = std::min<long long>(nrec, HIST_CAP);
    const long long take = std::min<long long>(avail, max_rows);
    std::vector<double> all((size_t)HIST_CAP * HCOLS);
    if (cudaMemcpy(all.data(), ctx->ka.hist, all.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
        return 0;
    for (long long r = 0; r < take; ++r) {
        const long long idx = (nrec - take + r) % HIST_CAP;
        memcpy(out + r * HCOLS, all.data() + idx * HCOLS, HCOLS * 8);
    }
    return take;
}

admm_status admm_get_engine(const admm_ctx* ctx, int32_t* engine, int64_t* launches) {
    if (!ctx) return ADMM_ERR_INVALID;
    if (engine) *engine = ctx->last_engine;
    if (launches) *launches = ctx->launches;
    return ADMM_OK;
}

admm_status admm_set_coeff_precision(admm_ctx* ctx, int32_t bits) {
    if (!ctx) return ADMM_ERR_INVALID;
    if (bits != 64 && bits != 32) return fail(ctx, ADMM_ERR_INVALID, "coefficient precision must be 64 or 32");
    if (bits != ctx->coeff_bits) {
        ctx->coeff_bits = bits;
        ctx->has_problem = false;  // the loaded problem was stored in the other precision
        ctx->graph_dirty = true;
    }
    return ADMM_OK;
}

admm_status admm_get_coeff_precision(const admm_ctx* ctx, int32_t* bits) {
    if (!ctx || !bits) return ADMM_ERR_INVALID;
    *bits = ctx->coeff_bits;
    return ADMM_OK;
}

admm_status admm_get_timing(admm_ctx* ctx, double out[2]) {
    if (!ctx || !out) return ADMM_ERR_INVALID;
    out[0] = ctx->t_sweep_ms;
    out[1] = ctx->t_call_ms;
    return ADMM_OK;
}

const char* admm_last_error(const admm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void admm_destroy(admm_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    if (ctx->graph) cudaGraphDestroy(ctx->graph);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    if (ctx->owns_ws && ctx->ws) cudaFree(ctx->ws);
    if (ctx->h_ctrl) cudaFreeHost(ctx->h_ctrl);
    if (ctx->h_iter) cudaFreeHost(ctx->h_iter);
    if (ctx->e0) cudaEventDestroy(ctx->e0);
    if (ctx->e1) cudaEventDestroy(ctx->e1);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    delete ctx;
}

}  // extern "C"

namespace {
// per-device stream-ordered pool of the batch dispatch's decision words (release threshold
// = max: freed blocks stay in the pool, so an allocation per call costs no driver call)
cudaMemPool_t qb_pool(int dev) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    if (dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p;
        if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return nullptr;
        unsigned long long thr = ~0ull;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
        pools[dev] = p;
    }
    return pools[dev];
}
}  // namespace

extern "C" {

admm_status quartic_minimize_batch(const double* A, const double* B, const double* C,
                                   const double* D, const double* lo, const double* hi, double* x,
                                   int64_t N, int32_t box_mode, void* cuda_stream) {
    if (N < 0 || !A || !B || !C || !D || !x || (box_mode != 0 && box_mode != 1))
        return ADMM_ERR_INVALID;
    if (N == 0) return ADMM_OK;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto al = [](const void* p) { return p == nullptr || ((uintptr_t)p % 16) == 0; };
    const bool vec = (N % 2 == 0) && al(A) && al(B) && al(C) && al(D) && al(lo) && al(hi) && al(x);
    const int bs = 256;
    if (vec) {
        const long long N2 = N / 2;
        const int grid = (int)std::min<long long>((N2 + bs - 1) / bs, (long long)sms * 8);
        // default: sample the batch on the device and run the per-lane or the warp-compacted
        // kernel; ADMM_QB_WC=0 / 1 forces one of them (experiments)
        const char* wc = getenv("ADMM_QB_WC");
        if (wc && (wc[0] == '0' || wc[0] == '1')) {
            if (wc[0] == '1') {
                if (box_mode == 1) quartic_batch_wc_kernel<1><<<grid, QWC_NW * 32, 0, st>>>(A, B, C, D, lo, hi, x, N2);
                else quartic_batch_wc_kernel<0><<<grid, QWC_NW * 32, 0, st>>>(A, B, C, D, lo, hi, x, N2);
            } else if (box_mode == 1) {
                quartic_batch_vec_kernel<1><<<grid, bs, 0, st>>>(A, B, C, D, lo, hi, x, N2);
            } else {
                quartic_batch_vec_kernel<0><<<grid, bs, 0, st>>>(A, B, C, D, lo, hi, x, N2);
            }
        } else {
            // the decision word is a stream-ordered allocation private to this call, from a
            // library-owned pool that never trims (cheap reuse; calls on concurrent streams
            // cannot share a word)
            cudaMemPool_t pool = qb_pool(dev);
            if (!pool) return ADMM_ERR_CUDA;
            int* flag = nullptr;
            if (cudaMallocFromPoolAsync((void**)&flag, sizeof(int), pool, st) != cudaSuccess) return ADMM_ERR_CUDA;
            quartic_sample_kernel<<<1, 512, 0, st>>>(A, B, C, D, N, flag);
            if (box_mode == 1) {
                quartic_batch_vec_kernel<1><<<grid, bs, 0, st>>>(A, B, C, D, lo, hi, x, N2, flag);
                quartic_batch_wc_kernel<1><<<grid, QWC_NW * 32, 0, st>>>(A, B, C, D, lo, hi, x, N2, flag);
            } else {
                quartic_batch_vec_kernel<0><<<grid, bs, 0, st>>>(A, B, C, D, lo, hi, x, N2, flag);
                quartic_batch_wc_kernel<0><<<grid, QWC_NW * 32, 0, st>>>(A, B, C, D, lo, hi, x, N2, flag);
            }
            cudaFreeAsync(flag, st);
        }
    } else {
        const int grid = (int)std::min<long long>((N + bs - 1) / bs, (long long)sms * 8);
        if (box_mode == 1)
            quartic_batch_kernel<1><<<grid, bs, 0, st>>>(A, B, C, D, lo, hi, x, N);
        else
            quartic_batch_kernel<0><<<grid, bs, 0, st>>>(A, B, C, D, lo, hi, x, N);
    }
    return cudaGetLastError() == cudaSuccess ? ADMM_OK : ADMM_ERR_CUDA;
}

const char* admm_build_info(void) {
    return "libadmm_b200 (arXiv 1903.10041 ADMM hot path), sm_100a fp64, CUDA " 
#define STR2(x) #x
#define STR(x) STR2(x)
        STR(__CUDACC_VER_MAJOR__) "." STR(__CUDACC_VER_MINOR__);
}

}  // extern "C"

#ifdef ADMM_PHASE_PROF
extern "C" int admm_debug_phase(unsigned long long* out24) {
    return cudaMemcpyFromSymbol(out24, admm_dev::g_phase, sizeof(admm_dev::g_phase)) == cudaSuccess ? 0 : 1;
}
#endif
