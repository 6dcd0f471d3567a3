// admm_stream.cuh -- streaming ADMM sweep for problems that do not fit on chip
// (BASELINE.json configs[2] n >= 1e5, configs[3] q >= 1e3): one launch = one
// ADMM iteration (Appendix A, Eq. (6a)-(6i)), HBM-bound.
//
//  * persistent grid, one CTA per SM; the CTA walks its work units (row j,
//    segment of TPS tiles of TL cells) in a fixed order (deterministic);
//  * 1-D TMA bulk copies (cp.async.bulk, mbarrier complete_tx) feed a
//    3-stage shared-memory ring; the warp that releases a stage last (shared
//    counter) refills it with the tile NS ahead, so no warp ever waits for a
//    producer and the warps never meet at a block barrier inside the sweep:
//    HBM streams continuously under the fp64 work;
//  * one cell per thread: Gauss-Seidel over the sources in registers (6a),
//    (6e)/(6f) in-thread (identity I2), x and v written straight from
//    registers (coalesced);
//  * row sums sum_k (b2 x^2 + b1 x) in exact 64-bit fixed point (scale of
//    admm_onchip.cuh): warp redux.sync limbs into per-warp slots, the last
//    warp to arrive (shared counter) sums the slots and finalises the row;
//    rows split over CTAs (S > 1) add into global accumulators with an
//    arrival counter, the last segment finalising -- order-independent,
//    so deterministic;
//  * the next row's scalars (lam, zeta, nu) are prefetched one unit ahead;
//  * consensus / residual partials per CTA, reduced by the last CTA in CTA
//    order, which also runs the check and writes the next control block.
#pragma once
#include "admm_onchip.cuh"

namespace admm_dev {

template <int M>
struct StreamCfg {
    static constexpr int TL = (M <= 2) ? 512 : 256;  // cells per tile = threads per CTA
    static constexpr int NS = 3;                     // pipeline stages
    static constexpr int NSTREAM = 7 * M + 2;        // x a2 a1 b2 b1 lo hi per source, y, v
    static constexpr size_t SMEM = (size_t)NS * NSTREAM * TL * 8;
};

struct SArgs {
    int TL, TPR, S, TPS, U, G;             // tile length, tiles/row, segments/row, tiles/segment, units, grid
    double fx_scale[MAXM], fx_inv[MAXM];   // fixed-point scale of the row sums
    unsigned long long* rowacc;            // [q][MAXM] fixed-point row sums (S > 1), kept zero
    unsigned long long* rowdg;             // [q][2 MAXM] row max / min keys of dg (S > 1, checks)
    unsigned* rowcnt;                      // [q][MAXM] segment arrivals (S > 1), kept zero
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned phase) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// the CTA's tile sequence: units u = g, g+G, ...; tiles [s TPS, min(TPR, (s+1) TPS)) of row j
struct TileIter {
    long long u;
    int tile, tend;
    long long j;
    __device__ void start(const SArgs& s, int g) {
        u = g;
        set_unit(s);
    }
    __device__ void set_unit(const SArgs& s) {
        if (u < s.U) {
            j = u / s.S;
            const int seg = (int)(u - j * s.S);
            tile = seg * s.TPS;
            tend = min(s.TPR, tile + s.TPS);
        }
    }
    __device__ bool valid(const SArgs& s) const { return u < s.U; }
    __device__ void next(const SArgs& s) {
        if (++tile >= tend) {
            u += s.G;
            set_unit(s);
        }
    }
};

template <int M>
__device__ __forceinline__ void issue_tile(const KArgs& a, long long j, int tile, double* stage,
                                           unsigned long long* bar) {
    constexpr int TL = StreamCfg<M>::TL;
    const int k0 = tile * TL;
    const int nc = min(TL, a.n - k0);
    const unsigned bytes = (unsigned)(((nc + 1) & ~1) * 8);  // 16-byte multiple (rows padded to 4)
    const long long qn = a.q * (long long)a.n_pad;
    mbar_expect_tx(bar, bytes * StreamCfg<M>::NSTREAM);
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const long long e = (long long)i * qn + j * a.n_pad + k0;
        const long long bk = (long long)i * a.n_pad + k0;
        double* d = stage + (size_t)(7 * i) * TL;
        tma_load_1d(d, a.x + e, bytes, bar);
        tma_load_1d(d + TL, a.a2 + e, bytes, bar);
        tma_load_1d(d + 2 * TL, a.a1 + e, bytes, bar);
        tma_load_1d(d + 3 * TL, a.b2 + e, bytes, bar);
        tma_load_1d(d + 4 * TL, a.b1 + e, bytes, bar);
        tma_load_1d(d + 5 * TL, a.lo + bk, bytes, bar);
        tma_load_1d(d + 6 * TL, a.hi + bk, bytes, bar);
    }
    double* d = stage + (size_t)(7 * M) * TL;
    tma_load_1d(d, a.y + j * a.n_pad + k0, bytes, bar);
    tma_load_1d(d + TL, a.v + j * a.n_pad + k0, bytes, bar);
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int M, int MODE>
__global__ void __launch_bounds__(StreamCfg<M>::TL, 1) sweep_tma_kernel(KArgs a, SArgs sa) {
    constexpr int TL = StreamCfg<M>::TL;
    constexpr int NS = StreamCfg<M>::NS;
    constexpr int NSTREAM = StreamCfg<M>::NSTREAM;
    constexpr int NW = TL / 32;  // warps
    constexpr int UB = 4;        // unit slots in flight (> NS tiles of skew between warps)
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) unsigned long long s_full[NS];
    __shared__ unsigned s_rel[NS];  // warps done with the stage's current tile
    __shared__ unsigned long long s_fxw[UB][NW][M];  // per-warp fixed-point row partials
    __shared__ double s_dgw[UB][NW][2 * M];         // per-warp dg extrema (checks)
    __shared__ unsigned s_arrive[UB];
    __shared__ double s_wred[NW][2];
    __shared__ double s_rowt[NW][4];
    __shared__ double acc[XB];
    __shared__ int s_last;

    const long long it = *(volatile long long*)a.iter;
    const Ctrl& cin = a.ctrl[it & 1];
    if (cin.done || it >= a.prm->iter_limit) return;
    const int ce = a.prm->check_every;
    const bool is_check = ce > 0 && ((it + 1) % ce) == 0;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    if (tid < XB) {
        double init = 0.0;
        if (tid >= MAXM && tid < MAXM + M) init = -INFINITY;       // x0max
        if (tid >= 2 * MAXM && tid < 2 * MAXM + M) init = INFINITY;  // x0min
        acc[tid] = init;
    }
    if (tid < UB) s_arrive[tid] = 0u;
    if (tid < NS) s_rel[tid] = 0u;
    TileIter ahead;  // the tile NS positions ahead of the current one (the refill of its stage)
    ahead.start(sa, blockIdx.x);
    if (tid == 0) {
        for (int st = 0; st < NS; ++st) mbar_init(&s_full[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    for (int st = 0; st < NS && ahead.valid(sa); ++st) {
        if (tid == 0) issue_tile<M>(a, ahead.j, ahead.tile, sm + (size_t)st * NSTREAM * TL, &s_full[st]);
        ahead.next(sa);
    }
    {
        // ================= all warps consume: one cell per thread
        double rho[4], f[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            rho[l] = cin.rho[l];
            f[l] = cin.f[l];
        }
        double fxs[M];
#pragma unroll
        for (int i = 0; i < M; ++i) fxs[i] = sa.fx_scale[i];
        const double iq = a.inv_q;
        const long long qn = a.q * (long long)a.n_pad;
        double my_r1 = 0.0, my_s3 = 0.0;                              // per-thread cell maxima
        double my_r2 = 0.0, my_r3 = 0.0, my_s1 = 0.0, my_s2 = 0.0;  // row terms (lanes i < M)

        TileIter cons;
        cons.start(sa, blockIdx.x);
        int st = 0;
        unsigned ph = 0;
        // row scalars of the current unit, prefetched one unit ahead (lane i < M: source i)
        double pz = 0.0, pnu = 0.0;
        auto fetch = [&](long long jj, bool k0row) {
            pz = 0.0;
            pnu = 0.0;
            if (lane < M) {
                const long long rix = (long long)lane * a.q + jj;
                pz = __ldcg(a.zeta + rix) + __ldcg(a.lam + rix) * f[0];
                if (k0row && wid == 0) pnu = __ldcg(a.nu + rix);
            }
        };
        if (cons.valid(sa)) fetch(cons.j, cons.tile == 0);
        long long unit = 0;
        while (cons.valid(sa)) {
            const long long j = cons.j;
            const bool has_k0 = (cons.tile == 0);
            double zl[M];
#pragma unroll
            for (int i = 0; i < M; ++i) zl[i] = __shfl_sync(0xffffffffu, pz, i);
            double nu_row[M];  // raw nu of row j (warp 0, k = 0 tile only)
#pragma unroll
            for (int i = 0; i < M; ++i) nu_row[i] = __shfl_sync(0xffffffffu, pnu, i);
            {   // prefetch the next unit's row scalars
                TileIter nx = cons;
                nx.u += sa.G;
                nx.set_unit(sa);
                if (nx.valid(sa)) fetch(nx.j, nx.tile == 0);
            }
            long long fx[M];
            double dgx[M], dgn[M];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                fx[i] = 0;
                dgx[i] = -INFINITY;
                dgn[i] = INFINITY;
            }
            double k0nu[M], k0x1nu[M];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                k0nu[i] = 0.0;
                k0x1nu[i] = 0.0;
            }
            while (true) {
                const int tile = cons.tile;
                const int k = tile * TL + tid;
                const bool valid = k < a.n;
                const double* sp = sm + (size_t)st * NSTREAM * TL;
                while (!mbar_try_wait(&s_full[st], ph)) {
                }
                if (valid) {
                    double xo[M], xn[M], ca2[M], ca1[M], cb2[M], cb1[M], clo[M], chi[M];
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        const double* d = sp + (size_t)(7 * i) * TL + tid;
                        xo[i] = d[0];
                        ca2[i] = d[TL];
                        ca1[i] = d[2 * TL];
                        cb2[i] = d[3 * TL];
                        cb1[i] = d[4 * TL];
                        clo[i] = d[5 * TL];
                        chi[i] = d[6 * TL];
                    }
                    const double yv = sp[(size_t)(7 * M) * TL + tid];
                    const double vv = sp[(size_t)(7 * M + 1) * TL + tid];
                    const bool k0 = (k == 0);
                    if (k0) {
                        // lazy (6h) of the previous iteration, then its dual rescale
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            double nu = nu_row[i];
                            if (cin.nu_pending) nu = nu + cin.x1[i] - xo[i];
                            k0nu[i] = nu * f[3];
                            k0x1nu[i] = cin.x1[i] + k0nu[i];
                            __stcg(a.nu + (long long)i * a.q + j, k0nu[i]);
                        }
                    }
                    const double s_e = fmax(vv, 0.0);
                    const double mu_e = vv < 0.0 ? -vv * f[2] : 0.0;
                    gs_cell<M, MODE>(ca2, ca1, cb2, cb1, clo, chi, xo, xn, yv, s_e, mu_e, zl, rho, iq,
                                     k0, k0x1nu);
                    const double vnew = cell_tail<M>(xo, xn, yv, vv, f[2], is_check, my_r1, my_s3);
                    a.v[j * a.n_pad + k] = vnew;
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        a.x[(long long)i * qn + j * a.n_pad + k] = xn[i];
                        fx[i] += __double2ll_rn(fma(cb2[i], xn[i], cb1[i]) * xn[i] * fxs[i]);
                        if (is_check) {
                            const double dg = (xn[i] - xo[i]) * fma(cb2[i], xn[i] + xo[i], cb1[i]);
                            dgx[i] = fmax(dgx[i], dg);
                            dgn[i] = fmin(dgn[i], dg);
                        }
                    }
                    if (k0) {
                        // (6c) contribution x_1 - nu (nu before (6h)), in this CTA's unit order
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            acc[i] += xn[i] - k0nu[i];
                            acc[MAXM + i] = fmax(acc[MAXM + i], xn[i]);
                            acc[2 * MAXM + i] = fmin(acc[2 * MAXM + i], xn[i]);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    // the warp that releases the stage last refills it with the tile NS ahead
                    __threadfence_block();
                    if (atomicAdd(&s_rel[st], 1u) == (unsigned)NW - 1) {
                        s_rel[st] = 0u;
                        if (ahead.valid(sa)) {
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            issue_tile<M>(a, ahead.j, ahead.tile, sm + (size_t)st * NSTREAM * TL, &s_full[st]);
                        }
                    }
                }
                ahead.next(sa);
                if (++st == NS) {
                    st = 0;
                    ph ^= 1u;
                }
                const long long u_before = cons.u;
                cons.next(sa);
                if (cons.u != u_before) break;  // unit finished
            }

            // ---- unit end: warp partials into slot b; the last warp finalises row j
            const int b = (int)(unit & (UB - 1));
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const unsigned long long ws = warp_sum_u64((unsigned long long)fx[i]);
                if (lane == 0) s_fxw[b][wid][i] = ws;
                if (is_check) {
                    const double mx = warp_max(dgx[i]), mn = warp_min(dgn[i]);
                    if (lane == 0) {
                        s_dgw[b][wid][i] = mx;
                        s_dgw[b][wid][M + i] = mn;
                    }
                }
            }
            unsigned last = 0;
            if (lane == 0) {
                __threadfence_block();
                last = (atomicAdd(&s_arrive[b], 1u) == (unsigned)NW - 1);
                __threadfence_block();
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            __syncwarp();  // memory ordering: lane 0 acquired the slot writes, the warp reads them
            if (last) {
                if (lane < M) {
                    const int i = lane;
                    unsigned long long part = 0ull;
                    double mx = -INFINITY, mn = INFINITY;
                    for (int w = 0; w < NW; ++w) {
                        part += s_fxw[b][w][i];
                        if (is_check) {
                            mx = fmax(mx, s_dgw[b][w][i]);
                            mn = fmin(mn, s_dgw[b][w][M + i]);
                        }
                    }
                    bool fin = true;
                    if (sa.S > 1) {
                        // rows split over CTAs: global exact sums, the last segment finalises
                        atomicAdd(sa.rowacc + j * MAXM + i, part);
                        if (is_check) {
                            atomicMax(sa.rowdg + j * 2 * MAXM + i, okey(mx));
                            atomicMin(sa.rowdg + j * 2 * MAXM + MAXM + i, okey(mn));
                        }
                        __threadfence();
                        fin = (atomicAdd(sa.rowcnt + j * MAXM + i, 1u) == (unsigned)sa.S - 1);
                        if (fin) {
                            __threadfence();
                            part = atomicExch(sa.rowacc + j * MAXM + i, 0ull);
                            if (is_check) {
                                mx = okey_inv(atomicExch(sa.rowdg + j * 2 * MAXM + i, 0ull));
                                mn = okey_inv(atomicExch(sa.rowdg + j * 2 * MAXM + MAXM + i, ~0ull));
                            }
                            sa.rowcnt[j * MAXM + i] = 0u;
                        }
                    }
                    if (fin) {
                        const double Sg = (double)(long long)part * sa.fx_inv[i];
                        double r2, r3, s1, s2;
                        finalize_row(a, cin, i, j, Sg, mx, mn, &r2, &r3, &s1, &s2);
                        if (is_check) {
                            my_r2 = fmax(my_r2, r2);
                            my_r3 = fmax(my_r3, r3);
                            my_s1 = fmax(my_s1, s1);
                            my_s2 = fmax(my_s2, s2);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) s_arrive[b] = 0u;
            }
            ++unit;
        }
        // ---- this warp's check partials
        if (is_check) {
            const double r1 = warp_max(my_r1), s3 = warp_max(my_s3);
            const double r2 = warp_max(my_r2), r3 = warp_max(my_r3);
            const double s1 = warp_max(my_s1), s2 = warp_max(my_s2);
            if (lane == 0) {
                s_wred[wid][0] = r1;
                s_wred[wid][1] = s3;
                s_rowt[wid][0] = r2;
                s_rowt[wid][1] = r3;
                s_rowt[wid][2] = s1;
                s_rowt[wid][3] = s2;
            }
        }
    }
    __syncthreads();
    if (is_check && tid == 0) {
        double r1m = 0.0, s3m = 0.0, r2 = 0.0, r3 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int w = 0; w < NW; ++w) {
            r1m = fmax(r1m, s_wred[w][0]);
            s3m = fmax(s3m, s_wred[w][1]);
            r2 = fmax(r2, s_rowt[w][0]);
            r3 = fmax(r3, s_rowt[w][1]);
            s1 = fmax(s1, s_rowt[w][2]);
            s2 = fmax(s2, s_rowt[w][3]);
        }
        acc[3 * MAXM + 0] = r1m;
        acc[3 * MAXM + 1] = r2;
        acc[3 * MAXM + 2] = r3;
        acc[3 * MAXM + 3] = s1;
        acc[3 * MAXM + 4] = s2;
        acc[3 * MAXM + 5] = s3m;
    }
    __syncthreads();
    if (tid < XB) __stcg(a.cta_part + (size_t)blockIdx.x * XB + tid, acc[tid]);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(a.glob_cnt, 1) == sa.G - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // ---- last CTA: reduce the G CTA partials in CTA order (lane = slot, warp w takes
    // CTAs w, w + NW, ...; then slot-wise over warps in order) => deterministic
    {
        __shared__ double wred[NW][XB];
        const int s = lane;
        const bool is_sum = s < MAXM;
        const bool is_min = s >= 2 * MAXM && s < 3 * MAXM;
        const double ident = is_sum ? 0.0 : (is_min ? INFINITY : (s >= 3 * MAXM ? 0.0 : -INFINITY));
        double v = ident;
        for (int g = wid; g < sa.G; g += NW) {
            const double t = __ldcg(a.cta_part + (size_t)g * XB + s);
            v = is_sum ? v + t : (is_min ? fmin(v, t) : fmax(v, t));
        }
        wred[wid][s] = v;
        __syncthreads();
        if (tid < XB) {
            double r = ident;
            for (int w = 0; w < NW; ++w) {
                const double t = wred[w][tid];
                r = is_sum ? r + t : (is_min ? fmin(r, t) : fmax(r, t));
            }
            acc[tid] = r;
        }
        __syncthreads();
    }
    if (tid < XB) a.xsend[tid] = acc[tid];
    if (tid == 0) {
        *a.glob_cnt = 0;
        if (a.world == 1) {
            Ctrl& cout = a.ctrl[(it + 1) & 1];
            finalize_global(a, acc, 1, it, cin, cout, is_check);
            __threadfence();
            *(volatile long long*)a.iter = it + 1;
        }
    }
}

}  // namespace admm_dev
