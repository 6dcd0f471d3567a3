// admm_sweep2.cuh -- the streaming ADMM sweep for problems that live in HBM
// (BASELINE.json configs[3] q >= 1e3, configs[2] n >= 1e5): one launch = one
// ADMM iteration, Appendix A Eq. (6a)-(6i) with the residuals of
// :464-479 on check iterations.  DESIGN.md §6 "TMA streaming sweep".
//
// Structure (B200):
//  * persistent grid of 128-thread CTAs, several per SM (4 at m = 2), each
//    owning whole work units (a scenario row j, or a segment of a long row)
//    in a fixed order: deterministic;
//  * every warp streams its own chunks of 64 cells (chunk c of a unit belongs
//    to warp c mod 4) HBM -> shared memory with three or four TMA tensor copies
//    (cp.async.bulk.tensor: x of every source as one 3-D box, a2/a1/b2/b1 of
//    every source as one 4-D box, y and v as one, the box bounds as one; mbarrier
//    complete_tx) into a private NS-stage ring issued by its lane 0: the fp64 work of chunk c overlaps the HBM reads of the
//    warp's next chunks without holding registers for loads in flight, and no
//    warp ever waits for another one (no barrier, no shared ring);
//  * two cells per thread: Gauss-Seidel over the sources (6a) with Algorithm 1
//    on both cells interleaved, (6e)/(6f) in the thread (identity I2),
//    x and v written back with 128-bit stores;
//  * the row sum sum_k (b2 x^2 + b1 x) of (6b) is accumulated per thread in
//    exact 64-bit fixed point across the unit's tiles, warp-summed with
//    redux.sync limbs, and the last warp to reach the unit's end finalises
//    the row ((6b), (6g), (6d), (6i) via identity I1) -- no block barrier in
//    the sweep; rows split into segments add their sums with integer atomics
//    and the last segment finalises (order-independent => deterministic);
//  * (6c) consensus partials (thread 0 owns k = 0 of every row it streams)
//    and the residual maxima are reduced by the last CTA in CTA order, which
//    also runs the check / rho adaptation and writes the next control block.
#pragma once
#include <cuda.h>

#include "admm_kernels.cuh"

namespace admm_dev {

struct S2Args {
    int TPR;      // chunks per row (ceil(n_pad / chunk))
    int S;        // segments per row
    int TPS;      // chunks per segment
    int G;        // grid size
    long long U;  // work units = q * S
};

constexpr int S2_NT = 128;  // threads per CTA
constexpr int S2_NW = S2_NT / 32;
constexpr int S2_UB = 8;    // unit slots of the row partials (flow-controlled by s_gen)

// TMA tensor maps of the arrays a sweep streams (built by the host, admm.cu plan_stream):
//   x   [m][q][n_pad] fp64, box {TL, 1, M}
//   c   [4][m][q][n_pad] (a2, a1, b2, b1 at one stride; fp64, or the fp32 copies), box {TL, 1, M, 4}
//   yv  [2][q][n_pad] (y, v adjacent) fp64, box {TL, 1, 2}
//   box [2][m][n_pad] (lo, hi adjacent) fp64, box {TL, M, 2} (BX layout only)
struct S2Maps {
    CUtensorMap x, c, yv, box;
};

// one stage of a warp's ring (chunk of TL = 32 L cells, L cells per lane): x_i (M, fp64),
// y, v (fp64), a2_i, a1_i, b2_i, b1_i (CT), and with BX the box lo_i, hi_i (fp64: horizon-
// type problems, where the box is not shared by many rows and would be an HBM stream of
// its own read through L1)
template <int M, typename CT, int L, bool BX>
struct S2Cfg {
    static constexpr int TL = 32 * L;
    static constexpr int YOFF = M * TL * 8;          // x: [M][TL]
    static constexpr int VOFF = (M + 1) * TL * 8;    // y, v: [2][TL]
    static constexpr int COFF = (M + 2) * TL * 8;    // coefficient c of source i: [4][M][TL]
    static constexpr int CSTR = M * TL * (int)sizeof(CT);  // bytes between coefficients
    static constexpr int BOFF = COFF + 4 * CSTR;     // lo, hi: [2][M][TL]
    static constexpr int STAGE = BOFF + (BX ? 2 * M * TL * 8 : 0);
    static constexpr unsigned BYTES = (unsigned)((M + 2 + (BX ? 2 * M : 0)) * TL * 8 + 4 * CSTR);
};

__device__ __forceinline__ unsigned s2_smem(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// shared-memory operands are passed as 32-bit shared addresses computed once (the
// conversion inside a polling loop would be redone on every try)
__device__ __forceinline__ void s2_bar_init(unsigned bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void s2_expect(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool s2_try(unsigned bar, unsigned phase) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void s2_wait(unsigned bar, unsigned phase) {
    while (!s2_try(bar, phase)) {
    }
}
__device__ __forceinline__ void s2_tma(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// first chunk (offset from the unit's start) of warp wid in the CTA's lu-th unit:
// the assignment rotates by one warp per unit, so the short last chunk of a row
// and the consensus cell k = 0 visit every warp in turn (balanced warps)
__device__ __forceinline__ int s2_first(int wid, unsigned lu) { return (int)((wid - lu) & (S2_NW - 1)); }

// position in one warp's chunk sequence: units u = blockIdx.x, + G, ...; chunks
// cs + s2_first, + NW, ... < ce of unit u (row j); units without a chunk for this
// warp are skipped
struct S2Pos {
    long long u, j;
    int c, ce;
    unsigned lu;  // CTA-local unit count: chunk c of a unit goes to warp (c - cs + lu) mod NW
    __device__ __forceinline__ void set(const S2Args& s, int wid) {
        while (u < s.U) {
            int cs;
            if (s.S == 1) {
                j = u;
                cs = 0;
                ce = s.TPR;
            } else {
                j = u / s.S;
                cs = (int)(u - j * s.S) * s.TPS;
                ce = min(s.TPR, cs + s.TPS);
            }
            c = cs + s2_first(wid, lu);
            if (c < ce) return;
            u += s.G;
            ++lu;
        }
    }
    __device__ __forceinline__ void next(const S2Args& s, int wid) {
        c += S2_NW;
        if (c >= ce) {
            u += s.G;
            ++lu;
            set(s, wid);
        }
    }
};

// few-row (horizon-type) layout: the rows are streamed once per iteration with an L2
// evict-first hint (measured: n = 1e6 0.56 -> 0.61 of the HBM peak); the many-rows layout
// keeps the default policy (the hint cost it 0.71 -> 0.68: more DRAM reads)
__device__ __forceinline__ unsigned long long s2_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long s2_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// two consecutive doubles through the non-coherent path with an L2 cache policy
__device__ __forceinline__ void s2_ld2_keep(const double* p, double* o, unsigned long long pol) {
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(o[0]), "=d"(o[1])
                 : "l"(p), "l"(pol));
}
template <bool EF>
__device__ __forceinline__ void s2_tmap3(unsigned dst, const CUtensorMap* m, int c0, int c1, unsigned bar) {
    if constexpr (EF) asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(
            dst),
        "l"(m), "r"(c0), "r"(c1), "r"(0), "r"(bar), "l"(s2_evict_first())
        : "memory");
    else asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            dst),
        "l"(m), "r"(c0), "r"(c1), "r"(0), "r"(bar)
        : "memory");
}
template <bool EF>
__device__ __forceinline__ void s2_tmap4(unsigned dst, const CUtensorMap* m, int c0, int c1, unsigned bar) {
    if constexpr (EF) asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(
            dst),
        "l"(m), "r"(c0), "r"(c1), "r"(0), "r"(0), "r"(bar), "l"(s2_evict_first())
        : "memory");
    else asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
            dst),
        "l"(m), "r"(c0), "r"(c1), "r"(0), "r"(0), "r"(bar)
        : "memory");
}

// one chunk (row j, chunk t) into a stage: three tensor copies (four with the box); a
// chunk past n_pad is zero-filled by the TMA unit and counts its full box
template <int M, typename CT, int L, bool BX>
__device__ __forceinline__ void s2_issue(const S2Maps& tm, long long j, int t, unsigned st, unsigned bar) {
    using C = S2Cfg<M, CT, L, BX>;
    const int k0 = t * C::TL;
    s2_expect(bar, C::BYTES);
    s2_tmap3<BX>(st, &tm.x, k0, (int)j, bar);
    s2_tmap4<BX>(st + C::COFF, &tm.c, k0, (int)j, bar);
    s2_tmap3<BX>(st + C::YOFF, &tm.yv, k0, (int)j, bar);
    if constexpr (BX) s2_tmap3<true>(st + C::BOFF, &tm.box, k0, 0, bar);
}

// L consecutive values of a shared-memory stream (fp64 or fp32), widened
template <typename CT, int L>
__device__ __forceinline__ void s2_ldL(const unsigned char* p, double* o) {
    if constexpr (L == 1) {
        o[0] = (double)*reinterpret_cast<const CT*>(p);
    } else if constexpr (sizeof(CT) == 8) {
        const double2 t = *reinterpret_cast<const double2*>(p);
        o[0] = t.x;
        o[1] = t.y;
    } else {
        const float2 t = *reinterpret_cast<const float2*>(p);
        o[0] = (double)t.x;
        o[1] = (double)t.y;
    }
}
template <int L>
__device__ __forceinline__ void s2_stL(double* p, const double* v) {
    if constexpr (L == 1) *p = v[0];
    else *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
}

#ifndef SWEEP2_MINB
#define SWEEP2_MINB 4
#endif

// L = 2: two cells per lane (M <= 2, many rows: the configs[3] kernel); L = 1 with the box
// staged (BX): horizon-type problems (few rows, M up to 4) -- half the registers per lane,
// so more warps per SM, and no L1 misses on the box
template <int M, int MODE, typename CT, int NS, int L, bool BX>
__global__ void __launch_bounds__(S2_NT, L == 1 ? 3 : (M <= 2 ? SWEEP2_MINB : 2))
    sweep2_kernel(KArgs a, S2Args s, const __grid_constant__ S2Maps tm) {
    using C = S2Cfg<M, CT, L, BX>;
    constexpr int TL = C::TL;
    extern __shared__ __align__(128) unsigned char s2_sm[];
    __shared__ __align__(8) unsigned long long s_full[S2_NW][NS];  // per-warp rings
    __shared__ unsigned long long s_fxw[S2_UB][S2_NW][M];  // per-warp fixed-point row partials
    __shared__ double s_dgw[S2_UB][S2_NW][2 * M];         // per-warp dg extrema (checks)
    __shared__ unsigned s_arr[S2_UB];                      // warps arrived at the unit's end
    __shared__ unsigned s_gen[S2_UB];                      // finalisations done per slot
    __shared__ double s_red[S2_NW][6];
    __shared__ double s_rc[S2_NW][M][4];   // row check terms of the finalising lanes
    // row scalars (raw lam, zeta, p, h, sum b0, nu) of source i, per warp and unit parity:
    // copied with cp.async by lanes i < M one unit ahead (no registers held in flight)
    __shared__ double s_sc[S2_NW][2][6][M];
    __shared__ double s_nue[S2_NW][M];     // nu after (6h), cell k = 0 (lane 0 of its warp)
    // (6c) partials of the k = 0 cells each warp owned, in unit order: sum x_1 - nu,
    // max, min (combined in warp order at the end: deterministic)
    __shared__ double s_cons[S2_NW][3][M];
    __shared__ double acc[XB];
    __shared__ int s_last;

    const long long it = *(volatile long long*)a.iter;
    const Ctrl& cin = a.ctrl[it & 1];
    if (cin.done || it >= a.prm->iter_limit) return;
    const int ce = a.prm->check_every;
    const bool chk = ce > 0 && ((it + 1) % ce) == 0;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    if (tid < XB) {
        double init = 0.0;
        if (tid >= MAXM && tid < MAXM + M) init = -INFINITY;        // x0max
        if (tid >= 2 * MAXM && tid < 2 * MAXM + M) init = INFINITY;  // x0min
        acc[tid] = init;
    }
    if (tid < S2_UB) {
        s_arr[tid] = 0u;
        s_gen[tid] = 0u;
    }
    if (tid < S2_NW * M * 4) (&s_rc[0][0][0])[tid] = 0.0;
    if (tid < S2_NW * M) {
        s_cons[tid / M][0][tid % M] = 0.0;
        s_cons[tid / M][1][tid % M] = -INFINITY;
        s_cons[tid / M][2][tid % M] = INFINITY;
    }
    if (tid < S2_NW * NS) {
        s2_bar_init(s2_smem(&s_full[0][0] + tid));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    unsigned char* const ring = s2_sm + (size_t)wid * NS * C::STAGE;  // this warp's stages
    const unsigned ring_s = s2_smem(ring), bar_s = s2_smem(&s_full[wid][0]);
    S2Pos ahead;  // this warp's chunk NS positions ahead of the consumer: the refill of its stage
    ahead.u = blockIdx.x;
    ahead.lu = 0;
    ahead.set(s, wid);
    for (int st = 0; st < NS && ahead.u < s.U; ++st) {
        if (lane == 0) s2_issue<M, CT, L, BX>(tm, ahead.j, ahead.c, ring_s + st * C::STAGE, bar_s + 8 * st);
        ahead.next(s, wid);
    }

    const double R1 = cin.rho[0], R3 = cin.rho[2], R4 = cin.rho[3], f2 = cin.f[2];
    const double iq = a.inv_q;
    const long long qn = a.q * (long long)a.n_pad;
    const bool nu_pending = cin.nu_pending != 0;

    double my_r1 = 0.0, my_s3 = 0.0;  // cell terms of the check (every thread)

    int st = 0;
    unsigned ph = 0;
    auto fetch = [&](long long uu, int slot) {
        if (lane < M && uu < s.U) {
            const long long rix = (long long)lane * a.q + (s.S == 1 ? uu : uu / s.S);
            double* d = &s_sc[wid][slot][0][lane];
            cp_async8(d, a.lam + rix);
            cp_async8(d + M, a.zeta + rix);
            cp_async8(d + 2 * M, a.p + rix);
            cp_async8(d + 3 * M, a.h + rix);
            cp_async8(d + 4 * M, a.sb0 + rix);
            cp_async8(d + 5 * M, a.nu + rix);
        }
        cp_async_commit();
    };
    fetch(blockIdx.x, 0);
    long long unit = 0;
    for (long long uu = blockIdx.x; uu < s.U; uu += s.G, ++unit) {
        long long j;
        int cs, ce;
        if (s.S == 1) {
            j = uu;
            cs = 0;
            ce = s.TPR;
        } else {
            j = uu / s.S;
            cs = (int)(uu - j * s.S) * s.TPS;
            ce = min(s.TPR, cs + s.TPS);
        }
        const int slot = (int)(unit & 1);
        fetch(uu + s.G, slot ^ 1);
        cp_async_wait1();  // this unit's row scalars (issued one unit ago) have landed
        __syncwarp();
        const double(*sc)[M] = s_sc[wid][slot];
        double zl[M];  // zeta + lam of source i (lam with its pending rescale)
#pragma unroll
        for (int i = 0; i < M; ++i) zl[i] = sc[1][i] + sc[0][i] * cin.f[0];

        long long fx[M];
        double dgx[M], dgn[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            fx[i] = 0;
            dgx[i] = -INFINITY;
            dgn[i] = INFINITY;
        }
        for (int c = cs + s2_first(wid, (unsigned)unit); c < ce; c += S2_NW) {
            const int k = c * TL + L * lane;  // first of this thread's L cells
            const unsigned char* sp = ring + (size_t)st * C::STAGE;
            s2_wait(bar_s + 8 * st, ph);
            if (k < a.n_pad) {
                const bool k0 = (k == 0) && a.k0own;
                bool vc[L];
#pragma unroll
                for (int u = 0; u < L; ++u) vc[u] = (k + u) < a.n;
                double y[L], v[L], xo[M][L], xn[M][L];
                s2_ldL<double, L>(sp + C::YOFF + 8 * L * lane, y);
                s2_ldL<double, L>(sp + C::VOFF + 8 * L * lane, v);
#pragma unroll
                for (int i = 0; i < M; ++i) s2_ldL<double, L>(sp + (size_t)i * TL * 8 + 8 * L * lane, xo[i]);
                double s_e[L], mu_e[L];
#pragma unroll
                for (int u = 0; u < L; ++u) {
                    s_e[u] = fmax(v[u], 0.0);
                    mu_e[u] = v[u] < 0.0 ? -v[u] * f2 : 0.0;
                }
                // ---- (6a) Gauss-Seidel over sources (same arithmetic as gs_cellU)
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const unsigned char* cp = sp + C::COFF + (size_t)i * TL * sizeof(CT) +
                                              L * sizeof(CT) * lane;
                    double a2[L], a1[L], b2[L], b1[L];
                    s2_ldL<CT, L>(cp, a2);
                    s2_ldL<CT, L>(cp + C::CSTR, a1);
                    double Cq[L], Dq[L], bn[L], cn[L], dn[L], lo[L], hi[L];
                    if constexpr (BX) {
                        s2_ldL<double, L>(sp + C::BOFF + (size_t)i * TL * 8 + 8 * L * lane, lo);
                        s2_ldL<double, L>(sp + C::BOFF + (size_t)(M + i) * TL * 8 + 8 * L * lane, hi);
                    } else if constexpr (L == 2) {
                        // the box is re-read by every row: keep it in L2 (evict-last hint)
                        const unsigned long long pol_keep = s2_evict_last();
                        s2_ld2_keep(a.lo + (long long)i * a.n_pad + k, lo, pol_keep);
                        s2_ld2_keep(a.hi + (long long)i * a.n_pad + k, hi, pol_keep);
                    } else {
                        lo[0] = __ldg(a.lo + (long long)i * a.n_pad + k);
                        hi[0] = __ldg(a.hi + (long long)i * a.n_pad + k);
                    }
                    // k = 0 (consensus) cell: lazy (6h) of the previous iteration, then its
                    // dual rescale; adds the rho4 term of (6a)
                    auto k0_term = [&](double xoi, double& Cc, double& Dc) {
                        double nu = sc[5][i];
                        if (nu_pending) nu = nu + cin.x1[i] - xoi;
                        const double nu_e = nu * cin.f[3];
                        __stcg(a.nu + (long long)i * a.q + j, nu_e);
                        s_nue[wid][i] = nu_e;
                        Cc += 0.5 * R4;
                        Dc += -R4 * (cin.x1[i] + nu_e);
                    };
                    if ((a.gfree >> i) & 1u) {
                        // g = 0 on the box (b2 = b1 = 0 everywhere): the (6a) objective is the
                        // convex quadratic (a2/q + rho3/2 [+ rho4/2]) x^2 + (a1/q - rho3 phi [...]) x;
                        // the same C, D as below with the b terms exactly zero
#pragma unroll
                        for (int u = 0; u < L; ++u) {
                            double others = 0.0;
#pragma unroll
                            for (int l = 0; l < M; ++l)
                                if (l != i) others += (l < i) ? xn[l][u] : xo[l][u];
                            const double phi = ((s_e[u] - others) + y[u]) + mu_e[u];
                            Cq[u] = fma(a2[u], iq, 0.5 * R3);
                            Dq[u] = fma(a1[u], iq, -R3 * phi);
                            if (k0 && u == 0) k0_term(xo[i][u], Cq[u], Dq[u]);
                            xn[i][u] = clampd(-Dq[u] * rcp_nr(2.0 * Cq[u]), lo[u], hi[u]);
                        }
                        continue;
                    }
                    s2_ldL<CT, L>(cp + 2 * C::CSTR, b2);
                    s2_ldL<CT, L>(cp + 3 * C::CSTR, b1);
                    bool allq = true, anyq = false;
#pragma unroll
                    for (int u = 0; u < L; ++u) {
                        double others = 0.0;
#pragma unroll
                        for (int l = 0; l < M; ++l)
                            if (l != i) others += (l < i) ? xn[l][u] : xo[l][u];
                        const double phi = ((s_e[u] - others) + y[u]) + mu_e[u];
                        const double xoi = xo[i][u];
                        const double e = fma(fma(b2[u], xoi, b1[u]), xoi, zl[i]);
                        Cq[u] = fma(0.5 * R1, fma(b1[u], b1[u], -2.0 * b2[u] * e), fma(a2[u], iq, 0.5 * R3));
                        Dq[u] = fma(-R1 * b1[u], e, fma(a1[u], iq, -R3 * phi));
                        if (k0 && u == 0) k0_term(xoi, Cq[u], Dq[u]);
                        const bool qu = (b2[u] != 0.0);
                        allq = allq && qu;
                        anyq = anyq || qu;
                        const double ia2 = rcp_nr(qu ? R1 * b2[u] * b2[u] : 1.0);  // 1 / 2A
                        bn[u] = 1.5 * (R1 * b2[u] * b1[u]) * ia2;
                        cn[u] = Cq[u] * ia2;
                        dn[u] = 0.5 * Dq[u] * ia2;
                    }
                    if (allq) {
                        double r[L];
                        quartic_coreU<MODE, L>(bn, cn, dn, Cq, Dq, lo, hi, r);
#pragma unroll
                        for (int u = 0; u < L; ++u) xn[i][u] = r[u];
                    } else if (!anyq) {  // a source without g (A = B = 0): quadratic
#pragma unroll
                        for (int u = 0; u < L; ++u) xn[i][u] = clampd(-Dq[u] * rcp_nr(2.0 * Cq[u]), lo[u], hi[u]);
                    } else {
#pragma unroll
                        for (int u = 0; u < L; ++u)
                            xn[i][u] = (b2[u] != 0.0) ? quartic_core<MODE>(bn[u], cn[u], dn[u], Cq[u], Dq[u], lo[u], hi[u])
                                                      : clampd(-Dq[u] * rcp_nr(2.0 * Cq[u]), lo[u], hi[u]);
                    }
                }
                // ---- (6e)/(6f) per cell, reduced state v = s - mu (identity I2)
                double vn[L];
#pragma unroll
                for (int u = 0; u < L; ++u) {
                    double txo[M], txn[M];
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        txo[i] = xo[i][u];
                        txn[i] = xn[i][u];
                    }
                    const bool valid = vc[u];
                    double r1l = my_r1, s3l = my_s3;
                    const double vnew = cell_tail<M>(txo, txn, y[u], v[u], f2, chk && valid, r1l, s3l);
                    my_r1 = r1l;
                    my_s3 = s3l;
                    vn[u] = valid ? vnew : 0.0;
                }
                s2_stL<L>(a.v + j * a.n_pad + k, vn);
                // ---- row partials: exact fixed point, dg extrema on checks
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const unsigned char* cp = sp + C::COFF + 2 * C::CSTR + (size_t)i * TL * sizeof(CT) +
                                              L * sizeof(CT) * lane;
                    double b2[L], b1[L];
                    s2_ldL<CT, L>(cp, b2);
                    s2_ldL<CT, L>(cp + C::CSTR, b1);
#pragma unroll
                    for (int u = 0; u < L; ++u)
                        if (!vc[u]) xn[i][u] = 0.0;  // padding stays 0
                    s2_stL<L>(a.x + i * qn + j * a.n_pad + k, xn[i]);
                    if ((a.gfree >> i) & 1u) continue;  // g = 0 on the box: no row sum, dg = 0
#pragma unroll
                    for (int u = 0; u < L; ++u) {
                        if (vc[u]) {
                            fx[i] += __double2ll_rn(fma(b2[u], xn[i][u], b1[u]) * xn[i][u] * a.fx_scale[i]);
                            if (chk) {  // sigma's z-term only
                                const double dg = (xn[i][u] - xo[i][u]) * fma(b2[u], xn[i][u] + xo[i][u], b1[u]);
                                dgx[i] = fmax(dgx[i], dg);
                                dgn[i] = fmin(dgn[i], dg);
                            }
                        }
                    }
                }
                if (k0) {
                    // (6c) contribution x_1 - nu, in this warp's unit order
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        s_cons[wid][0][i] += xn[i][0] - s_nue[wid][i];
                        s_cons[wid][1][i] = fmax(s_cons[wid][1][i], xn[i][0]);
                        s_cons[wid][2][i] = fmin(s_cons[wid][2][i], xn[i][0]);
                    }
                }
            }
            __syncwarp();  // every lane is done reading the stage
            if (lane == 0 && ahead.u < s.U) {
                // refill the stage with this warp's chunk NS positions ahead
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                s2_issue<M, CT, L, BX>(tm, ahead.j, ahead.c, ring_s + st * C::STAGE, bar_s + 8 * st);
            }
            ahead.next(s, wid);
            if (++st == NS) {
                st = 0;
                ph ^= 1u;
            }
        }

        // ---- unit end: warp partials into slot b (free once unit - UB is finalised);
        // the last warp to arrive finalises
        const int b = (int)(unit & (S2_UB - 1));
        if (lane == 0)
            while (*(volatile unsigned*)&s_gen[b] != (unsigned)(unit / S2_UB)) __nanosleep(64);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const unsigned long long ws = warp_sum_u64((unsigned long long)fx[i]);
            if (lane == 0) s_fxw[b][wid][i] = ws;
            if (chk) {
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
            last = (atomicAdd(&s_arr[b], 1u) == (unsigned)S2_NW - 1);
            __threadfence_block();
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        __syncwarp();
        if (last) {
            if (lane < M) {
                const int i = lane;
                unsigned long long part = 0ull;
                double mx = -INFINITY, mn = INFINITY;
#pragma unroll
                for (int w = 0; w < S2_NW; ++w) {
                    part += s_fxw[b][w][i];
                    if (chk) {
                        mx = fmax(mx, s_dgw[b][w][i]);
                        mn = fmin(mn, s_dgw[b][w][M + i]);
                    }
                }
                bool fin = true;
                if (a.hz) {
                    // horizon blocks: this rank's partial row sum and dg extrema; the ranks'
                    // values are all-reduced after the sweep and hz_rows_kernel finalises
                    atomicAdd(a.rowacc + j * MAXM + i, part);
                    if (chk) {
                        atomicMax(a.hzdg + j * 2 * MAXM + i, okey(mx));
                        atomicMax(a.hzdg + j * 2 * MAXM + MAXM + i, okey(-mn));
                    }
                    fin = false;
                } else if (s.S > 1) {  // row split over segments: global exact sums, the last one finalises
                    atomicAdd(a.rowacc + j * MAXM + i, part);
                    if (chk) {
                        atomicMax(a.rowdg + j * 2 * MAXM + i, okey(mx));
                        atomicMin(a.rowdg + j * 2 * MAXM + MAXM + i, okey(mn));
                    }
                    __threadfence();
                    fin = (atomicAdd(a.rowcnt + j * MAXM + i, 1u) == (unsigned)s.S - 1);
                    if (fin) {
                        __threadfence();
                        part = atomicExch(a.rowacc + j * MAXM + i, 0ull);
                        if (chk) {
                            mx = okey_inv(atomicExch(a.rowdg + j * 2 * MAXM + i, 0ull));
                            mn = okey_inv(atomicExch(a.rowdg + j * 2 * MAXM + MAXM + i, ~0ull));
                        }
                        a.rowcnt[j * MAXM + i] = 0u;
                    }
                }
                if (fin) {
                    if ((a.gfree >> i) & 1u) mx = mn = 0.0;  // dg = 0 for every k
                    // (6b), (6g), (6d), (6i) for row (i, j) (PAPER.md:432-448 via I1)
                    const long long rix = (long long)i * a.q + j;
                    const RowOut o = row_update((double)(long long)part * a.fx_inv[i], sc[4][i],
                                                sc[0][i] * cin.f[0], sc[2][i] * cin.f[1], sc[3][i], sc[1][i],
                                                a.c[i], a.nd, cin.rho, mx, mn);
                    __stcg(a.lam + rix, o.lam);
                    __stcg(a.zeta + rix, o.zeta);
                    __stcg(a.h + rix, o.h);
                    __stcg(a.p + rix, o.p);
                    if (chk) {
                        double* rc = s_rc[wid][i];
                        rc[0] = fmax(rc[0], o.r2);
                        rc[1] = fmax(rc[1], o.r3);
                        rc[2] = fmax(rc[2], o.s1);
                        rc[3] = fmax(rc[3], o.s2);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) {
                s_arr[b] = 0u;
                __threadfence_block();
                atomicAdd(&s_gen[b], 1u);  // release the slot to unit + UB
            }
        }
    }

    // ---- per-CTA partials: consensus (warps in order) and the check maxima
    __syncthreads();
    if (tid < M) {
        double cs = 0.0, cx = -INFINITY, cn = INFINITY;
        for (int w = 0; w < S2_NW; ++w) {
            cs += s_cons[w][0][tid];
            cx = fmax(cx, s_cons[w][1][tid]);
            cn = fmin(cn, s_cons[w][2][tid]);
        }
        acc[tid] = cs;
        acc[MAXM + tid] = cx;
        acc[2 * MAXM + tid] = cn;
    }
    if (chk) {
        my_r1 = warp_max(my_r1);
        my_s3 = warp_max(my_s3);
        if (lane == 0) {
            s_red[wid][0] = my_r1;
            s_red[wid][1] = my_s3;
        }
    }
    __syncthreads();
    if (chk && tid == 0) {
        double r1 = 0.0, s3 = 0.0, r2 = 0.0, r3 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int w = 0; w < S2_NW; ++w) {
            r1 = fmax(r1, s_red[w][0]);
            s3 = fmax(s3, s_red[w][1]);
            for (int i = 0; i < M; ++i) {
                r2 = fmax(r2, s_rc[w][i][0]);
                r3 = fmax(r3, s_rc[w][i][1]);
                s1 = fmax(s1, s_rc[w][i][2]);
                s2 = fmax(s2, s_rc[w][i][3]);
            }
        }
        acc[3 * MAXM + 0] = r1;
        acc[3 * MAXM + 1] = r2;
        acc[3 * MAXM + 2] = r3;
        acc[3 * MAXM + 3] = s1;
        acc[3 * MAXM + 4] = s2;
        acc[3 * MAXM + 5] = s3;
    }
    __syncthreads();
    if (tid < XB) __stcg(a.cta_part + (size_t)blockIdx.x * XB + tid, acc[tid]);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(a.glob_cnt, 1) == s.G - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // ---- last CTA: reduce the G CTA partials; lane = slot, warp w takes CTAs w, w + NW,
    // ... 32 loads in flight per lane per pass (the pass count, not the bytes, sets this
    // tail's latency: G = 592 at q = 1e3 takes 5 L2 round trips instead of 19), folded
    // into eight accumulators in a fixed order (fixed assignment => deterministic)
    {
        __shared__ double wred[S2_NW][XB];
        const int sl = lane;
        const bool is_sum = sl < MAXM;
        const bool is_min = sl >= 2 * MAXM && sl < 3 * MAXM;
        const double ident = is_sum ? 0.0 : (is_min ? INFINITY : (sl >= 3 * MAXM ? 0.0 : -INFINITY));
        double vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) vv[u] = ident;
        for (int g0 = wid; g0 < s.G; g0 += 32 * S2_NW) {
            double t[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const int g = g0 + u * S2_NW;
                t[u] = g < s.G ? __ldcg(a.cta_part + (size_t)g * XB + sl) : ident;
            }
#pragma unroll
            for (int u = 0; u < 32; ++u)
                vv[u & 7] = is_sum ? vv[u & 7] + t[u] : (is_min ? fmin(vv[u & 7], t[u]) : fmax(vv[u & 7], t[u]));
        }
        double vr = vv[0];
#pragma unroll
        for (int u = 1; u < 8; ++u) vr = is_sum ? vr + vv[u] : (is_min ? fmin(vr, vv[u]) : fmax(vr, vv[u]));
        wred[wid][sl] = vr;
        __syncthreads();
        if (tid < XB) {
            double r = ident;
            for (int w = 0; w < S2_NW; ++w) {
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
        if (!a.dist) {
            Ctrl& cout = a.ctrl[(it + 1) & 1];
            finalize_global(a, acc, 1, it, cin, cout, chk);
            __threadfence();
            *(volatile long long*)a.iter = it + 1;
        }
    }
}

// Horizon-block sharding: after the sweep the m q fixed-point row
// sums (rowacc) and dg extrema (hzdg) have been all-reduced over the ranks; every
// rank finalises every row identically ((6b), (6g), (6d), (6i) via identity I1,
// PAPER.md:432-448), adds the row check terms to the all-gathered aggregates and
// runs the check / rho adaptation (finalize_global).  One CTA of 256 threads.
#ifndef ADMM_KERNELS_NO_GLOBALS  // defined once, in admm.cu's translation unit
__global__ void __launch_bounds__(256) hz_rows_kernel(KArgs a) {
    __shared__ double red[8][4];
    const long long it = *(volatile long long*)a.iter;
    const Ctrl& cin = a.ctrl[it & 1];
    if (cin.done || it >= a.prm->iter_limit) return;
    const int ce = a.prm->check_every;
    const bool chk = ce > 0 && ((it + 1) % ce) == 0;
    double r2 = 0.0, r3 = 0.0, s1 = 0.0, s2 = 0.0;
    const long long R = (long long)a.m * a.q;
    for (long long rix = threadIdx.x; rix < R; rix += blockDim.x) {
        const int i = (int)(rix / a.q);
        const long long j = rix - (long long)i * a.q;
        const unsigned long long part = a.rowacc[j * MAXM + i];
        a.rowacc[j * MAXM + i] = 0ull;
        double mx = okey_inv(a.hzdg[j * 2 * MAXM + i]);
        double mn = -okey_inv(a.hzdg[j * 2 * MAXM + MAXM + i]);
        a.hzdg[j * 2 * MAXM + i] = 0ull;
        a.hzdg[j * 2 * MAXM + MAXM + i] = 0ull;
        if (((a.gfree >> i) & 1u) || !chk) mx = mn = 0.0;  // dg = 0 (g-free), unused (no check)
        const RowOut o = row_update((double)(long long)part * a.fx_inv[i], a.sb0[rix], a.lam[rix] * cin.f[0],
                                    a.p[rix] * cin.f[1], a.h[rix], a.zeta[rix], a.c[i], a.nd, cin.rho, mx, mn);
        a.lam[rix] = o.lam;
        a.zeta[rix] = o.zeta;
        a.h[rix] = o.h;
        a.p[rix] = o.p;
        r2 = fmax(r2, o.r2);
        r3 = fmax(r3, o.r3);
        s1 = fmax(s1, o.s1);
        s2 = fmax(s2, o.s2);
    }
    if (chk) {
        r2 = warp_max(r2);
        r3 = warp_max(r3);
        s1 = warp_max(s1);
        s2 = warp_max(s2);
        if ((threadIdx.x & 31) == 0) {
            red[threadIdx.x >> 5][0] = r2;
            red[threadIdx.x >> 5][1] = r3;
            red[threadIdx.x >> 5][2] = s1;
            red[threadIdx.x >> 5][3] = s2;
        }
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (chk) {
        // the ranks reported no row terms (no row was finalised in the sweep): rank 0's
        // slots carry the rows' terms, identical on every rank
        double* g = a.xall;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            g[3 * MAXM + 1] = fmax(g[3 * MAXM + 1], red[w][0]);
            g[3 * MAXM + 2] = fmax(g[3 * MAXM + 2], red[w][1]);
            g[3 * MAXM + 3] = fmax(g[3 * MAXM + 3], red[w][2]);
            g[3 * MAXM + 4] = fmax(g[3 * MAXM + 4], red[w][3]);
        }
    }
    finalize_global(a, a.xall, a.world, it, cin, a.ctrl[(it + 1) & 1], chk);
    __threadfence();
    *(volatile long long*)a.iter = it + 1;
}
#endif

// host side (sweep2.cu): kernel pointer, stage count and dynamic shared memory
// for (m, box mode, coefficient bytes); nullptr when m is not supported
// and the chunk length it streams (64 cells: two per lane, or 32 with the box staged)
const void* sweep2_pick(int m, int mode, int coeff_bytes, long long q, int* ns, size_t* smem, int* tl);
// work decomposition for q rows of n_pad cells in chunks of tl over at most g_max CTAs
S2Args sweep2_plan(long long q, long long n_pad, int tl, int g_max);

}  // namespace admm_dev
