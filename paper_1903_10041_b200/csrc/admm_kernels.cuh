// admm_kernels.cuh -- device code of the per-iteration ADMM hot path
// (Appendix A, Eq. (6a)-(6i), residuals :464-479, adaptive rho
// :318-324) for sm_100a, fp64.
//
// One kernel launch = one ADMM iteration ("sweep"):
//   * a persistent grid of G CTAs walks work items (scenario j, horizon tile)
//     in a fixed round-robin order (static => deterministic); three layouts
//     (DESIGN.md §6): the row loop (RLT = 128: small CTAs, four per SM, each
//     owning whole rows -- the default for m <= 2 with many rows), the staged
//     four-cell CTA (U = 4) and the two-cell 512-thread CTA (m > 2);
//   * each thread owns U = 2 (or 4) consecutive steps k of one scenario (128-bit
//     double2 loads/stores of every SoA stream) and runs the Gauss-Seidel loop
//     over sources i in registers: build the (6a) quartic, Algorithm 1, box;
//   * (6e)/(6f) per cell in-thread (reduced state v = s - mu, identity I2);
//   * (6b)/(6g)/(6d)/(6i) per row (i,j) from a deterministic block reduction of
//     sum_k g(x_k) (identity I1: lam constant over k, z = g(x) + zeta);
//     rows longer than one tile are finalised by the last-arriving tile CTA;
//   * (6c) consensus partial sums and the residual maxima per CTA; the last
//     CTA to arrive reduces them in CTA order, computes x1, r, sigma, the
//     termination test and the rho adaptation, and writes the control block
//     of the next iteration.  (6h) and the dual rescale are applied lazily by
//     the next sweep when it loads nu / lam / p / mu.
// DESIGN.md "Kernels" gives the byte model and the readings.
#pragma once
#include <cstdint>

#include "quartic.cuh"

namespace admm_dev {

constexpr int MAXM = 8;
constexpr int CPT = 2;          // cells (steps k) per thread: one double2
constexpr int XB = 3 * MAXM + 8; // = 32 per-rank aggregate slots: cons[M], x0max[M], x0min[M], r1..r3, s1..s3
static_assert(XB == 32, "one warp lane per aggregate slot");
constexpr int HCOLS = 16;

struct Ctrl {
    double rho[4];   // rho used by the iteration that reads this block
    double f[4];     // pending rescale of lam, p, mu, nu (rho_old / rho_new)
    double x1[MAXM]; // consensus x1 of the previous iteration
    double r, sigma; // last check
    int nu_pending;  // apply (6h) of the previous iteration on load
    int done;        // solve converged or numerical error: kernels no-op
    int status;      // last check met the thresholds
    int checks;      // checks done
    int err;         // NaN / Inf in r or sigma
    int pad[3];
};

struct DParams {
    double tau, hi_ratio, lo_ratio, r_bar, sigma_bar;
    long long iter_limit;  // sweeps with iter >= iter_limit are no-ops
    int check_every, adapt, rescale, box_mode, stop_on_conv, pad;
};

struct KArgs {
    int m, n, n_pad, T, tile, G, world, rank;
    int dist;   // collective path (admm_dist given): kernels write xsend, finalize_kernel finishes
    int hz;     // horizon-block sharding: row sums are all-reduced, hz_rows_kernel finalises rows
    int k0own;  // this rank holds the consensus cell k = 1 (global k = 0)
    double nd;  // horizon length n of the whole problem (row length in (6b), kappa)
    long long q, q_total;
    double inv_q;
    // problem (padded SoA)
    const double *a2, *a1, *a0, *b2, *b1, *b0;  // [m][q][n_pad]
    const double *lo, *hi;                      // [m][n_pad]
    const double *y;                            // [q][n_pad]
    const double *c;                            // [m]
    const double *sb0;                          // [m][q]  sum_k b0
    // reduced state
    double *x;                                  // [m][q][n_pad]
    double *v;                                  // [q][n_pad]   s - mu
    double *lam, *zeta, *h, *p, *nu;            // [m][q]
    // scratch
    double *cta_part;                           // [G][XB]
    double *row_part;                           // [m][q][T][3]
    int *row_cnt;                               // [q]
    int *glob_cnt;                              // [1]
    double *xsend, *xall;                       // [XB], [world][XB]
    Ctrl *ctrl;                                 // [2]
    long long *iter;                            // [1] iterations done
    const DParams *prm;
    double *hist;
    int hist_cap;
    // fixed-point row sums (streaming sweep, FX variant): scale 2^E_i, accumulators for
    // rows split over tiles (kept zero between uses), see admm_onchip.cuh / DESIGN.md §5
    double fx_scale[MAXM], fx_inv[MAXM];
    unsigned long long *rowacc;  // [q][MAXM]
    unsigned long long *rowdg;   // [q][2 MAXM] ordered keys (checks)
    unsigned *rowcnt;            // [q][MAXM]
    unsigned long long *hzdg;    // [q][2 MAXM] horizon mode: max keys of dg, of -dg (zero between uses)
    unsigned gfree;              // bit i: g^{(i)} = 0 on the box (row sums 0, no capacity bookkeeping)
    // F2: fp32 copies of the per-element coefficients, read by the
    // streaming sweep when the context stores coefficients in fp32 (admm_set_coeff_precision)
    const float *fa2, *fa1, *fb2, *fb1;          // [m][q][n_pad]
};

// two consecutive coefficients (k, k+1) of a stream stored as CT, widened to fp64
template <typename CT>
__device__ __forceinline__ void ld2(const CT* p, double* o);
template <>
__device__ __forceinline__ void ld2<double>(const double* p, double* o) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = t.x;
    o[1] = t.y;
}
template <>
__device__ __forceinline__ void ld2<float>(const float* p, double* o) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(p));
    o[0] = (double)t.x;
    o[1] = (double)t.y;
}

// order-preserving map double -> uint64 (max/min of keys = max/min of values)
__device__ __forceinline__ unsigned long long okey(double x) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(x);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
    const unsigned long long u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)u);
}

// exact warp sum of 64-bit two's-complement values (mod 2^64): three 21/21/22-bit
// limbs, each summed by redux.sync (no carries lost: 32 * 2^22 < 2^32)
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
    const unsigned l0 = __reduce_add_sync(0xffffffffu, (unsigned)(v & 0x1FFFFFull));
    const unsigned l1 = __reduce_add_sync(0xffffffffu, (unsigned)((v >> 21) & 0x1FFFFFull));
    const unsigned l2 = __reduce_add_sync(0xffffffffu, (unsigned)(v >> 42));
    return (unsigned long long)l0 + ((unsigned long long)l1 << 21) + ((unsigned long long)l2 << 42);
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ------------------------------------------------ per-cell / per-row math
// (6a) for one cell (j,k): Gauss-Seidel over sources i = 0..M-1
// (PAPER.md:423-429 in the theta/phi form :452-463; reading G2).
//   phi   = s - sum_{l != i} x^{(l)} + y + mu   (new x for l < i, old for l > i)
//   e     = theta - b0 = g(x_old) + zeta + lam - b0      (identity I1: z = g(x) + zeta)
//   A..D  = coefficients of the (6a) quartic
// zl[i] = zeta + lam_e of row (i,j); x1nu[i] = x1 + nu_e (used when k0).
template <int M, int MODE>
__device__ __forceinline__ void gs_cell(const double* ca2, const double* ca1, const double* cb2,
                                        const double* cb1, const double* clo, const double* chi,
                                        const double* xo, double* xn, double y, double s_e,
                                        double mu_e, const double* zl, const double* rho, double iq,
                                        bool k0, const double* x1nu) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double others = 0.0;
#pragma unroll
        for (int l = 0; l < M; ++l)
            if (l != i) others += (l < i) ? xn[l] : xo[l];
        const double phi = ((s_e - others) + y) + mu_e;
        const double xoi = xo[i];
        const double b2 = cb2[i], b1 = cb1[i];
        const double e = fma(fma(b2, xoi, b1), xoi, zl[i]);
        double C = fma(0.5 * rho[0], fma(b1, b1, -2.0 * b2 * e), fma(ca2[i], iq, 0.5 * rho[2]));
        double D = fma(-rho[0] * b1, e, fma(ca1[i], iq, -rho[2] * phi));
        if (k0) {
            C += 0.5 * rho[3];
            D += -rho[3] * x1nu[i];
        }
        if (b2 != 0.0) {
            // A = rho1 b2^2 / 2, B = rho1 b2 b1: b = 3B/4A, c = C/2A, d = D/4A
            const double ia2 = rcp_nr(rho[0] * b2 * b2);  // 1 / 2A
            xn[i] = quartic_core<MODE>(1.5 * (rho[0] * b2 * b1) * ia2, C * ia2, 0.5 * D * ia2, C, D,
                                       clo[i], chi[i]);
        } else {
            xn[i] = clampd(-D * rcp_nr(2.0 * C), clo[i], chi[i]);  // A = B = 0: quadratic
        }
    }
}

// Same update from per-element constants prepared once per problem (on-chip
// engines): a2q = a2/q, a1q = a1/q, bq = 1.5 b1/b2 (= b, independent of rho),
// ib2s = 1/b2^2 (0 when b2 = 0).  R = {rho1, rho3, rho4, 1/rho1}.
template <int M, int MODE>
__device__ __forceinline__ void gs_cell_prep(const double* a2q, const double* a1q, const double* cb2,
                                             const double* cb1, const double* bq, const double* ib2s,
                                             const double* clo, const double* chi, const double* xo,
                                             double* xn, double y, double s_e, double mu_e,
                                             const double* zl, const double* R, bool k0,
                                             const double* x1nu) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double others = 0.0;
#pragma unroll
        for (int l = 0; l < M; ++l)
            if (l != i) others += (l < i) ? xn[l] : xo[l];
        const double phi = ((s_e - others) + y) + mu_e;
        const double xoi = xo[i];
        const double b2 = cb2[i], b1 = cb1[i];
        const double e = fma(fma(b2, xoi, b1), xoi, zl[i]);
        double C = fma(0.5 * R[0], fma(b1, b1, -2.0 * b2 * e), a2q[i] + 0.5 * R[1]);
        double D = fma(-R[0] * b1, e, fma(-R[1], phi, a1q[i]));
        if (k0) {
            C += 0.5 * R[2];
            D += -R[2] * x1nu[i];
        }
        if (b2 != 0.0) {
            const double ia2 = ib2s[i] * R[3];  // 1 / 2A = 1 / (rho1 b2^2)
            xn[i] = quartic_core<MODE>(bq[i], C * ia2, 0.5 * D * ia2, C, D, clo[i], chi[i]);
        } else {
            xn[i] = clampd(-D * rcp_nr(2.0 * C), clo[i], chi[i]);
        }
    }
}

// gs_cell_prep on two cells (c[0], c[1]) of one thread with interleaved chains
// (on-chip engines).  Coefficients are read from the shared-memory tile (row
// stride TCM) where they are used, which keeps the two-cell register footprint
// small; xo/xn are [M][2].  Never the consensus cell.
template <int M, int MODE>
__device__ __forceinline__ void gs_cell2_smem(const double* s_a2q, const double* s_a1q,
                                              const double* s_b2, const double* s_b1,
                                              const double* s_bq, const double* s_ib,
                                              const double* s_lo, const double* s_hi, int TCM,
                                              const int* c, const double (*xo)[2], double (*xn)[2],
                                              const double* y, const double* s_e,
                                              const double* mu_e, const double* zl,
                                              const double* R) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double C[2], D[2], cn[2], dn[2], bn[2], lo[2], hi[2];
        bool quart[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int e = i * TCM + c[u];
            double others = 0.0;
#pragma unroll
            for (int l = 0; l < M; ++l)
                if (l != i) others += (l < i) ? xn[l][u] : xo[l][u];
            const double phi = ((s_e[u] - others) + y[u]) + mu_e[u];
            const double xoi = xo[i][u];
            const double b2 = s_b2[e], b1 = s_b1[e];
            const double ee = fma(fma(b2, xoi, b1), xoi, zl[i]);
            C[u] = fma(0.5 * R[0], fma(b1, b1, -2.0 * b2 * ee), s_a2q[e] + 0.5 * R[1]);
            D[u] = fma(-R[0] * b1, ee, fma(-R[1], phi, s_a1q[e]));
            quart[u] = (b2 != 0.0);
            const double ia2 = s_ib[e] * R[3];
            bn[u] = s_bq[e];
            cn[u] = C[u] * ia2;
            dn[u] = 0.5 * D[u] * ia2;
            lo[u] = s_lo[e];
            hi[u] = s_hi[e];
        }
        if (quart[0] && quart[1]) {
            double r[2];
            quartic_core2<MODE>(bn, cn, dn, C, D, lo, hi, r);
            xn[i][0] = r[0];
            xn[i][1] = r[1];
        } else {
#pragma unroll
            for (int u = 0; u < 2; ++u)
                xn[i][u] = quart[u] ? quartic_core<MODE>(bn[u], cn[u], dn[u], C[u], D[u], lo[u], hi[u])
                                    : clampd(-D[u] * rcp_nr(2.0 * C[u]), lo[u], hi[u]);
        }
    }
}

// U consecutive values of a stream (U = 2: one 128-bit load, U = 4: two)
template <typename CT, int U>
__device__ __forceinline__ void ldU(const CT* p, double* o) {
#pragma unroll
    for (int h = 0; h < U; h += 2) ld2<CT>(p + h, o + h);
}
// read-write state (x, v): plain (L1-coherent) 128-bit loads
template <int U>
__device__ __forceinline__ void ldvU(const double* p, double* o) {
#pragma unroll
    for (int h = 0; h < U; h += 2) {
        const double2 t = *reinterpret_cast<const double2*>(p + h);
        o[h] = t.x;
        o[h + 1] = t.y;
    }
}
template <int U>
__device__ __forceinline__ void stU(double* p, const double* v) {
#pragma unroll
    for (int h = 0; h < U; h += 2) *reinterpret_cast<double2*>(p + h) = make_double2(v[h], v[h + 1]);
}

// Algorithm 1 on U independent cells: when all take the trigonometric branch the U
// straight-line evaluations interleave (ILP U); results bit-identical to quartic_core.
template <int MODE, int U>
__device__ __forceinline__ void quartic_coreU(const double* b, const double* c, const double* d,
                                              const double* C, const double* D, const double* lo,
                                              const double* hi, double* out) {
    double Q[U], R[U], De[U];
    bool all = true;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const double bb = b[u] * b[u];
        Q[u] = fma(3.0, c[u], -bb) * (1.0 / 9.0);
        R[u] = fma(b[u], fma(9.0, c[u], -2.0 * bb), -27.0 * d[u]) * (1.0 / 54.0);
        De[u] = fma(Q[u] * Q[u], Q[u], R[u] * R[u]);
        all = all && isfinite(De[u]) && !(De[u] > 0.0) && !(Q[u] == 0.0 && R[u] == 0.0);
    }
    if (all) {
#pragma unroll
        for (int u = 0; u < U; ++u) out[u] = trig_pick<MODE>(b[u], c[u], d[u], Q[u], R[u], De[u], lo[u], hi[u]);
    } else {
#pragma unroll
        for (int u = 0; u < U; ++u) out[u] = quartic_core<MODE>(b[u], c[u], d[u], C[u], D[u], lo[u], hi[u]);
    }
}

// (6a) for U cells of one thread (arrays [M][U], cell index last): source i of all
// U cells is built, then minimised together (quartic_coreU: straight-line trig
// evaluations that the scheduler interleaves); same arithmetic as U gs_cell calls.
// k0 marks cell 0 as the consensus cell.
template <int M, int MODE, int U>
__device__ __forceinline__ void gs_cellU(const double (*ca2)[U], const double (*ca1)[U],
                                         const double (*cb2)[U], const double (*cb1)[U],
                                         const double (*clo)[U], const double (*chi)[U],
                                         const double (*xo)[U], double (*xn)[U], const double* y,
                                         const double* s_e, const double* mu_e, const double* zl,
                                         const double* rho, double iq, bool k0, const double* x1nu) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double C[U], D[U], bn[U], cn[U], dn[U], lo[U], hi[U];
        bool allq = true, anyq = false;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double others = 0.0;
#pragma unroll
            for (int l = 0; l < M; ++l)
                if (l != i) others += (l < i) ? xn[l][u] : xo[l][u];
            const double phi = ((s_e[u] - others) + y[u]) + mu_e[u];
            const double xoi = xo[i][u];
            const double b2 = cb2[i][u], b1 = cb1[i][u];
            const double e = fma(fma(b2, xoi, b1), xoi, zl[i]);
            C[u] = fma(0.5 * rho[0], fma(b1, b1, -2.0 * b2 * e), fma(ca2[i][u], iq, 0.5 * rho[2]));
            D[u] = fma(-rho[0] * b1, e, fma(ca1[i][u], iq, -rho[2] * phi));
            if (k0 && u == 0) {
                C[u] += 0.5 * rho[3];
                D[u] += -rho[3] * x1nu[i];
            }
            const bool qu = (b2 != 0.0);
            allq = allq && qu;
            anyq = anyq || qu;
            const double ia2 = rcp_nr(qu ? rho[0] * b2 * b2 : 1.0);  // 1 / 2A
            bn[u] = 1.5 * (rho[0] * b2 * b1) * ia2;
            cn[u] = C[u] * ia2;
            dn[u] = 0.5 * D[u] * ia2;
            lo[u] = clo[i][u];
            hi[u] = chi[i][u];
        }
        if (allq) {
            double r[U];
            quartic_coreU<MODE, U>(bn, cn, dn, C, D, lo, hi, r);
#pragma unroll
            for (int u = 0; u < U; ++u) xn[i][u] = r[u];
        } else if (!anyq) {  // a source without g (A = B = 0): quadratic for every cell
#pragma unroll
            for (int u = 0; u < U; ++u) xn[i][u] = clampd(-D[u] * rcp_nr(2.0 * C[u]), lo[u], hi[u]);
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u)
                xn[i][u] = (cb2[i][u] != 0.0) ? quartic_core<MODE>(bn[u], cn[u], dn[u], C[u], D[u], lo[u], hi[u])
                                              : clampd(-D[u] * rcp_nr(2.0 * C[u]), lo[u], hi[u]);
        }
    }
}

// ------------------------------------------- staged 4-cell Gauss-Seidel (U = 4)
// The per-cell values that live across Algorithm 1 (x old/new, y, v and the
// normalised cubic of the source being solved) sit in a per-thread shared-memory
// slab instead of registers, and the coefficient streams are read (L1/L2) where
// they are used, so the four interleaved trigonometric chains get the register
// file.  Slab: field f, thread t, cell u at ((f * bs + t) * 4 + u) doubles.
template <int M>
struct Slab4 {
    static constexpr int XO = 0, XN = M, Y = 2 * M, V = 2 * M + 1, BN = 2 * M + 2, CN = 2 * M + 3,
                         DN = 2 * M + 4, CC = 2 * M + 5, DD = 2 * M + 6, NF = 2 * M + 7;
};
__device__ __forceinline__ void rd4(const double* p, double* o) {
    const double2 t0 = *reinterpret_cast<const double2*>(p), t1 = *reinterpret_cast<const double2*>(p + 2);
    o[0] = t0.x; o[1] = t0.y; o[2] = t1.x; o[3] = t1.y;
}
__device__ __forceinline__ void wr4(double* p, const double* v) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
}

// Same arithmetic, in the same order, as gs_cellU<M, MODE, 4> (bit-identical);
// inputs XO, Y, V in the slab, output XN in the slab.  e0 = j * n_pad + kl.
template <int M, int MODE, typename CT>
__device__ __forceinline__ void staged_gs4(const KArgs& a, double* slab, int bs, int tid, long long e0,
                                           long long qn, long long bk0, const double* zl,
                                           const double* rho, double iq, bool k0, const double* x1nu,
                                           double f2) {
    using SL = Slab4<M>;
    auto S = [&](int f) { return slab + ((size_t)f * bs + tid) * 4; };
    const CT *pa2, *pa1, *pb2, *pb1;
    if constexpr (sizeof(CT) == 4) {
        pa2 = a.fa2; pa1 = a.fa1; pb2 = a.fb2; pb1 = a.fb1;
    } else {
        pa2 = reinterpret_cast<const CT*>(a.a2); pa1 = reinterpret_cast<const CT*>(a.a1);
        pb2 = reinterpret_cast<const CT*>(a.b2); pb1 = reinterpret_cast<const CT*>(a.b1);
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
        bool qf[4];
        bool allq = true, anyq = false;
        {
            double b2[4], b1[4], a2[4], a1[4], xoi[4], y[4], v[4], oth[4] = {0.0, 0.0, 0.0, 0.0};
            const long long e = (long long)i * qn + e0;
            ldU<CT, 4>(pb2 + e, b2);
            ldU<CT, 4>(pb1 + e, b1);
            ldU<CT, 4>(pa2 + e, a2);
            ldU<CT, 4>(pa1 + e, a1);
            rd4(S(SL::XO + i), xoi);
            rd4(S(SL::Y), y);
            rd4(S(SL::V), v);
#pragma unroll
            for (int l = 0; l < M; ++l) {
                if (l == i) continue;
                double t[4];
                rd4(S(l < i ? SL::XN + l : SL::XO + l), t);
#pragma unroll
                for (int u = 0; u < 4; ++u) oth[u] += t[u];
            }
            double bn[4], cn[4], dn[4], C[4], D[4], xq[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double s_e = fmax(v[u], 0.0);
                const double mu_e = v[u] < 0.0 ? -v[u] * f2 : 0.0;
                const double phi = ((s_e - oth[u]) + y[u]) + mu_e;
                const double ee = fma(fma(b2[u], xoi[u], b1[u]), xoi[u], zl[i]);
                C[u] = fma(0.5 * rho[0], fma(b1[u], b1[u], -2.0 * b2[u] * ee), fma(a2[u], iq, 0.5 * rho[2]));
                D[u] = fma(-rho[0] * b1[u], ee, fma(a1[u], iq, -rho[2] * phi));
                if (k0 && u == 0) {
                    C[u] += 0.5 * rho[3];
                    D[u] += -rho[3] * x1nu[i];
                }
                qf[u] = (b2[u] != 0.0);
                allq = allq && qf[u];
                anyq = anyq || qf[u];
                const double ia2 = rcp_nr(qf[u] ? rho[0] * b2[u] * b2[u] : 1.0);  // 1 / 2A
                bn[u] = 1.5 * (rho[0] * b2[u] * b1[u]) * ia2;
                cn[u] = C[u] * ia2;
                dn[u] = 0.5 * D[u] * ia2;
            }
            if (!allq) {  // quadratic cells (A = B = 0) are finished here
                double lo[4], hi[4];
                ldU<double, 4>(a.lo + (long long)i * a.n_pad + bk0, lo);
                ldU<double, 4>(a.hi + (long long)i * a.n_pad + bk0, hi);
#pragma unroll
                for (int u = 0; u < 4; ++u) xq[u] = qf[u] ? 0.0 : clampd(-D[u] * rcp_nr(2.0 * C[u]), lo[u], hi[u]);
                wr4(S(SL::XN + i), xq);
            }
            if (anyq) {
                wr4(S(SL::BN), bn);
                wr4(S(SL::CN), cn);
                wr4(S(SL::DN), dn);
                wr4(S(SL::CC), C);
                wr4(S(SL::DD), D);
            }
        }
        if (anyq) {
            double bn[4], cn[4], dn[4], C[4], D[4], lo[4], hi[4], r[4];
            rd4(S(SL::BN), bn);
            rd4(S(SL::CN), cn);
            rd4(S(SL::DN), dn);
            rd4(S(SL::CC), C);
            rd4(S(SL::DD), D);
            ldU<double, 4>(a.lo + (long long)i * a.n_pad + bk0, lo);
            ldU<double, 4>(a.hi + (long long)i * a.n_pad + bk0, hi);
            if (allq) {
                quartic_coreU<MODE, 4>(bn, cn, dn, C, D, lo, hi, r);
                wr4(S(SL::XN + i), r);
            } else {
                double xq[4];
                rd4(S(SL::XN + i), xq);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (qf[u]) xq[u] = quartic_core<MODE>(bn[u], cn[u], dn[u], C[u], D[u], lo[u], hi[u]);
                wr4(S(SL::XN + i), xq);
            }
        }
    }
}

// (6e)/(6f) for one cell with the reduced state v = s - mu (identity I2);
// returns v_new and updates the check maxima |s - sum x + y| and
// |(s - s~) - sum_i (x - x~)|.
template <int M>
__device__ __forceinline__ double cell_tail(const double* xo, const double* xn, double y,
                                            double v_old, double f3, bool chk, double& r1,
                                            double& s3) {
    double sx = 0.0, dx = 0.0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        sx += xn[i];
        dx += xn[i] - xo[i];
    }
    const double mu_e = v_old < 0.0 ? -v_old * f3 : 0.0;
    const double s_o = fmax(v_old, 0.0);
    const double vnew = (sx - y) - mu_e;
    if (chk) {
        const double s_n = fmax(vnew, 0.0);
        r1 = fmax(r1, fabs((s_n - sx) + y));
        s3 = fmax(s3, fabs((s_n - s_o) - dx));
    }
    return vnew;
}

// Row (i,j) update from Sg = sum_k (b2 x^2 + b1 x) (PAPER.md:432-448 via I1):
//   W = Sg + sum_k b0 - n lam,  t = h + p - W,  lam' = kappa t  (kappa = rho2/(rho1 + n rho2)),
//   zeta' = lam' - lam,  1'z = W + n lam',  h' = min(c, 1'z - p),  p' = p + h' - 1'z.
struct RowOut {
    double lam, zeta, h, p;   // new values
    double r2, r3, s1, s2;    // check terms: |z - g|, |h - 1'z|, max_k |dz|, |dh|
};
__device__ __forceinline__ RowOut row_update(double Sg, double sb0, double lam_e, double p_e,
                                             double h_o, double zeta_o, double c, double nd,
                                             const double* rho, double dgmax, double dgmin) {
    RowOut o;
    const double W = (Sg + sb0) - nd * lam_e;
    const double kap = rho[1] / (rho[0] + nd * rho[1]);
    const double t = (h_o + p_e) - W;
    o.lam = kap * t;
    o.zeta = o.lam - lam_e;
    const double oneTz = W + nd * o.lam;
    o.h = fmin(c, oneTz - p_e);
    o.p = (p_e + o.h) - oneTz;
    const double dz = o.zeta - zeta_o;
    o.r2 = fabs(o.zeta);
    o.r3 = fabs(o.h - oneTz);
    o.s1 = fmax(dgmax + dz, -(dgmin + dz));
    o.s2 = fabs(o.h - h_o);
    return o;
}

// rho adaptation + termination at a check (readings
// G10-G12).  t = {r1..r4, raw sigma terms}.  Returns conv; writes rho_new, f.
__device__ __forceinline__ int check_decide(const DParams& P, const double* rho, const double* t,
                                            double* rho_new, double* f, double* r_out,
                                            double* s_out, double* fac_out, double* s123) {
    const double s1 = rho[0] * t[4], s2 = rho[1] * t[5], s3 = rho[2] * t[6];
    const double r = fmax(fmax(t[0], t[1]), fmax(t[2], t[3]));
    const double sg = fmax(s1, fmax(s2, s3));
    const int conv = (r < P.r_bar) && (sg < P.sigma_bar);
    double fac = 1.0;
    for (int l = 0; l < 4; ++l) {
        rho_new[l] = rho[l];
        f[l] = 1.0;
    }
    if (!conv && P.adapt) {
        const double thr_hi = P.hi_ratio * P.r_bar / P.sigma_bar;
        const double thr_lo = P.lo_ratio * P.r_bar / P.sigma_bar;
        const double ratio = (sg > 0.0) ? r / sg : INFINITY;  // reading G12
        int dir = 0;
        if (ratio > thr_hi) dir = 1;
        else if (ratio < thr_lo) dir = -1;
        if (dir != 0) {
            for (int l = 0; l < 4; ++l) {
                const double old = rho[l];
                const double nw = dir > 0 ? old * P.tau : old / P.tau;
                rho_new[l] = nw;
                f[l] = P.rescale ? old / nw : 1.0;
            }
            fac = dir > 0 ? P.tau : 1.0 / P.tau;
        }
    }
    *r_out = r;
    *s_out = sg;
    *fac_out = fac;
    s123[0] = s1;
    s123[1] = s2;
    s123[2] = s3;
    return conv;
}

__device__ __forceinline__ void write_hist(double* h, long long it1, double r, double sg,
                                           const double* rho, const double* t, const double* s123,
                                           int conv, double fac) {
    h[0] = (double)it1;
    h[1] = r;
    h[2] = sg;
    for (int l = 0; l < 4; ++l) h[3 + l] = rho[l];
    for (int l = 0; l < 4; ++l) h[7 + l] = t[l];
    h[11] = s123[0];
    h[12] = s123[1];
    h[13] = s123[2];
    h[14] = conv;
    h[15] = fac;
}

// ------------------------------------------------------- global finalisation
// Consumes the per-rank aggregates (rank order), computes (6c), the residuals
// r / sigma, the termination test and the rho adaptation, and writes the next
// control block.  Runs on one thread.
__device__ inline void finalize_global(const KArgs& a, const double* agg, int world, long long it,
                                const Ctrl& cin, Ctrl& cout, bool is_check) {
    const DParams& P = *a.prm;
    const int m = a.m;
    // (6c) PAPER.md:436 with the mean (reading G1): x1 = (1/q) sum_j (x_1 - nu)
    // loops over MAXM with a predicate (not over m): constant indices keep x1n and t in
    // registers (no local memory in the sweep kernels that inline this)
    double x1n[MAXM];
#pragma unroll
    for (int i = 0; i < MAXM; ++i) {
        double s = 0.0;
        if (i < m)
            for (int r = 0; r < world; ++r) s += agg[r * XB + i];
        x1n[i] = s / (double)a.q_total;
    }
    for (int l = 0; l < 4; ++l) {
        cout.rho[l] = cin.rho[l];
        cout.f[l] = 1.0;
    }
#pragma unroll
    for (int i = 0; i < MAXM; ++i) cout.x1[i] = i < m ? x1n[i] : 0.0;
    cout.r = cin.r;
    cout.sigma = cin.sigma;
    cout.nu_pending = 1;
    cout.done = cin.done;
    cout.status = cin.status;
    cout.checks = cin.checks;
    cout.err = cin.err;
    if (is_check) {
        double t[7] = {0, 0, 0, 0, 0, 0, 0};
        for (int r = 0; r < world; ++r) {
            const double* g = agg + r * XB;
            t[0] = fmax(t[0], g[3 * MAXM + 0]);
            t[1] = fmax(t[1], g[3 * MAXM + 1]);
            t[2] = fmax(t[2], g[3 * MAXM + 2]);
#pragma unroll
            for (int i = 0; i < MAXM; ++i) {
                // max_j |x_1^{(i,j)} - x1| = max(max_j x_1 - x1, x1 - min_j x_1) exactly
                if (i < m) t[3] = fmax(t[3], fmax(g[MAXM + i] - x1n[i], x1n[i] - g[2 * MAXM + i]));
            }
            t[4] = fmax(t[4], g[3 * MAXM + 3]);
            t[5] = fmax(t[5], g[3 * MAXM + 4]);
            t[6] = fmax(t[6], g[3 * MAXM + 5]);
        }
        double rn[4], fl[4], r, sg, fac, s123[3];
        const int conv = check_decide(P, cin.rho, t, rn, fl, &r, &sg, &fac, s123);
        for (int l = 0; l < 4; ++l) {
            cout.rho[l] = rn[l];
            cout.f[l] = fl[l];
        }
        cout.r = r;
        cout.sigma = sg;
        cout.status = conv;
        cout.checks = cin.checks + 1;
        if (!isfinite(r) || !isfinite(sg)) {
            cout.err = 1;
            cout.done = 1;
        }
        if (conv && P.stop_on_conv) cout.done = 1;
        if (a.hist && a.hist_cap > 0)
            write_hist(a.hist + (size_t)(cin.checks % a.hist_cap) * HCOLS, it + 1, r, sg, cin.rho, t,
                       s123, conv, fac);
    }
}

// ------------------------------------------------- per-thread async prefetch
// PF sweep (one-tile rows, M <= 2): every thread copies the cells it will own in
// the NEXT item into its own slots of a double-buffered shared-memory slab with
// cp.async (LDGSTS, no registers held while in flight), so an item's HBM reads
// overlap the previous item's fp64 work.  Each thread reads back only what it
// copied itself: cp.async.wait_group orders it, no barrier is needed.
__device__ __forceinline__ unsigned pf_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(pf_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(pf_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// bytes of one item's slab per thread: x (M), y, v as double2; a2, a1, b2, b1 (M each) as CT[2]
template <int M, typename CT>
struct PFCfg {
    static constexpr int XB16 = M + 2;                  // 16-byte chunks
    static constexpr int CB = 2 * (int)sizeof(CT);      // bytes of one coefficient pair
    static constexpr int PER_THREAD = 16 * XB16 + 4 * M * CB;
};

template <typename CT>
__device__ __forceinline__ void cp_async_pair(void* dst, const CT* src) {
    if constexpr (sizeof(CT) == 8) cp_async16(dst, src);
    else cp_async8(dst, src);
}
template <typename CT>
__device__ __forceinline__ void lds2(const unsigned char* p, double* o) {
    if constexpr (sizeof(CT) == 8) {
        const double2 t = *reinterpret_cast<const double2*>(p);
        o[0] = t.x;
        o[1] = t.y;
    } else {
        const float2 t = *reinterpret_cast<const float2*>(p);
        o[0] = (double)t.x;
        o[1] = (double)t.y;
    }
}

// issue this thread's copies of row jj (its cells kl, kl+1) into slab buffer buf
template <int M, typename CT>
__device__ __forceinline__ void pf_issue(const KArgs& a, unsigned char* buf, int bs, int tid,
                                         long long jj, int kl, long long qn) {
    using C = PFCfg<M, CT>;
    const long long ro = jj * a.n_pad + kl;
#pragma unroll
    for (int i = 0; i < M; ++i) cp_async16(buf + ((size_t)i * bs + tid) * 16, a.x + i * qn + ro);
    cp_async16(buf + ((size_t)M * bs + tid) * 16, a.y + ro);
    cp_async16(buf + ((size_t)(M + 1) * bs + tid) * 16, a.v + ro);
    unsigned char* cb = buf + (size_t)C::XB16 * bs * 16;
    const CT* src[4];
    if constexpr (sizeof(CT) == 4) {
        src[0] = a.fa2; src[1] = a.fa1; src[2] = a.fb2; src[3] = a.fb1;
    } else {
        src[0] = reinterpret_cast<const CT*>(a.a2); src[1] = reinterpret_cast<const CT*>(a.a1);
        src[2] = reinterpret_cast<const CT*>(a.b2); src[3] = reinterpret_cast<const CT*>(a.b1);
    }
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c)
            cp_async_pair<CT>(cb + ((size_t)(4 * i + c) * bs + tid) * C::CB, src[c] + i * qn + ro);
    cp_async_commit();
}

// ---------------------------------------------------------------- the sweep
// Row finalisation for (i, j) (PAPER.md:432-448 via identity I1):
//   W = sum_k (g(x_k) - lam) = Sg + sum_k b0 - n lam,  t = h + p - W,
//   lam' = kappa t, zeta' = lam' - lam (z' = g(x') + zeta'), 1'z' = W + n lam',
//   h' = min(c, 1'z' - p), p' = p + h' - 1'z'.
// Returns the check terms (r2, r3, s1raw, s2raw).
__device__ __forceinline__ void finalize_row(const KArgs& a, const Ctrl& cin, int i, long long j,
                                             double Sg, double dgmax, double dgmin, double* r2,
                                             double* r3, double* s1, double* s2) {
    const long long rix = (long long)i * a.q + j;
    const RowOut o = row_update(Sg, a.sb0[rix], __ldcg(a.lam + rix) * cin.f[0],
                                __ldcg(a.p + rix) * cin.f[1], __ldcg(a.h + rix),
                                __ldcg(a.zeta + rix), a.c[i], a.nd, cin.rho, dgmax, dgmin);
    __stcg(a.lam + rix, o.lam);
    __stcg(a.zeta + rix, o.zeta);
    __stcg(a.h + rix, o.h);
    __stcg(a.p + rix, o.p);
    *r2 = o.r2;
    *r3 = o.r3;
    *s1 = o.s1;
    *s2 = o.s2;
}

// Same update from row scalars the sweep loaded with the item (no global round
// trip at the end of the item): lam_e = lam f0, p_e = p f1, h_o, zeta_o, sb0_e.
__device__ __forceinline__ void finalize_row_v(const KArgs& a, const Ctrl& cin, int i, long long j,
                                               double Sg, double dgmax, double dgmin, double lam_e,
                                               double p_e, double h_o, double zeta_o, double sb0_e,
                                               double* r2, double* r3, double* s1, double* s2) {
    const long long rix = (long long)i * a.q + j;
    const RowOut o = row_update(Sg, sb0_e, lam_e, p_e, h_o, zeta_o, a.c[i], a.nd, cin.rho, dgmax,
                                dgmin);
    __stcg(a.lam + rix, o.lam);
    __stcg(a.zeta + rix, o.zeta);
    __stcg(a.h + rix, o.h);
    __stcg(a.p + rix, o.p);
    *r2 = o.r2;
    *r3 = o.r3;
    *s1 = o.s1;
    *s2 = o.s2;
}
// element i of a small register array without local-memory indexing
template <int M>
__device__ __forceinline__ double pick(const double* v, int i) {
    double r = v[0];
#pragma unroll
    for (int l = 1; l < M; ++l) r = (i == l) ? v[l] : r;
    return r;
}

// FX = true (every problem with a finite box): row sums in exact fixed point,
// per-warp slots and a last-warp finaliser -- no block barrier inside the item
// loop, so one warp's loads overlap another warp's fp64 work.  FX = false
// (an infinite bound): fp64 block reductions with barriers.
// CT = float: F2 mixed precision -- a2, a1, b2, b1 read from their fp32 copies
// (16 instead of 32 bytes per element), every operation in fp64.
// PF = true (one-tile rows, M <= 2): cp.async prefetch of the next
// item into a double-buffered dynamic shared-memory slab (see pf_issue).
#ifndef SWEEP_LB
#define SWEEP_LB 512
#endif
// U = cells (consecutive steps k) per thread: 2 (one double2 per stream) or 4
// (two; four interleaved Gauss-Seidel chains per thread, 256-thread CTAs).
// RL = true (row loop, U = 2, block-barrier reductions): small CTAs (128 threads,
// four per SM) each own whole rows and walk the row's tiles in order, keeping the
// row partials in the finalising threads' registers -- no cross-CTA row reduction,
// and four independent CTAs per SM overlap each other's load, compute and barrier
// phases (tools/stream_probe.cu: this structure moves 89-92 % of the HBM peak with
// no arithmetic, one 512-thread CTA per SM 70-73 %).
template <int M, int MODE, bool FX, typename CT, bool PF, int U, int RLT>
#ifndef SWEEP_RL_MINB
#define SWEEP_RL_MINB 4
#endif
__global__ void __launch_bounds__(RLT ? RLT : (U == 2 ? SWEEP_LB : 256), RLT ? (RLT == 128 ? SWEEP_RL_MINB : 512 / (RLT ? RLT : 1)) : (U == 2 ? 1 : 2))
    sweep_kernel(KArgs a) {
    constexpr bool RL = RLT != 0;  // row loop with RLT-thread CTAs
    static_assert(!RL || (U == 2 && !FX && !PF), "row loop: two-cell barrier variant only");
    static_assert(!PF || U == 2, "the prefetching sweep moves one double2 per stream");
    static_assert(U == 2 || U == 4, "2 or 4 cells per thread");
    // row scalars for the finalisation loaded with the item (U = 4 and PF: measured faster)
    constexpr bool PRELOAD = PF || U == 4;
    const long long it = *(volatile long long*)a.iter;
    const Ctrl& cin = a.ctrl[it & 1];
    if (cin.done || it >= a.prm->iter_limit) return;
    const int ce = a.prm->check_every;
    const bool is_check = ce > 0 && ((it + 1) % ce) == 0;

    // red is double-buffered by the CTA's row parity in the row loop: with no trailing
    // barrier a warp may reach the next row's reduction while warp 0 still reads this one
    __shared__ double red2[2][16][(3 * M + 2) > 6 ? (3 * M + 2) : 6];
    int rpar = 0;  // row loop: parity of the rows this CTA has reduced
    __shared__ double rowres[3 * M];
    __shared__ double k0x[M], k0nu[M];
    __shared__ double acc[XB];
    __shared__ int s_last;
    constexpr int UB = 4;                            // item slots in flight (FX)
    __shared__ unsigned long long s_fxw[UB][16][M];  // per-warp fixed-point row partials
    __shared__ double s_dgw[UB][16][2 * M];          // per-warp dg extrema (checks)
    __shared__ unsigned s_arr[UB], s_gen[UB];        // arrivals, finalisations per slot

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    if (FX && tid < UB) {
        s_arr[tid] = 0u;
        s_gen[tid] = 0u;
    }
    if (tid < XB) {
        double init = 0.0;
        if (tid >= MAXM && tid < MAXM + M) init = -INFINITY;      // x0max
        if (tid >= 2 * MAXM && tid < 2 * MAXM + M) init = INFINITY; // x0min
        acc[tid] = init;
    }

    double rho[4], f[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        rho[l] = cin.rho[l];
        f[l] = cin.f[l];
    }
    const double iq = a.inv_q;
    const long long nitems = a.q * a.T;
    const long long qn = a.q * (long long)a.n_pad;

    double my_r1 = 0.0, my_s3 = 0.0;  // per-thread check maxima over all its cells
    // row-level check maxima, held by thread i < M for source i
    double my_r2 = 0.0, my_r3 = 0.0, my_s1 = 0.0, my_s2 = 0.0;

    // slot counters (FX) and the consensus accumulators acc[] initialised before any use
    // (the row loop adds to acc from thread 0 before its first block barrier)
    if (FX || RL) __syncthreads();
    long long litem = 0;
    // (row, tile) of the item, advanced incrementally (no 64-bit division per item)
    long long j = RL ? (long long)blockIdx.x : (long long)blockIdx.x / a.T;
    int tile = RL ? 0 : (int)((long long)blockIdx.x - j * a.T);
    // RL with multi-tile rows: per-thread row partials carried across the row's tiles,
    // one block reduction per row (at its last tile)
    double rt_S[M], rt_x[M], rt_n[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        rt_S[i] = 0.0;
        rt_x[i] = -INFINITY;
        rt_n[i] = INFINITY;
    }
    const int gT = a.G / a.T, gR = a.G - gT * a.T;  // G = gT * T + gR
    double x1c[M];
#pragma unroll
    for (int i = 0; i < M; ++i) x1c[i] = cin.x1[i];
    const bool nu_pending = cin.nu_pending != 0;
    extern __shared__ __align__(16) unsigned char pf_sm[];
    const size_t pf_buf = (size_t)blockDim.x * PFCfg<M, CT>::PER_THREAD;
    const int pf_kl = (U * tid < a.n_pad) ? U * tid : 0;  // T == 1: tile 0 only
    double lam_nx[M], zeta_nx[M], nu_nx[M], p_nx[M], h_nx[M], sb0_nx[M];  // next row's scalars (PF)
    if constexpr (PF) {
        if (blockIdx.x < nitems) {
            pf_issue<M, CT>(a, pf_sm, blockDim.x, tid, blockIdx.x, pf_kl, qn);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const long long rix = (long long)i * a.q + blockIdx.x;
                lam_nx[i] = __ldcg(a.lam + rix);
                zeta_nx[i] = __ldcg(a.zeta + rix);
                p_nx[i] = __ldcg(a.p + rix);
                h_nx[i] = __ldcg(a.h + rix);
                sb0_nx[i] = __ldg(a.sb0 + rix);
                nu_nx[i] = tid == 0 ? __ldcg(a.nu + rix) : 0.0;
            }
        }
    }
    for (long long item = blockIdx.x; RL ? (j < a.q) : (item < nitems); item += a.G, ++litem,
                   j += RL ? ((++tile == a.T) ? a.G : 0) : gT + ((tile += gR) >= a.T ? 1 : 0),
                   tile -= (tile >= a.T ? a.T : 0)) {
        const int k = tile * a.tile + U * tid;  // first of this thread's U cells
        const bool inb = k < a.n_pad;           // n_pad % 4 == 0: all U cells in bounds
        bool vc[U];
#pragma unroll
        for (int c = 0; c < U; ++c) vc[c] = (k + c) < a.n;
        const int kl = inb ? k : 0;  // out-of-range threads load cell 0 (results discarded)

        double xo[M][U], xn[M][U];
        double Sg[M], dgx[M], dgn[M];
        double yv[U], vv[U];
        double ca2[M][U], ca1[M][U], cb2[M][U], cb1[M][U], clo[M][U], chi[M][U];
        double lam_e[M], zeta_o[M], nu_e[M], nu_ld[M], p_e[M], h_e[M], sb0_e[M];
        if constexpr (PF) {
            // next item's copies go out first, then this item's (issued one item ago) land
            const long long jn = j + a.G;
            unsigned char* cur = pf_sm + (size_t)(litem & 1) * pf_buf;
            if (jn < a.q) pf_issue<M, CT>(a, pf_sm + (size_t)((litem + 1) & 1) * pf_buf, blockDim.x, tid, jn,
                                          pf_kl, qn);
            else cp_async_commit();  // empty group: wait_group 1 below still means "this item"
#pragma unroll
            for (int i = 0; i < M; ++i) {
                lam_e[i] = lam_nx[i] * f[0];
                zeta_o[i] = zeta_nx[i];
                p_e[i] = p_nx[i] * f[1];
                h_e[i] = h_nx[i];
                sb0_e[i] = sb0_nx[i];
                nu_ld[i] = nu_nx[i];
            }
            if (jn < a.q) {
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const long long rix = (long long)i * a.q + jn;
                    lam_nx[i] = __ldcg(a.lam + rix);
                    zeta_nx[i] = __ldcg(a.zeta + rix);
                    p_nx[i] = __ldcg(a.p + rix);
                    h_nx[i] = __ldcg(a.h + rix);
                    sb0_nx[i] = __ldg(a.sb0 + rix);
                    nu_nx[i] = tid == 0 ? __ldcg(a.nu + rix) : 0.0;
                }
            }
            cp_async_wait1();
            const int bsz = blockDim.x;
            lds2<double>(cur + ((size_t)M * bsz + tid) * 16, yv);
            lds2<double>(cur + ((size_t)(M + 1) * bsz + tid) * 16, vv);
            const unsigned char* cb = cur + (size_t)PFCfg<M, CT>::XB16 * bsz * 16;
            constexpr int CB = PFCfg<M, CT>::CB;
#pragma unroll
            for (int i = 0; i < M; ++i) {
                lds2<double>(cur + ((size_t)i * bsz + tid) * 16, xo[i]);
                lds2<CT>(cb + ((size_t)(4 * i + 0) * bsz + tid) * CB, ca2[i]);
                lds2<CT>(cb + ((size_t)(4 * i + 1) * bsz + tid) * CB, ca1[i]);
                lds2<CT>(cb + ((size_t)(4 * i + 2) * bsz + tid) * CB, cb2[i]);
                lds2<CT>(cb + ((size_t)(4 * i + 3) * bsz + tid) * CB, cb1[i]);
                const long long bk = (long long)i * a.n_pad + kl;
                double2 t;
                t = __ldg(reinterpret_cast<const double2*>(a.lo + bk)); clo[i][0] = t.x; clo[i][1] = t.y;
                t = __ldg(reinterpret_cast<const double2*>(a.hi + bk)); chi[i][0] = t.x; chi[i][1] = t.y;
            }
        } else if constexpr (U == 4) {
            // staged: x, y, v into this thread's slab slots; coefficients read at use
            // (an L2 prefetch of them here measured slower, profiles/r01d)
            double* slab = reinterpret_cast<double*>(pf_sm);
            const int bsz = blockDim.x;
            double t[4];
            ldU<double, 4>(a.y + j * a.n_pad + kl, t);
            wr4(slab + ((size_t)Slab4<M>::Y * bsz + tid) * 4, t);
            ldvU<4>(a.v + j * a.n_pad + kl, t);
            wr4(slab + ((size_t)Slab4<M>::V * bsz + tid) * 4, t);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                ldvU<4>(a.x + (long long)i * qn + j * a.n_pad + kl, t);
                wr4(slab + ((size_t)(Slab4<M>::XO + i) * bsz + tid) * 4, t);
                xo[i][0] = t[0];  // consensus cell (lazy (6h) below)
            }
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const long long rix = (long long)i * a.q + j;
                lam_e[i] = __ldcg(a.lam + rix) * f[0];
                zeta_o[i] = __ldcg(a.zeta + rix);
                p_e[i] = __ldcg(a.p + rix) * f[1];
                h_e[i] = __ldcg(a.h + rix);
                sb0_e[i] = __ldg(a.sb0 + rix);
                nu_ld[i] = 0.0;
            }
        } else {
        ldU<double, U>(a.y + j * a.n_pad + kl, yv);
        ldvU<U>(a.v + j * a.n_pad + kl, vv);
        // coefficient streams, all issued up front
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const long long e = (long long)i * qn + j * a.n_pad + kl;
            ldvU<U>(a.x + e, xo[i]);
            if constexpr (sizeof(CT) == 4) {
                ldU<float, U>(a.fa2 + e, ca2[i]);
                ldU<float, U>(a.fa1 + e, ca1[i]);
                ldU<float, U>(a.fb2 + e, cb2[i]);
                ldU<float, U>(a.fb1 + e, cb1[i]);
            } else {
                ldU<double, U>(a.a2 + e, ca2[i]);
                ldU<double, U>(a.a1 + e, ca1[i]);
                ldU<double, U>(a.b2 + e, cb2[i]);
                ldU<double, U>(a.b1 + e, cb1[i]);
            }
            const long long bk = (long long)i * a.n_pad + kl;
            ldU<double, U>(a.lo + bk, clo[i]);
            ldU<double, U>(a.hi + bk, chi[i]);
        }
        // per-row scalars (uniform loads)
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const long long rix = (long long)i * a.q + j;
            lam_e[i] = __ldcg(a.lam + rix) * f[0];
            zeta_o[i] = __ldcg(a.zeta + rix);
            p_e[i] = 0.0;  // U == 2 without prefetch: the finaliser reads p, h, sb0 itself
            h_e[i] = 0.0;  // (fewer live registers measured faster, profiles/r01d)
            sb0_e[i] = 0.0;
            nu_ld[i] = 0.0;
        }
        }  // !PF loads
#pragma unroll
        for (int i = 0; i < M; ++i) nu_e[i] = 0.0;
        const bool owns_k0 = (k == 0);
        if (owns_k0) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const long long rix = (long long)i * a.q + j;
                double nu = PF ? nu_ld[i] : __ldcg(a.nu + rix);
                // lazy (6h) of the previous iteration, then its dual rescale
                if (nu_pending) nu = nu + x1c[i] - xo[i][0];
                nu_e[i] = nu * f[3];
                __stcg(a.nu + rix, nu_e[i]);
            }
        }

        // ---- (6a) Gauss-Seidel over sources, then (6e)/(6f), per cell
        double zl[M], x1nu[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            zl[i] = zeta_o[i] + lam_e[i];
            x1nu[i] = x1c[i] + nu_e[i];
        }
        double vn[U];
        {
            if constexpr (U == 4) {
                double* slab = reinterpret_cast<double*>(pf_sm);
                const int bsz = blockDim.x;
                staged_gs4<M, MODE, CT>(a, slab, bsz, tid, j * a.n_pad + kl, qn, kl, zl, rho, iq, owns_k0,
                                        x1nu, f[2]);
                // tail operands back into registers (live only from here on)
                rd4(slab + ((size_t)Slab4<M>::Y * bsz + tid) * 4, yv);
                rd4(slab + ((size_t)Slab4<M>::V * bsz + tid) * 4, vv);
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    rd4(slab + ((size_t)(Slab4<M>::XO + i) * bsz + tid) * 4, xo[i]);
                    rd4(slab + ((size_t)(Slab4<M>::XN + i) * bsz + tid) * 4, xn[i]);
                    const long long e = (long long)i * qn + j * a.n_pad + kl;
                    if constexpr (sizeof(CT) == 4) {
                        ldU<float, 4>(a.fb2 + e, cb2[i]);
                        ldU<float, 4>(a.fb1 + e, cb1[i]);
                    } else {
                        ldU<double, 4>(a.b2 + e, cb2[i]);
                        ldU<double, 4>(a.b1 + e, cb1[i]);
                    }
                }
            } else {
                double s_e[U], mu_e[U];
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    s_e[c] = fmax(vv[c], 0.0);
                    mu_e[c] = vv[c] < 0.0 ? -vv[c] * f[2] : 0.0;
                }
                gs_cellU<M, MODE, U>(ca2, ca1, cb2, cb1, clo, chi, xo, xn, yv, s_e, mu_e, zl, rho, iq,
                                     owns_k0, x1nu);
            }
#pragma unroll
            for (int c = 0; c < U; ++c) {
                double txo[M], txn[M];
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    txo[i] = xo[i][c];
                    txn[i] = xn[i][c];
                }
                const bool valid = vc[c];
                double r1l = my_r1, s3l = my_s3;
                const double vnew = cell_tail<M>(txo, txn, yv[c], vv[c], f[2], is_check && valid, r1l, s3l);
                my_r1 = r1l;
                my_s3 = s3l;
                vn[c] = valid ? vnew : 0.0;
            }
        }
#pragma unroll
        for (int i = 0; i < M; ++i) {
            Sg[i] = 0.0;
            dgx[i] = -INFINITY;
            dgn[i] = INFINITY;
#pragma unroll
            for (int c = 0; c < U; ++c) {
                const bool valid = vc[c];
                if (!valid) xn[i][c] = 0.0;  // padding stays 0
                if (valid) {
                    const double b2 = cb2[i][c], b1 = cb1[i][c];
                    Sg[i] += fma(b2, xn[i][c], b1) * xn[i][c];
                    if (is_check) {  // sigma's z-term only
                        const double dg = (xn[i][c] - xo[i][c]) * fma(b2, xn[i][c] + xo[i][c], b1);
                        dgx[i] = fmax(dgx[i], dg);
                        dgn[i] = fmin(dgn[i], dg);
                    }
                }
            }
        }
        if (inb) {
            stU<U>(a.v + j * a.n_pad + k, vn);
#pragma unroll
            for (int i = 0; i < M; ++i) stU<U>(a.x + (long long)i * qn + j * a.n_pad + k, xn[i]);
        }
        if (owns_k0) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                k0x[i] = xn[i][0];
                k0nu[i] = nu_e[i];
            }
        }

        if constexpr (FX) {
            // ---- (6c) consensus contribution of k = 0 (thread 0 of warp 0: item order)
            if (owns_k0 && tile == 0) {
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    acc[i] += xn[i][0] - nu_e[i];
                    acc[MAXM + i] = fmax(acc[MAXM + i], xn[i][0]);
                    acc[2 * MAXM + i] = fmin(acc[2 * MAXM + i], xn[i][0]);
                }
            }
            // ---- row partials: exact fixed point into this warp's slot of item litem
            const int b = (int)(litem & (UB - 1));
            if (lane == 0)  // slot b free: the finaliser of item litem - UB is done with it
                while (*(volatile unsigned*)&s_gen[b] != (unsigned)(litem >> 2)) {
                }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < M; ++i) {
                long long fx = 0;
#pragma unroll
                for (int c = 0; c < U; ++c)
                    if (vc[c])
                        fx += __double2ll_rn(fma(cb2[i][c], xn[i][c], cb1[i][c]) * xn[i][c] * a.fx_scale[i]);
                const unsigned long long ws = warp_sum_u64((unsigned long long)fx);
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
                last = (atomicAdd(&s_arr[b], 1u) == (unsigned)nw - 1);
                __threadfence_block();
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            __syncwarp();  // memory ordering: lane 0 acquired the slot writes, the warp reads them
            if (last) {
                // ---- this warp arrived last: row finalisation (6b),(6g),(6d),(6i)
                if (lane < M) {
                    const int i = lane;
                    unsigned long long part = 0ull;
                    double mx = -INFINITY, mn = INFINITY;
                    for (int w = 0; w < nw; ++w) {
                        part += s_fxw[b][w][i];
                        if (is_check) {
                            mx = fmax(mx, s_dgw[b][w][i]);
                            mn = fmin(mn, s_dgw[b][w][M + i]);
                        }
                    }
                    bool fin = true;
                    if (a.T > 1) {  // row split over tiles: global exact sums, last tile finalises
                        atomicAdd(a.rowacc + j * MAXM + i, part);
                        if (is_check) {
                            atomicMax(a.rowdg + j * 2 * MAXM + i, okey(mx));
                            atomicMin(a.rowdg + j * 2 * MAXM + MAXM + i, okey(mn));
                        }
                        __threadfence();
                        fin = (atomicAdd(a.rowcnt + j * MAXM + i, 1u) == (unsigned)a.T - 1);
                        if (fin) {
                            __threadfence();
                            part = atomicExch(a.rowacc + j * MAXM + i, 0ull);
                            if (is_check) {
                                mx = okey_inv(atomicExch(a.rowdg + j * 2 * MAXM + i, 0ull));
                                mn = okey_inv(atomicExch(a.rowdg + j * 2 * MAXM + MAXM + i, ~0ull));
                            }
                            a.rowcnt[j * MAXM + i] = 0u;
                        }
                    }
                    if (fin) {
                        double r2, r3, s1, s2;
                        if constexpr (PRELOAD)
                            finalize_row_v(a, cin, i, j, (double)(long long)part * a.fx_inv[i], mx, mn,
                                           pick<M>(lam_e, i), pick<M>(p_e, i), pick<M>(h_e, i),
                                           pick<M>(zeta_o, i), pick<M>(sb0_e, i), &r2, &r3, &s1, &s2);
                        else
                            finalize_row(a, cin, i, j, (double)(long long)part * a.fx_inv[i], mx, mn, &r2,
                                         &r3, &s1, &s2);
                        my_r2 = fmax(my_r2, r2);
                        my_r3 = fmax(my_r3, r3);
                        my_s1 = fmax(my_s1, s1);
                        my_s2 = fmax(my_s2, s2);
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    s_arr[b] = 0u;
                    __threadfence_block();
                    atomicAdd(&s_gen[b], 1u);  // release the slot to item litem + UB
                }
            }
            continue;
        }
        if constexpr (RL) {
            if (a.T > 1) {
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    rt_S[i] += Sg[i];
                    rt_x[i] = fmax(rt_x[i], dgx[i]);
                    rt_n[i] = fmin(rt_n[i], dgn[i]);
                }
                if (owns_k0) {  // (6c) contribution of k = 0 (thread 0, row order)
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        acc[i] += xn[i][0] - nu_e[i];
                        acc[MAXM + i] = fmax(acc[MAXM + i], xn[i][0]);
                        acc[2 * MAXM + i] = fmin(acc[2 * MAXM + i], xn[i][0]);
                    }
                }
                if (tile < a.T - 1) continue;  // row not finished: no reduction yet
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    Sg[i] = rt_S[i];
                    dgx[i] = rt_x[i];
                    dgn[i] = rt_n[i];
                    rt_S[i] = 0.0;
                    rt_x[i] = -INFINITY;
                    rt_n[i] = INFINITY;
                }
            }
        }
        // ---- deterministic block reduction of Sg (sum), dg (max/min) per source
#pragma unroll
        for (int i = 0; i < M; ++i) {
            Sg[i] = warp_sum(Sg[i]);
            if (is_check) {
                dgx[i] = warp_max(dgx[i]);
                dgn[i] = warp_min(dgn[i]);
            }
        }
        auto red = red2[rpar];
        if (RL) rpar ^= 1;
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                red[wid][3 * i] = Sg[i];
                red[wid][3 * i + 1] = dgx[i];
                red[wid][3 * i + 2] = dgn[i];
            }
        }
        __syncwarp();
        __syncthreads();
        if (wid == 0) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                double s = lane < nw ? red[lane][3 * i] : 0.0;
                double mx = lane < nw ? red[lane][3 * i + 1] : -INFINITY;
                double mn = lane < nw ? red[lane][3 * i + 2] : INFINITY;
                s = warp_sum(s);
                if (is_check) {
                    mx = warp_max(mx);
                    mn = warp_min(mn);
                }
                if (lane == 0) {
                    rowres[3 * i] = s;
                    rowres[3 * i + 1] = mx;
                    rowres[3 * i + 2] = mn;
                }
            }
        }
        __syncwarp();
        // RL: rowres is produced and consumed by warp 0 only (the finalising threads
        // are tid < M), so the other warps go on to the next row without a second barrier
        if (!(RL && a.T > 1)) __syncthreads();

        // ---- row finalisation (6b),(6g),(6d),(6i)
        if (RL && a.T > 1) {  // this CTA owns every tile of the row (last tile here)
            if (tid < M) {
                double r2, r3, s1, s2;
                finalize_row(a, cin, tid, j, rowres[3 * tid], rowres[3 * tid + 1], rowres[3 * tid + 2],
                             &r2, &r3, &s1, &s2);
                my_r2 = fmax(my_r2, r2);
                my_r3 = fmax(my_r3, r3);
                my_s1 = fmax(my_s1, s1);
                my_s2 = fmax(my_s2, s2);
            }
        } else if (a.T == 1) {
            if (tid < M) {
                double r2, r3, s1, s2;
                if constexpr (PRELOAD)
                    finalize_row_v(a, cin, tid, j, rowres[3 * tid], rowres[3 * tid + 1], rowres[3 * tid + 2],
                                   pick<M>(lam_e, tid), pick<M>(p_e, tid), pick<M>(h_e, tid),
                                   pick<M>(zeta_o, tid), pick<M>(sb0_e, tid), &r2, &r3, &s1, &s2);
                else
                    finalize_row(a, cin, tid, j, rowres[3 * tid], rowres[3 * tid + 1],
                                 rowres[3 * tid + 2], &r2, &r3, &s1, &s2);
                my_r2 = fmax(my_r2, r2);
                my_r3 = fmax(my_r3, r3);
                my_s1 = fmax(my_s1, s1);
                my_s2 = fmax(my_s2, s2);
            }
        } else {
            if (tid < M) {
                double* rp = a.row_part + (((long long)tid * a.q + j) * a.T + tile) * 3;
                __stcg(rp, rowres[3 * tid]);
                __stcg(rp + 1, rowres[3 * tid + 1]);
                __stcg(rp + 2, rowres[3 * tid + 2]);
            }
            __threadfence();
            __syncwarp();
        __syncthreads();
            if (tid == 0) s_last = (atomicAdd(a.row_cnt + j, 1) == a.T - 1);
            __syncwarp();
        __syncthreads();
            if (s_last) {
                __threadfence();
                // tile partials of row j: lane-strided loads (all in flight), fixed-order
                // per-lane sums and a butterfly (deterministic); lane i keeps source i
                double Sgs = 0.0, mx = -INFINITY, mn = INFINITY;
                if (wid == 0) {
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        const double* rp = a.row_part + ((long long)i * a.q + j) * a.T * 3;
                        double ls = 0.0, lx = -INFINITY, ln = INFINITY;
                        for (int t = lane; t < a.T; t += 32) {
                            ls += __ldcg(rp + 3 * t);
                            lx = fmax(lx, __ldcg(rp + 3 * t + 1));
                            ln = fmin(ln, __ldcg(rp + 3 * t + 2));
                        }
                        ls = warp_sum(ls);
                        lx = warp_max(lx);
                        ln = warp_min(ln);
                        if (lane == i) {
                            Sgs = ls;
                            mx = lx;
                            mn = ln;
                        }
                    }
                }
                if (tid < M) {
                    double r2, r3, s1, s2;
                    if constexpr (PRELOAD)
                        finalize_row_v(a, cin, tid, j, Sgs, mx, mn, pick<M>(lam_e, tid), pick<M>(p_e, tid),
                                       pick<M>(h_e, tid), pick<M>(zeta_o, tid), pick<M>(sb0_e, tid), &r2,
                                       &r3, &s1, &s2);
                    else
                        finalize_row(a, cin, tid, j, Sgs, mx, mn, &r2, &r3, &s1, &s2);
                    my_r2 = fmax(my_r2, r2);
                    my_r3 = fmax(my_r3, r3);
                    my_s1 = fmax(my_s1, s1);
                    my_s2 = fmax(my_s2, s2);
                }
                if (tid == 0) a.row_cnt[j] = 0;
            }
        }
        // ---- (6c) consensus contributions of k = 0, in this CTA's item order
        if (tile == 0 && tid < M && !(RL && a.T > 1)) {
            acc[tid] += k0x[tid] - k0nu[tid];
            acc[MAXM + tid] = fmax(acc[MAXM + tid], k0x[tid]);
            acc[2 * MAXM + tid] = fmin(acc[2 * MAXM + tid], k0x[tid]);
        }
        __syncwarp();
        // red/rowres/k0x reused by the next item.  RL: red alternates between two
        // buffers by row parity (warp 0 reads red[p] of row r before it arrives at row
        // r+1's barrier, so no warp can write red[p] again for row r+2 before that read),
        // rowres stays within warp 0, and k0x is not used (thread 0 adds the consensus
        // term itself), so no barrier is needed
        if (!(RL && a.T > 1)) __syncthreads();
    }

    // ---- per-CTA partials: block max of r1, s3 and of the row terms (held by the
    // finalising lanes: threads < M, or lanes < M of any warp in the FX variant)
    __syncthreads();
    if (is_check) {
        my_r1 = warp_max(my_r1);
        my_s3 = warp_max(my_s3);
        my_r2 = warp_max(my_r2);
        my_r3 = warp_max(my_r3);
        my_s1 = warp_max(my_s1);
        my_s2 = warp_max(my_s2);
        auto red = red2[0];
        if (lane == 0) {
            red[wid][0] = my_r1;
            red[wid][1] = my_s3;
            red[wid][2] = my_r2;
            red[wid][3] = my_r3;
            red[wid][4] = my_s1;
            red[wid][5] = my_s2;
        }
        __syncthreads();
        if (tid == 0) {
            double r1 = 0.0, s3 = 0.0, r2 = 0.0, r3 = 0.0, s1 = 0.0, s2 = 0.0;
            for (int w = 0; w < nw; ++w) {
                r1 = fmax(r1, red[w][0]);
                s3 = fmax(s3, red[w][1]);
                r2 = fmax(r2, red[w][2]);
                r3 = fmax(r3, red[w][3]);
                s1 = fmax(s1, red[w][4]);
                s2 = fmax(s2, red[w][5]);
            }
            acc[3 * MAXM + 0] = r1;
            acc[3 * MAXM + 1] = r2;
            acc[3 * MAXM + 2] = r3;
            acc[3 * MAXM + 3] = s1;
            acc[3 * MAXM + 4] = s2;
            acc[3 * MAXM + 5] = s3;
        }
        __syncthreads();
    }
    if (tid < XB) __stcg(a.cta_part + (size_t)blockIdx.x * XB + tid, acc[tid]);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(a.glob_cnt, 1) == a.G - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    // ---- last CTA: reduce the G CTA partials; lane = slot, warp w takes
    // CTAs g = w, w + nw, ... (fixed assignment => deterministic), then
    // thread s < XB combines the warps in order.
    {
        const int s = lane;  // XB == 32 slots
        const bool is_sum = s < MAXM;
        const bool is_min = s >= 2 * MAXM && s < 3 * MAXM;
        const double ident = is_sum ? 0.0 : (is_min ? INFINITY : (s >= 3 * MAXM ? 0.0 : -INFINITY));
        // eight independent accumulators per lane (loads in flight together: with
        // 592 small CTAs a serial chain cost ~50 us per launch), combined in a fixed order
        double vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) vv[u] = ident;
        for (int g0 = wid; g0 < a.G; g0 += 8 * nw) {
            double t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int g = g0 + u * nw;
                t[u] = g < a.G ? __ldcg(a.cta_part + (size_t)g * XB + s) : ident;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) vv[u] = is_sum ? vv[u] + t[u] : (is_min ? fmin(vv[u], t[u]) : fmax(vv[u], t[u]));
        }
        double v = vv[0];
#pragma unroll
        for (int u = 1; u < 8; ++u) v = is_sum ? v + vv[u] : (is_min ? fmin(v, vv[u]) : fmax(v, vv[u]));
        __shared__ double wred[16][XB];
        wred[wid][s] = v;
        __syncthreads();
        if (tid < XB) {
            double r = ident;
            for (int w = 0; w < nw; ++w) {
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
            finalize_global(a, acc, 1, it, cin, cout, is_check);
            __threadfence();
            *(volatile long long*)a.iter = it + 1;
        }
    }
}

#ifndef ADMM_KERNELS_NO_GLOBALS  // translation units other than admm.cu (sweep2.cu)
// multi-GPU: after ncclAllGather(xsend -> xall) on the stream
__global__ void finalize_kernel(KArgs a) {
    const long long it = *(volatile long long*)a.iter;
    const Ctrl& cin = a.ctrl[it & 1];
    if (cin.done || it >= a.prm->iter_limit) return;
    if (threadIdx.x != 0) return;
    const int ce = a.prm->check_every;
    const bool is_check = ce > 0 && ((it + 1) % ce) == 0;
    finalize_global(a, a.xall, a.world, it, cin, a.ctrl[(it + 1) & 1], is_check);
    __threadfence();
    *(volatile long long*)a.iter = it + 1;
}
#endif

}  // namespace admm_dev
