// admm_onchip2.cuh -- cluster-row on-chip engine, message-passing protocol
// (the default on-chip engine for PHEV-sized problems, BASELINE.json configs[0],
// [1]; Appendix A, Eq. (6a)-(6i), residuals :464-479, adaptive rho
// :318-324).  Same arithmetic as persist_cluster_kernel (admm_onchip.cuh); what
// changes is where the work sits and how the three couplings of an iteration travel:
//
//  * rows over more SMs: scenario row j = one cluster of T CTAs of NW warps, T and
//    NW chosen by the host plan so that the q*T CTAs cover every SM with about one
//    cell per thread (PHEV q = 50: 5 CTAs of 7 warps per row, two CTAs per SM,
//    instead of 2 CTAs of 16 warps on 100 SMs);
//  * row sums (6b)/(6g) without a cluster barrier: every warp sends its exact
//    fixed-point partial sums (and, on check iterations, the order-preserving keys
//    of its dg extrema and cell residual maxima) to every CTA of its row with
//    st.async into a per-(tile, warp) slot of the mate's shared memory, completing
//    bytes on the mate's mbarrier of the iteration's parity (the payload is the
//    signal: no fence).  Warp 0 of each CTA (the "row warp") waits on its own
//    mbarrier, sums the slots (integer addition: exact and order-independent),
//    performs the row update in lanes i < M, and one __syncthreads hands zeta + lam
//    to the cells.  Reuse of a parity two iterations later is safe: no CTA can send
//    iteration t+2's partials before every CTA of the row has consumed iteration t's;
//  * consensus (6c)/(6h) through L2 with "LL" words: a double is stored as two
//    64-bit words, each {32 data bits, 32-bit epoch}; a reader polls until both
//    epochs match.  No sentinel resets and no fences (the flag travels inside the
//    8-byte single-copy-atomic store).  Four rotating buffers make reuse safe:
//    before a CTA writes the publication of iteration t+4 it has observed one
//    publication of iteration t+2 or t+3 from every row, and each of those implies
//    that every CTA of that row has passed its barrier of iteration t+1, i.e.
//    finished every read of iteration t;
//  * residual checks without a grid barrier or fence: each row publishes its six
//    maxima (tile 0's row warp) and its x_1 (the consensus warp) as LL words, then
//    bumps a relaxed arrival counter; tile 0's row warp of every row polls the
//    counter (one lane), reads all rows' words (retrying the rare word whose epoch
//    is not yet visible), reduces them in a fixed order, takes the termination /
//    rho decision (same inputs, same order => same bits in every row) and forwards
//    it to the row's other CTAs with st.async on a per-check-parity mbarrier;
//  * the consensus warp sends its k = 0 partial right after the cell on non-check
//    iterations (the row update waits on it), before the cell's bookkeeping.

#pragma once
#include <cooperative_groups.h>

#include "admm_kernels.cuh"

namespace admm_dev {

constexpr int OC2_MAX_W = 16;  // warps per CTA (tile 0: NW-1 bulk warps + the consensus warp)
constexpr int OC2_REGS = 128;  // registers per thread (4 warps of 128 fill one SM sub-partition's 16K)
constexpr int OC2_MAX_T = 16;  // CTAs per cluster
constexpr int OC2_BUFS = 4;    // rotating LL buffers: (6c) contributions, check words
constexpr int OC2_CHKV = 6;    // per-row check values: r1 r2 r3 s1 s2 s3

struct C2Args {
    int TC0, TC, T, G;                    // cells of tile 0 / of the other tiles, tiles per row, CTAs
    double fx_scale[MAXM], fx_inv[MAXM];  // fixed-point scale 2^E_i of the row sums
    const double *bq, *ib2s;              // prepared per-element constants (admm_onchip.cuh)
    unsigned long long* pub;              // [4][M][q] LL pairs: x_1 - nu   (epoch = iteration in call + 1)
    unsigned long long* chkv;             // [4][q][6] LL pairs: row check maxima (epoch = check in call + 1)
    unsigned long long* chkx;             // [4][M][q] LL pairs: x_1 at checks
    unsigned long long* cnt;              // check arrivals in this call (2 q per check), relaxed
    double thr_hi, thr_lo;                // hi_ratio r_bar / sigma_bar, lo_ratio r_bar / sigma_bar
    DParams prm;                          // the call's parameters (kernel-parameter space, not L1)
};

// ------------------------------------------------------------------ LL words
__device__ __forceinline__ void ll_store(unsigned long long* p, double v, unsigned ep) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned long long e = (unsigned long long)ep << 32;
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"((b & 0xffffffffull) | e),
                 "l"((b >> 32) | e)
                 : "memory");
}
// true iff both halves carry epoch ep; *v = the double
__device__ __forceinline__ bool ll_load(const unsigned long long* p, unsigned ep, double* v) {
    unsigned long long w0, w1;
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    *v = __longlong_as_double((long long)((w0 & 0xffffffffull) | (w1 << 32)));
    return (unsigned)(w0 >> 32) == ep && (unsigned)(w1 >> 32) == ep;
}

// (6c) x1^{(i)} = (1/q) sum_j c^{(i,j)} over one LL buffer [M][q] (reading G1: the mean).
// Warp-collective; lane-strided partial sums in j order + a fixed butterfly: every
// warp that reads the same buffer gets the same bits.
template <int M>
__device__ __forceinline__ void ll_consensus(const unsigned long long* buf, long long q, unsigned ep,
                                             double qtot, double* x1) {
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
                    v[u][i] = 0.0;
                    if (jj < q) ok = ll_load(buf + 2 * ((long long)i * q + jj), ep, &v[u][i]) && ok;
                }
            }
        } while (!__all_sync(0xffffffffu, ok));
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < M; ++i) s[i] += v[u][i];
    }
    // M independent butterflies, interleaved
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < M; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
#pragma unroll
    for (int i = 0; i < M; ++i) x1[i] = s[i] * (1.0 / qtot);
}

// ------------------------------------------------------- cluster messaging
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned mapa_u32(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// 16 bytes into a mate's shared memory, completing 16 bytes of its mbarrier's transaction
__device__ __forceinline__ void st_async2(unsigned raddr, unsigned long long a, unsigned long long b,
                                          unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(
                     raddr),
                 "l"(a), "l"(b), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void gred_add_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64c(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// bits of a non-negative double order like the double (NaN above +inf)
__device__ __forceinline__ unsigned long long nbits(double v) {
    return (unsigned long long)__double_as_longlong(v);
}
__device__ __forceinline__ double nbits_inv(unsigned long long k) { return __longlong_as_double((long long)k); }
// warp maximum of a u64 key with two 32-bit redux (high word, then low word among the maxima)
__device__ __forceinline__ unsigned long long warp_max_key(unsigned long long k) {
    const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(k >> 32));
    const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(k >> 32) == hi ? (unsigned)k : 0u);
    return ((unsigned long long)hi << 32) | lo;
}

#ifdef ADMM_PHASE_PROF  // development build only: per-phase clock64() totals of 4 threads
__device__ unsigned long long g_phase2[4][10];
__device__ unsigned long long g_phase2all[1024][2][11];  // every CTA: [0] row warp lane 0, [1] consensus lane 0; [10] = smid
__device__ unsigned long long g_phase2c[2][6];  // check sub-phases, row warps of CTAs 0 and 1
#define PHASE2(k)                                 \
    if (prof_who >= 0) {                          \
        const unsigned long long _c = clock64();  \
        ph_acc[k] += _c - ph_last;                \
        ph_last = _c;                             \
    }
#define CPHASE(k)                                                       \
    if (lane == 0 && blockIdx.x < 2) {                                  \
        const unsigned long long _c = clock64();                        \
        atomicAdd(&g_phase2c[blockIdx.x][k], _c - c_last);              \
        c_last = _c;                                                    \
    }
#else
#define PHASE2(k)
#define CPHASE(k)
#endif

template <int M>
struct OC2 {
    static constexpr int MS = (M + 1) & ~1;  // u64 per row-sum slot (even: 16-byte stores)
    static constexpr int CW = 2 * M + 2;     // u64 keys per check slot: dg max [M], -dg max [M], r1, s3
    static constexpr int L = M <= 1 ? 1 : M <= 2 ? 2 : 4;  // lanes per slot group (power of two >= M)
};
// message area (dynamic shared memory after the cell arrays): row sums [2][NS][MS], check
// keys [2][NS][CW], NS = T * nw slots per parity
__host__ __device__ inline size_t oc2_msg_bytes(int M, int T, int nw) {
    return (size_t)2 * T * nw * (((M + 1) & ~1) + 2 * M + 2) * 8;
}

// Residual check of iteration it (row warp of every CTA).  Tile 0 of each row publishes the
// row's six maxima (LL words) and counts the arrival, waits until all 2q arrivals of check c
// are in (one lane polls the relaxed counter), reads every row's words and this iteration's
// (6c) contributions (LL: a word not yet visible is re-read), reduces them in a fixed order
// and takes the termination / rho decision (readings G10-G12;
// the arithmetic of check_decide); it then forwards the decision (16 doubles) to the other
// CTAs of its row with st.async on their decision mbarrier, so only q warps read L2, not q T.
// Every CTA rescales lam / p (reading G11) and hands rho, f, x1, r, sigma and the flags to
// its cells through shared memory.  x1 is summed in the order of ll_consensus (lane-strided
// j, then the butterfly): the bits the consensus warps compute.
constexpr int OC2_DEC = 16;  // decision record: rho_new[4] f[4] r sigma conv dir x1[M <= 4]

template <int M>
__device__ __noinline__ void oc2_check(const C2Args& p, double* hist, int hist_cap, double nd, int tile, int T,
                                       long long j, long long qq, double qtot, long long u, long long it,
                                       unsigned nchk, double r2, double r3, double s1, double s2,
                                       unsigned long long kr1, unsigned long long ks3, double* s_rho,
                                       double* s_f, double* s_R, double* s_t, int* s_flag, int* s_chk,
                                       double* s_kap, double* s_x1, double* r_lam, double* r_p,
                                       double* s_dec, unsigned dbar0) {
    const int lane = threadIdx.x & 31;
    const DParams& P = p.prm;
#ifdef ADMM_PHASE_PROF
    unsigned long long c_last = clock64();
#endif
    const unsigned cep = nchk + 1, pep = (unsigned)(u + 1);
    const unsigned db = nchk & 1u;                 // decision buffer / mbarrier of this check
    double dec[OC2_DEC];
    if (tile == 0) {
        unsigned long long* cbuf = p.chkv + 2 * (size_t)(nchk & (OC2_BUFS - 1)) * qq * OC2_CHKV;
        // row maxima over the sources (lanes i < M hold r2, r3, s1, s2 >= 0, or NaN)
        const unsigned long long k2 = warp_max_key(nbits(r2)), k3 = warp_max_key(nbits(r3));
        const unsigned long long k4 = warp_max_key(nbits(s1)), k5 = warp_max_key(nbits(s2));
        if (lane < OC2_CHKV) {
            const unsigned long long mine = lane == 0 ? kr1 : lane == 1 ? k2 : lane == 2 ? k3
                                          : lane == 3 ? k4 : lane == 4 ? k5 : ks3;
            ll_store(cbuf + 2 * ((size_t)j * OC2_CHKV + lane), nbits_inv(mine), cep);
        }
        __syncwarp();
        if (lane == 0) gred_add_relaxed(p.cnt, 1ull);
        CPHASE(0)
        const unsigned long long target = 2ull * (unsigned long long)qq * (nchk + 1ull);
        if (lane == 0)
            while (ld_relaxed_u64c(p.cnt) < target) __nanosleep(20);
        __syncwarp();
        CPHASE(1)
        // rows j = lane + 32 b: six maxima, x_1, (6c) contribution (LL words, re-read until current)
        const unsigned long long* xbuf = p.chkx + 2 * (size_t)(nchk & (OC2_BUFS - 1)) * M * qq;
        const unsigned long long* pbuf = p.pub + 2 * (size_t)(u & (OC2_BUFS - 1)) * M * qq;
        unsigned long long km[OC2_CHKV + 2 * M];  // maxima keys: r1..s3 bits, okey(x_1), okey(-x_1)
        double xs[M];
#pragma unroll
        for (int s = 0; s < OC2_CHKV + 2 * M; ++s) km[s] = 0ull;
#pragma unroll
        for (int i = 0; i < M; ++i) xs[i] = 0.0;
        for (long long jb = 0; jb < qq; jb += 32) {
            const long long jj = jb + lane;
            double v[OC2_CHKV], xv[M], pv[M];
            for (;;) {
                bool ok = true;
                if (jj < qq) {
#pragma unroll
                    for (int s = 0; s < OC2_CHKV; ++s)
                        ok = ll_load(cbuf + 2 * ((size_t)jj * OC2_CHKV + s), cep, &v[s]) && ok;
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        ok = ll_load(xbuf + 2 * ((size_t)i * qq + jj), cep, &xv[i]) && ok;
                        ok = ll_load(pbuf + 2 * ((size_t)i * qq + jj), pep, &pv[i]) && ok;
                    }
                }
                if (__all_sync(0xffffffffu, ok)) break;
            }
            if (jj < qq) {
#pragma unroll
                for (int s = 0; s < OC2_CHKV; ++s) km[s] = max(km[s], nbits(v[s]));
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    km[OC2_CHKV + i] = max(km[OC2_CHKV + i], okey(xv[i]));
                    km[OC2_CHKV + M + i] = max(km[OC2_CHKV + M + i], okey(-xv[i]));
                    xs[i] += pv[i];
                }
            } else {
#pragma unroll
                for (int i = 0; i < M; ++i) xs[i] += 0.0;
            }
        }
        CPHASE(2)
#pragma unroll
        for (int s = 0; s < OC2_CHKV + 2 * M; ++s) km[s] = warp_max_key(km[s]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int i = 0; i < M; ++i) xs[i] += __shfl_xor_sync(0xffffffffu, xs[i], o);
        double x1v[M];
#pragma unroll
        for (int i = 0; i < M; ++i) x1v[i] = xs[i] * (1.0 / qtot);
        // max_j |x_1^{(i,j)} - x1| = max(max_j x_1 - x1, x1 - min_j x_1) exactly
        double t3 = 0.0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const double xmx = okey_inv(km[OC2_CHKV + i]);
            const double xmn = -okey_inv(km[OC2_CHKV + M + i]);
            t3 = fmax(t3, fmax(xmx - x1v[i], x1v[i] - xmn));
        }
        const double tt[7] = {nbits_inv(km[0]), nbits_inv(km[1]), nbits_inv(km[2]), t3,
                              nbits_inv(km[3]), nbits_inv(km[4]), nbits_inv(km[5])};
        // check_decide (admm_kernels.cuh) with the thresholds prepared on the host
        const double rho[4] = {s_rho[0], s_rho[1], s_rho[2], s_rho[3]};
        const double sg1 = rho[0] * tt[4], sg2 = rho[1] * tt[5], sg3 = rho[2] * tt[6];
        const double r = fmax(fmax(tt[0], tt[1]), fmax(tt[2], tt[3]));
        const double sg = fmax(sg1, fmax(sg2, sg3));
        const int conv = (r < P.r_bar) && (sg < P.sigma_bar);
        int dir = 0;
        if (!conv && P.adapt) {
            const double ratio = (sg > 0.0) ? r / sg : INFINITY;  // reading G12
            if (ratio > p.thr_hi) dir = 1;
            else if (ratio < p.thr_lo) dir = -1;
        }
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            dec[l] = dir > 0 ? rho[l] * P.tau : dir < 0 ? rho[l] / P.tau : rho[l];
            dec[4 + l] = (dir != 0 && P.rescale) ? rho[l] / dec[l] : 1.0;
        }
        dec[8] = r;
        dec[9] = sg;
        dec[10] = conv;
        dec[11] = dir;
#pragma unroll
        for (int i = 0; i < OC2_DEC - 12; ++i) dec[12 + i] = i < M ? x1v[i < M ? i : 0] : 0.0;
        if (blockIdx.x == 0 && lane == 0 && hist && hist_cap > 0) {
            const double s123[3] = {sg1, sg2, sg3};
            const double fac = dir > 0 ? P.tau : dir < 0 ? 1.0 / P.tau : 1.0;
            write_hist(hist + (size_t)(*s_chk % hist_cap) * HCOLS, it + 1, r, sg, rho, tt, s123, conv, fac);
        }
        // forward the decision to the row's other CTAs (lane t -> CTA t)
        if (lane >= 1 && lane < T) {
            const unsigned rb = mapa_u32(dbar0 + 8 * db, (unsigned)lane);
            const unsigned rd = mapa_u32(smem_u32(s_dec + db * OC2_DEC), (unsigned)lane);
#pragma unroll
            for (int s = 0; s < OC2_DEC; s += 2) st_async2(rd + 8 * s, nbits(dec[s]), nbits(dec[s + 1]), rb);
        }
    } else {
        // the decision of this row's tile 0
        if (lane == 0) {
            mbar_expect(dbar0 + 8 * db, (unsigned)(OC2_DEC * 8));
            mbar_wait_cluster(dbar0 + 8 * db, (nchk >> 1) & 1u);
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < OC2_DEC; ++s) dec[s] = ((volatile double*)s_dec)[db * OC2_DEC + s];
    }
    CPHASE(3)
    const int conv = dec[10] != 0.0, dir = (int)dec[11];
    const double r = dec[8], sg = dec[9];
    __syncwarp();
    if (lane < M) {  // dual rescale (reading G11): lam<->rho1, p<->rho2 (factors 1 without a change)
        *r_lam *= dec[4];
        *r_p *= dec[5];
#pragma unroll
        for (int i = 0; i < M; ++i)
            if (lane == i) s_x1[i] = dec[12 + i];
    }
    if (lane == 0) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            s_rho[l] = dec[l];
            s_f[l] = dec[4 + l];
        }
        if (dir != 0) {
            s_R[0] = dec[0];
            s_R[1] = dec[2];
            s_R[2] = dec[3];
            s_R[3] = 1.0 / dec[0];
            *s_kap = dec[1] / (dec[0] + nd * dec[1]);
        }
        s_t[0] = r;
        s_t[1] = sg;
        s_flag[0] = conv;
        s_flag[1] = s_flag[1] | ((!isfinite(r) || !isfinite(sg)) ? 1 : 0);
        *s_chk = *s_chk + 1;
    }
    __syncwarp();
    CPHASE(4)
}

template <int M, int MODE>
__global__ void __launch_bounds__(OC2_MAX_W * 32) persist_cluster2_kernel(KArgs a, C2Args p) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    constexpr int MS = OC2<M>::MS, CW = OC2<M>::CW, LG = OC2<M>::L;
    extern __shared__ __align__(16) double sm[];
    const int T = p.T;
    const int TCM = max(p.TC0, p.TC);  // shared-memory row stride
    const int nw = blockDim.x >> 5;
    const int NS = T * nw;  // message slots per parity
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
    // message area, 16-byte aligned: row sums [2][NS][MS], check keys [2][NS][CW]
    unsigned long long* s_rs =
        reinterpret_cast<unsigned long long*>(sm + (((size_t)(9 * M + 2) * TCM + 1) & ~(size_t)1));
    unsigned long long* s_ck = s_rs + (size_t)2 * NS * MS;

    __shared__ __align__(8) unsigned long long s_mbar[2];
    __shared__ __align__(8) unsigned long long s_dbar[2];  // check decisions from tile 0 (by check parity)
    __shared__ __align__(16) double s_dec[2][OC2_DEC];
    __shared__ double s_zl[M], s_x1[M], s_R[4], s_rho[4], s_f[4], s_t[2], s_kap;
    __shared__ int s_flag[2], s_chk;  // conv, err; checks done (all calls)
    // role state kept in shared memory, not registers (the cell code needs them):
    // row warp lane i < M: lam, p, h, zeta, c, sum_k b0 of row (i, j);
    // consensus warp lane i < M: nu, x1, x_1 and the last contribution, pending f4
    __shared__ double s_row[6][M], s_con[5][M];

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int tile = (int)cluster.block_rank();
    const bool cons_warp = (tile == 0 && wid == nw - 1);
    const int nbt = (tile == 0 ? nw - 1 : nw) * 32;  // bulk threads of this CTA
    const long long j = blockIdx.x / T;
    const int k0 = tile == 0 ? 0 : p.TC0 + (tile - 1) * p.TC;
    const int ncell = min(tile == 0 ? p.TC0 : p.TC, a.n - k0);
    const long long qn = a.q * (long long)a.n_pad;
    const long long qq = a.q;
    const DParams& P = p.prm;
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
    // row scalars of source i: s_row[.][i], used by lane i (< M) of warp 0, the row warp
    if (tid < M) {
        const long long rix = (long long)tid * qq + j;
        const double lam = a.lam[rix] * cin.f[0], zeta = a.zeta[rix];
        s_row[0][tid] = lam;
        s_row[1][tid] = a.p[rix] * cin.f[1];
        s_row[2][tid] = a.h[rix];
        s_row[3][tid] = zeta;
        s_row[4][tid] = a.c[tid];
        s_row[5][tid] = a.sb0[rix];
        s_zl[tid] = zeta + lam;
        s_x1[tid] = cin.x1[tid];
    }
    // consensus warp (tile 0), lane i < M: nu, x1, x_1 and the last contribution of source i
    if (cons_warp && lane < M) {
        const long long rix = (long long)lane * qq + j;
        double nu = a.nu[rix];
        if (cin.nu_pending) nu = nu + cin.x1[lane] - a.x[(long long)lane * qn + j * a.n_pad];
        s_con[0][lane] = nu * cin.f[3];
        s_con[1][lane] = cin.x1[lane];
        s_con[2][lane] = 0.0;
        s_con[3][lane] = 0.0;
        s_con[4][lane] = 1.0;
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
        s_t[0] = cin.r;
        s_t[1] = cin.sigma;
        s_flag[0] = cin.status;
        s_flag[1] = cin.err;
        s_chk = cin.checks;
        mbar_init(smem_u32(&s_mbar[0]), 1);
        mbar_init(smem_u32(&s_mbar[1]), 1);
        mbar_init(smem_u32(&s_dbar[0]), 1);
        mbar_init(smem_u32(&s_dbar[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    int l_done = 0;
    const int ce = P.check_every;
    unsigned nchk = 0;     // checks done in this call
    bool x1_known = true;  // consensus warp: s_con[1] holds x1 of the previous iteration
    __syncthreads();
    cluster.sync();  // mates' shared memory and mbarriers are live before any message

    // this warp's message destinations in mate `lane` (lanes < T)
    const unsigned rank_l = (unsigned)min(lane, T - 1);
    const unsigned my_rs = smem_u32(s_rs + (size_t)(tile * nw + wid) * MS);
    const unsigned my_ck = smem_u32(s_ck + (size_t)(tile * nw + wid) * CW);
    const unsigned bar0 = smem_u32(&s_mbar[0]);
    const unsigned rs_par = (unsigned)(NS * MS * 8), ck_par = (unsigned)(NS * CW * 8);
#ifdef ADMM_PHASE_PROF
    // 0: tile 0 row warp lane 0, 1: consensus lane 0, 2: tile 1 row warp lane 0, 3: tile 1 warp 1 lane 0,
    // 4: any other row-warp / consensus lane 0 (only g_phase2all)
    const int prof_who = blockIdx.x == 0 ? (tid == 0 ? 0 : (cons_warp && lane == 0 ? 1 : -1))
                       : blockIdx.x == 1 ? (tid == 0 ? 2 : (tid == 32 ? 3 : (cons_warp && lane == 0 ? 4 : -1)))
                       : ((tid == 0 || (cons_warp && lane == 0)) ? 4 : -1);
    unsigned long long ph_acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, ph_last = clock64();
#endif

    const long long lim = P.iter_limit;
    int until_chk = ce > 0 ? (int)(ce - 1 - it0 % ce) : -1;  // iterations until the next check
    long long it = it0;
    for (; it < lim; ++it) {
        const long long u = it - it0;
        const int par = (int)(u & 1);
        const unsigned mph = (unsigned)((u >> 1) & 1);
        const bool is_check = (until_chk == 0);
        until_chk = is_check ? ce - 1 : until_chk - 1;
        if (tid == 0) mbar_expect(bar0 + 8 * par, rs_par + (is_check ? ck_par : 0u));
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
        bool sent = false;  // the consensus warp sends its partial early (non-check iterations)
        if (!cons_warp) {
            // ---- bulk cells c = tid (mod nbt), except the consensus cell k = 0.
            // Pairs (cc, cc + nbt) go through the interleaved two-cell chain.
            for (int cc = tid; cc < ncell && tid < nbt; cc += 2 * nbt) {
                const int c2 = cc + nbt;
                const bool two = (c2 < ncell) && (k0 + cc != 0);
                if (two) {
                    const int cs2[2] = {cc, c2};
                    double xo[M][2], xn[M][2], yy[2], vv[2], se[2], me[2];
#pragma unroll
                    for (int w = 0; w < 2; ++w) {
#pragma unroll
                        for (int i = 0; i < M; ++i) xo[i][w] = s_x[i * TCM + cs2[w]];
                        vv[w] = s_v[cs2[w]];
                        yy[w] = s_y[cs2[w]];
                        se[w] = fmax(vv[w], 0.0);
                        me[w] = vv[w] < 0.0 ? -vv[w] : 0.0;
                    }
                    gs_cell2_smem<M, MODE>(s_a2q, s_a1q, s_b2, s_b1, s_bq, s_ib, s_lo, s_hi, TCM, cs2,
                                           xo, xn, yy, se, me, zl, R);
#pragma unroll
                    for (int w = 0; w < 2; ++w) {
                        const int c = cs2[w];
                        double txo[M], txn[M];
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            txo[i] = xo[i][w];
                            txn[i] = xn[i][w];
                        }
                        s_v[c] = cell_tail<M>(txo, txn, yy[w], vv[w], 1.0, is_check, my_r1, my_s3);
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            const double b2 = s_b2[i * TCM + c], b1 = s_b1[i * TCM + c];
                            s_x[i * TCM + c] = txn[i];
                            if ((a.gfree >> i) & 1u) continue;  // g = 0: no row sum, dg = 0
                            fx[i] += __double2ll_rn(fma(b2, txn[i], b1) * txn[i] * p.fx_scale[i]);
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
                        fx[i] += __double2ll_rn(fma(cb2[i], xn[i], cb1[i]) * xn[i] * p.fx_scale[i]);
                        if (is_check) {
                            const double dg = (xn[i] - xo[i]) * fma(cb2[i], xn[i] + xo[i], cb1[i]);
                            dgx[i] = fmax(dgx[i], dg);
                            dgn[i] = fmin(dgn[i], dg);
                        }
                    }
                }
            }
        } else {
            // ---- consensus warp: x1 of iteration it-1 and (6h), then the k = 0 cell
            const int li = lane < M ? lane : 0;
            double c_nu = s_con[0][li], c_x1 = s_con[1][li];
            if (!x1_known) {
                double x1v[M];
                if (single) {
#pragma unroll
                    for (int i = 0; i < M; ++i) x1v[i] = s_con[3][i];
                } else {
                    ll_consensus<M>(p.pub + (size_t)((u - 1) & 3) * 2 * M * qq, qq, (unsigned)u, qtot, x1v);
                }
#pragma unroll
                for (int i = 0; i < M; ++i)
                    if (lane == i) c_x1 = x1v[i];
                c_nu = (c_nu + c_x1 - s_con[2][li]) * s_con[4][li];  // (6h) of iteration it-1
            }
            x1_known = false;
            PHASE2(0)
            double x1nu[M], cnu[M];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                cnu[i] = __shfl_sync(0xffffffffu, c_nu, i);
                x1nu[i] = __shfl_sync(0xffffffffu, c_x1, i) + cnu[i];
            }
            double xk0[M], xo[M], cb2[M], cb1[M];
            double yy = 0.0, vv = 0.0;
#pragma unroll
            for (int i = 0; i < M; ++i) xk0[i] = xo[i] = cb2[i] = cb1[i] = 0.0;
            if (lane == 0) {
                double a2q[M], a1q[M], bq[M], ib[M], clo[M], chi[M];
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const int e = i * TCM;
                    a2q[i] = s_a2q[e]; a1q[i] = s_a1q[e]; cb2[i] = s_b2[e]; cb1[i] = s_b1[e];
                    bq[i] = s_bq[e]; ib[i] = s_ib[e]; clo[i] = s_lo[e]; chi[i] = s_hi[e];
                    xo[i] = s_x[e];
                }
                vv = s_v[0];
                yy = s_y[0];
                gs_cell_prep<M, MODE>(a2q, a1q, cb2, cb1, bq, ib, clo, chi, xo, xk0, yy, fmax(vv, 0.0),
                                      vv < 0.0 ? -vv : 0.0, zl, R, true, x1nu);
            }
            PHASE2(1)
            // (6c)'s contribution x_1 - nu (nu before (6h)), lane i publishes source i
            double x0[M];
#pragma unroll
            for (int i = 0; i < M; ++i) x0[i] = __shfl_sync(0xffffffffu, xk0[i], 0);
            double c_x0 = 0.0, c_pub = 0.0;
#pragma unroll
            for (int i = 0; i < M; ++i)
                if (lane == i) {
                    c_x0 = x0[i];
                    c_pub = x0[i] - cnu[i];
                }
            if (lane < M && (!single || is_check))  // q = 1: only the residual check reads it
                ll_store(p.pub + 2 * ((size_t)(u & 3) * M * qq + (size_t)lane * qq + j), c_pub, (unsigned)(u + 1));
            if (!is_check) {
                // the row update waits on this partial: send it before the cell's bookkeeping
                unsigned long long w0[MS];
#pragma unroll
                for (int i = 0; i < MS; ++i) {
                    long long f = 0;
                    if (i < M && !((a.gfree >> i) & 1u))
                        f = __double2ll_rn(fma(cb2[i], x0[i], cb1[i]) * x0[i] * p.fx_scale[i]);
                    w0[i] = (unsigned long long)__shfl_sync(0xffffffffu, f, 0);
                }
                if (lane < T) {
                    const unsigned rb = mapa_u32(bar0 + 8 * par, rank_l);
                    const unsigned rs = mapa_u32(my_rs + par * rs_par, rank_l);
#pragma unroll
                    for (int i = 0; i < MS; i += 2) st_async2(rs + 8 * i, w0[i], w0[i + 1], rb);
                }
                sent = true;
            }
            if (lane < M) {
                s_con[0][lane] = c_nu;
                s_con[1][lane] = c_x1;
                s_con[2][lane] = c_x0;
                s_con[3][lane] = c_pub;
                s_con[4][lane] = 1.0;
            }
            if (is_check) {  // x_1 for the consensus residual, then one arrival of this row
                if (lane < M)
                    ll_store(p.chkx + 2 * ((size_t)(nchk & (OC2_BUFS - 1)) * M * qq + (size_t)lane * qq + j),
                             c_x0, nchk + 1);
                __syncwarp();
                if (lane == 0) gred_add_relaxed(p.cnt, 1ull);
            }
            if (lane == 0) {
                s_v[0] = cell_tail<M>(xo, xk0, yy, vv, 1.0, is_check, my_r1, my_s3);
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    s_x[i * TCM] = xk0[i];
                    if ((a.gfree >> i) & 1u) continue;
                    fx[i] += __double2ll_rn(fma(cb2[i], xk0[i], cb1[i]) * xk0[i] * p.fx_scale[i]);
                    if (is_check) {
                        const double dg = (xk0[i] - xo[i]) * fma(cb2[i], xk0[i] + xo[i], cb1[i]);
                        dgx[i] = fmax(dgx[i], dg);
                        dgn[i] = fmin(dgn[i], dg);
                    }
                }
            }
        }
        PHASE2(2)

        // ---- every warp: exact fixed-point warp sums (+ check keys) to every mate (st.async)
        if (!sent) {
            unsigned long long ws[MS];
#pragma unroll
            for (int i = 0; i < MS; ++i) ws[i] = i < M ? warp_sum_u64((unsigned long long)fx[i]) : 0ull;
            unsigned long long kk[CW];
            if (is_check) {
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    kk[i] = warp_max_key(okey(dgx[i]));
                    kk[M + i] = warp_max_key(okey(-dgn[i]));
                }
                kk[2 * M] = warp_max_key(nbits(my_r1));
                kk[2 * M + 1] = warp_max_key(nbits(my_s3));
            }
            if (lane < T) {
                const unsigned rb = mapa_u32(bar0 + 8 * par, rank_l);
                const unsigned rs = mapa_u32(my_rs + par * rs_par, rank_l);
#pragma unroll
                for (int i = 0; i < MS; i += 2) st_async2(rs + 8 * i, ws[i], ws[i + 1], rb);
                if (is_check) {
                    const unsigned ck = mapa_u32(my_ck + par * ck_par, rank_l);
#pragma unroll
                    for (int i = 0; i < CW; i += 2) st_async2(ck + 8 * i, kk[i], kk[i + 1], rb);
                }
            }
        }
        PHASE2(3)

        // ---- row warp: wait for the row's messages, row update, (check), publish to the CTA
        if (wid == 0) {
            const int li = lane < M ? lane : 0;
            // operands of the row update that do not depend on this iteration's sums
            double r_lam = s_row[0][li], r_p = s_row[1][li];
            const double r_h = s_row[2][li], r_zeta = s_row[3][li], r_c = s_row[4][li], r_sb0 = s_row[5][li];
            const double kap = s_kap, ndlam = nd * r_lam, hp = r_h + r_p;
            mbar_wait_cluster(bar0 + 8 * par, mph);
            PHASE2(4)
            // slot sums: lane (i = lane % LG, g = lane / LG) adds source i of slots g, g + 32/LG, ...;
            // a butterfly over g leaves the row total of source i in lane i (exact, mod 2^64)
            const unsigned long long* rsl = s_rs + (size_t)par * NS * MS;
            const int gi = lane % LG, gg = lane / LG;
            unsigned long long part = 0ull;
            if (gi < M)
                for (int f = gg; f < NS; f += 32 / LG) part += rsl[(size_t)f * MS + gi];
#pragma unroll
            for (int o = 16; o >= LG; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            const unsigned long long mysum = part;
            double mx = 0.0, mn = 0.0;
            unsigned long long kr1 = 0ull, ks3 = 0ull;
            if (is_check) {
                unsigned long long km[CW];
#pragma unroll
                for (int s = 0; s < CW; ++s) km[s] = 0ull;
                const unsigned long long* ckl = s_ck + (size_t)par * NS * CW;
                for (int f = lane; f < NS; f += 32)
#pragma unroll
                    for (int s = 0; s < CW; ++s) km[s] = max(km[s], ckl[(size_t)f * CW + s]);
#pragma unroll
                for (int s = 0; s < CW; ++s) km[s] = warp_max_key(km[s]);
#pragma unroll
                for (int i = 0; i < M; ++i)
                    if (lane == i) {
                        mx = okey_inv(km[i]);
                        mn = -okey_inv(km[M + i]);
                    }
                kr1 = km[2 * M];
                ks3 = km[2 * M + 1];
            }
            PHASE2(8)
            // row update (6b),(6g),(6d),(6i) via identity I1, identical in every CTA of the row:
            //   W = sum_k g - n lam, t = h + p - W, lam' = kappa t, zeta' = lam' - lam,
            //   1'z' = W + n lam', h' = min(c, 1'z' - p), p' = p + h' - 1'z'
            double zeta = r_zeta, h = r_h;
            double r2 = 0.0, r3 = 0.0, s1 = 0.0, s2 = 0.0;
            if (lane < M) {
                const double sg = (double)(long long)mysum * p.fx_inv[lane];
                if ((a.gfree >> lane) & 1u) mx = mn = 0.0;  // g-free source: dg = 0 for every k
                const double W = (sg + r_sb0) - ndlam;
                const double t = hp - W;
                const double lam = kap * t;
                zeta = lam - r_lam;
                const double oneTz = W + nd * lam;
                h = fmin(r_c, oneTz - r_p);
                const double pn = (r_p + h) - oneTz;
                if (is_check) {
                    const double dz = zeta - r_zeta;
                    r2 = fabs(zeta);
                    r3 = fabs(h - oneTz);
                    s1 = fmax(mx + dz, -(mn + dz));
                    s2 = fabs(h - r_h);
                }
                r_lam = lam;
                r_p = pn;
            }
            PHASE2(5)
            if (is_check)
                oc2_check<M>(p, a.hist, a.hist_cap, nd, tile, T, j, qq, qtot, u, it, nchk, r2, r3, s1, s2, kr1, ks3,
                             s_rho, s_f, s_R, s_t, s_flag, &s_chk, &s_kap, s_x1, &r_lam, &r_p, &s_dec[0][0],
                             smem_u32(&s_dbar[0]));
            if (lane < M) {
                s_row[0][lane] = r_lam;
                s_row[1][lane] = r_p;
                s_row[2][lane] = h;
                s_row[3][lane] = zeta;
                s_zl[lane] = zeta + r_lam;
            }
        }
        PHASE2(9)
        __syncthreads();  // zeta + lam (and, at checks, rho / flags / x1) of this iteration
        PHASE2(7)
        if (is_check) {
            ++nchk;
            // the consensus warp applies (6h) with the x1 just computed, then f4
            if (cons_warp) {
                if (lane < M) {
                    s_con[0][lane] = (s_con[0][lane] + s_x1[lane] - s_con[2][lane]) * s_f[3];
                    s_con[1][lane] = s_x1[lane];
                }
                x1_known = true;
            }
            // mu <-> rho3 on the cells this thread owns (no other thread touches them)
            const double f2 = s_f[2];
            if (f2 != 1.0) {
                if (cons_warp) {
                    if (lane == 0 && s_v[0] < 0.0) s_v[0] *= f2;
                } else if (tid < nbt) {
                    for (int c = tid; c < ncell; c += nbt)
                        if (k0 + c != 0 && s_v[c] < 0.0) s_v[c] *= f2;
                }
            }
            if (s_flag[1] || (s_flag[0] && P.stop_on_conv)) l_done = 1;
            if (l_done) {
                ++it;
                break;
            }
        }
    }
#ifdef ADMM_PHASE_PROF
    if (prof_who >= 0 && prof_who < 4)
        for (int k = 0; k < 10; ++k) g_phase2[prof_who][k] = ph_acc[k];
    if ((tid == 0 || (cons_warp && lane == 0)) && blockIdx.x < 1024) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        for (int k = 0; k < 10; ++k) g_phase2all[blockIdx.x][tid == 0 ? 0 : 1][k] = ph_acc[k];
        g_phase2all[blockIdx.x][tid == 0 ? 0 : 1][10] = smid;
    }
#endif
    // ---- (6h) of the last iteration if it was not a check, then write back
    const long long un = it - it0;  // iterations done in this call
    double c_nu = 0.0, c_x1 = 0.0;
    if (cons_warp) {
        const int li = lane < M ? lane : 0;
        c_nu = s_con[0][li];
        c_x1 = x1_known ? s_x1[li] : 0.0;
        if (!x1_known) {
            double x1v[M];
            if (single) {
#pragma unroll
                for (int i = 0; i < M; ++i) x1v[i] = s_con[3][i];
            } else {
                ll_consensus<M>(p.pub + (size_t)((un - 1) & 3) * 2 * M * qq, qq, (unsigned)un, qtot, x1v);
            }
#pragma unroll
            for (int i = 0; i < M; ++i)
                if (lane == i) c_x1 = x1v[i];
            c_nu = (c_nu + c_x1 - s_con[2][li]) * s_con[4][li];
        }
    }
    __syncthreads();  // s_x1 of the last check is read before the consensus warp overwrites it
    if (cons_warp && lane < M) s_x1[lane] = c_x1;
    __syncthreads();
    for (int t = tid; t < M * TCM; t += blockDim.x) {
        const int i = t / TCM, c = t - i * TCM;
        if (c < ncell) a.x[(long long)i * qn + j * a.n_pad + k0 + c] = s_x[t];
    }
    for (int c = tid; c < ncell; c += blockDim.x) a.v[j * a.n_pad + k0 + c] = s_v[c];
    if (tile == 0 && tid < M) {
        const long long rix = (long long)tid * qq + j;
        a.lam[rix] = s_row[0][tid];
        a.zeta[rix] = s_row[3][tid];
        a.h[rix] = s_row[2][tid];
        a.p[rix] = s_row[1][tid];
    }
    if (cons_warp && lane < M) a.nu[(long long)lane * qq + j] = c_nu;
    if (blockIdx.x == 0 && tid == 0) {
        Ctrl& co = a.ctrl[it & 1];
        for (int l = 0; l < 4; ++l) {
            co.rho[l] = s_rho[l];
            co.f[l] = 1.0;
        }
        for (int i = 0; i < MAXM; ++i) co.x1[i] = i < M ? s_x1[i] : 0.0;
        co.r = s_t[0];
        co.sigma = s_t[1];
        co.nu_pending = 0;
        co.done = l_done;
        co.status = s_flag[0];
        co.checks = s_chk;
        co.err = s_flag[1];
        __threadfence();
        *(volatile long long*)a.iter = it;
    }
    cluster.sync();  // no CTA exits while a mate may still touch its shared memory
}

}  // namespace admm_dev
