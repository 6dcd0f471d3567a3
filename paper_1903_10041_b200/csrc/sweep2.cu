// sweep2.cu -- instantiations of the TMA streaming sweep (admm_sweep2.cuh) and
// its host-side plan; a translation unit of its own so the library builds in
// parallel (build.py).  The kernels are launched by admm.cu via sweep2_pick.
#define ADMM_KERNELS_NO_GLOBALS
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "admm_sweep2.cuh"

namespace admm_dev {

// Kernel choice.  Many rows (q >= 16, the box shared by every row and L1/L2-resident):
// two cells per lane, 64-cell chunks (four CTAs per SM at m <= 2).  Few rows (horizon-type
// problems): one cell per lane with the box staged by TMA next to the coefficients
// (32-cell chunks, up to three CTAs per SM at m = 4).  ADMM_S2_L=1/2 forces the layout.
// Two ring stages per warp.
const void* sweep2_pick(int m, int mode, int coeff_bytes, long long q, int* ns, size_t* smem, int* tl) {
    bool one = q < 16;
    if (const char* e = getenv("ADMM_S2_L")) one = (e[0] == '1');
#define S2K(MM, CT, LL, BB)                                                                      \
    if (m == MM) {                                                                               \
        *ns = 2;                                                                                 \
        *tl = S2Cfg<MM, CT, LL, BB>::TL;                                                         \
        *smem = (size_t)S2_NW * 2 * S2Cfg<MM, CT, LL, BB>::STAGE;                                \
        return mode == BOX_EXACT ? (const void*)sweep2_kernel<MM, BOX_EXACT, CT, 2, LL, BB>      \
                                 : (const void*)sweep2_kernel<MM, BOX_PROJECT, CT, 2, LL, BB>;  \
    }
    if (coeff_bytes == 8) {
        if (one) {
            S2K(1, double, 1, true) S2K(2, double, 1, true) S2K(3, double, 1, true) S2K(4, double, 1, true)
        } else {
            S2K(1, double, 2, false) S2K(2, double, 2, false) S2K(3, double, 2, false) S2K(4, double, 2, false)
        }
    } else {
        if (one) {
            S2K(1, float, 1, true) S2K(2, float, 1, true) S2K(3, float, 1, true) S2K(4, float, 1, true)
        } else {
            S2K(1, float, 2, false) S2K(2, float, 2, false) S2K(3, float, 2, false) S2K(4, float, 2, false)
        }
    }
#undef S2K
    return nullptr;
}

// Units = (row, segment of TPS chunks).  Whole rows (S = 1) unless splitting rows
// balances the CTAs better: the estimated time of a split is the largest unit count
// of a CTA x (its chunks per unit + a fixed per-unit cost).
S2Args sweep2_plan(long long q, long long n_pad, int tl, int g_max) {
    S2Args s{};
    s.TPR = (int)((n_pad + tl - 1) / tl);
    double best = 1e300;
    int best_S = 1;
    for (int S = 1; S <= s.TPR; ++S) {
        const int tps = (s.TPR + S - 1) / S;
        if ((s.TPR + tps - 1) / tps != S) continue;  // not a distinct split
        const long long U = q * S;
        const long long G = std::min<long long>(U, g_max);
        // + ~3 chunks of fixed cost per unit (row scalars, finalisation, row atomics):
        // measured at q = 1e3 (S = 1 / 2 / 4: 35 / 30 / 26 % of the HBM peak)
        const double t = (double)((U + G - 1) / G) * (tps + 3.0);
        if (t < best * 0.98) {
            best = t;
            best_S = S;
        }
        if (U >= 64LL * g_max) break;
    }
    if (const char* e = getenv("ADMM_S2_S")) best_S = std::max(1, std::min(s.TPR, atoi(e)));  // experiments
    s.TPS = (s.TPR + best_S - 1) / best_S;
    s.S = (s.TPR + s.TPS - 1) / s.TPS;
    s.U = q * s.S;
    s.G = (int)std::min<long long>(s.U, g_max);
    return s;
}

}  // namespace admm_dev
