// sweep2.cu -- instantiations of the TMA streaming sweep (admm_sweep2.cuh) and
// its host-side plan; a translation unit of its own so the library builds in
// parallel (build.py).  The kernels are launched by admm.cu via sweep2_pick.
#define ADMM_KERNELS_NO_GLOBALS
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "admm_sweep2.cuh"

namespace admm_dev {

// stages of each warp's ring: two (6 KB each at m = 2: four CTAs per SM, 192 KB);
// ADMM_S2_NS=3 for experiments
const void* sweep2_pick(int m, int mode, int coeff_bytes, int* ns, size_t* smem) {
    int want = 2;
    if (const char* e = getenv("ADMM_S2_NS")) want = atoi(e) == 3 ? 3 : 2;
#define S2K(MM, CT, NN)                                                                           \
    if (m == MM && want == NN) {                                                                  \
        *ns = NN;                                                                                 \
        *smem = (size_t)S2_NW * NN * S2Cfg<MM, CT>::STAGE;                                                \
        return mode == BOX_EXACT ? (const void*)sweep2_kernel<MM, BOX_EXACT, CT, NN>              \
                                 : (const void*)sweep2_kernel<MM, BOX_PROJECT, CT, NN>;          \
    }
    if (coeff_bytes == 8) {
        S2K(1, double, 2) S2K(2, double, 2) S2K(3, double, 2) S2K(4, double, 2)
        S2K(1, double, 3) S2K(2, double, 3) S2K(3, double, 3) S2K(4, double, 3)
    } else {
        S2K(1, float, 2) S2K(2, float, 2) S2K(3, float, 2) S2K(4, float, 2)
        S2K(1, float, 3) S2K(2, float, 3) S2K(3, float, 3) S2K(4, float, 3)
    }
#undef S2K
    return nullptr;
}

// Units = (row, segment of TPS tiles).  Whole rows (S = 1) unless splitting rows
// balances the CTAs better: the estimated time of a split is the largest unit count
// of a CTA x its tiles per unit (+2 % per extra segment for the global row atomics).
S2Args sweep2_plan(long long q, long long n_pad, int g_max) {
    S2Args s{};
    s.TPR = (int)((n_pad + S2_TL - 1) / S2_TL);
    double best = 1e300;
    int best_S = 1;
    for (int S = 1; S <= s.TPR; ++S) {
        const int tps = (s.TPR + S - 1) / S;
        if ((s.TPR + tps - 1) / tps != S) continue;  // not a distinct split
        const long long U = q * S;
        const long long G = std::min<long long>(U, g_max);
        const double t = (double)((U + G - 1) / G) * tps * (1.0 + 0.02 * (S > 1));
        if (t < best * 0.98) {
            best = t;
            best_S = S;
        }
        if (U >= 64LL * g_max) break;
    }
    s.TPS = (s.TPR + best_S - 1) / best_S;
    s.S = (s.TPR + s.TPS - 1) / s.TPS;
    s.U = q * s.S;
    s.G = (int)std::min<long long>(s.U, g_max);
    return s;
}

}  // namespace admm_dev
