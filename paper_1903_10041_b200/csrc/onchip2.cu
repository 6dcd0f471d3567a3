// onchip2.cu -- instantiations of the message-passing cluster-row engine
// (admm_onchip2.cuh); a translation unit of its own so the library builds in
// parallel (build.py).  Launched by admm.cu via cluster2_pick.
#define ADMM_KERNELS_NO_GLOBALS
#include <cuda_runtime.h>

#include "admm_onchip2.cuh"

namespace admm_dev {

const void* cluster2_pick(int m, int mode) {
#define S(MM)                                                                                   \
    if (m == MM)                                                                                \
        return mode == BOX_EXACT ? (const void*)persist_cluster2_kernel<MM, BOX_EXACT>          \
                                 : (const void*)persist_cluster2_kernel<MM, BOX_PROJECT>;
    S(1) S(2) S(3) S(4)
#undef S
    return nullptr;
}

}  // namespace admm_dev

#ifdef ADMM_PHASE_PROF
extern "C" int admm_debug_phase2(unsigned long long* out40) {
    return cudaMemcpyFromSymbol(out40, admm_dev::g_phase2, sizeof(admm_dev::g_phase2)) == cudaSuccess ? 0 : 1;
}
extern "C" int admm_debug_phase2all(unsigned long long* out) {  // [1024][2][11]
    return cudaMemcpyFromSymbol(out, admm_dev::g_phase2all, sizeof(admm_dev::g_phase2all)) == cudaSuccess ? 0 : 1;
}
extern "C" int admm_debug_phase2c(unsigned long long* out12) {  // and reset
    int rc = cudaMemcpyFromSymbol(out12, admm_dev::g_phase2c, sizeof(admm_dev::g_phase2c)) == cudaSuccess ? 0 : 1;
    unsigned long long z[12] = {0};
    cudaMemcpyToSymbol(admm_dev::g_phase2c, z, sizeof(z));
    return rc;
}
#endif
