// Latency probe: dependent-chain cycles of the fp64 building blocks of
// Algorithm 1 and of quartic_boxmin itself on one thread (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1903_10041_b200/csrc tools/lat_probe.cu -o /tmp/lat
#include <cstdio>
#include "quartic.cuh"
using namespace admm_dev;

#define CHAIN 256
template <int OP>
__global__ void lat(double seed, double* out, long long* cyc) {
    double x = seed;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < CHAIN; ++i) {
        if (OP == 0) x = sqrt(x + 1.0);
        if (OP == 1) x = 1.0 / (x + 1.0);
        if (OP == 2) x = cbrt(x + 1.0);
        if (OP == 3) x = atan2(x + 0.5, 0.3);
        if (OP == 4) { double s, c; sincos(x, &s, &c); x = s + c; }
        if (OP == 5) x = fma(x, 1.0000001, 1e-9);
        if (OP == 6) x = quartic_boxmin<0>(1e-10, 2e-6, 5e-5 + 1e-12 * x, -2.0, -5e4, 5e4) * 1e-20 + x;  // trig (PHEV-like)
        if (OP == 7) x = quartic_boxmin<0>(0.0, 0.0, 3e-6, -2.0 + 1e-12 * x, 0.0, 1e5) * 1e-20 + x;        // quadratic
        if (OP == 8) x = quartic_boxmin<0>(1.0, 1.0, 5.0 + 1e-12 * x, -2.0, -10., 10.) * 1e-20 + x;       // Cardano
        if (OP == 9) x = exp(x * 1e-3);
        if (OP == 10) x = log(x + 2.0);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* d; long long* c; cudaMalloc(&d, 1024 * 8); cudaMalloc(&c, 8);
    const char* names[] = {"sqrt", "rcp/div", "cbrt", "atan2", "sincos", "dfma", "boxmin trig", "boxmin quad", "boxmin cardano", "exp", "log"};
    void (*k[])(double, double*, long long*) = {lat<0>, lat<1>, lat<2>, lat<3>, lat<4>, lat<5>, lat<6>, lat<7>, lat<8>, lat<9>, lat<10>};
    for (int o = 0; o < 11; ++o) {
        long long h = 0;
        for (int rep = 0; rep < 3; ++rep) {
            k[o]<<<1, 32>>>(0.7, d, c);
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-16s %8.1f cycles/op (1 warp)\n", names[o], (double)h / CHAIN);
    }
    // throughput: many warps
    return 0;
}
