// Memory-structure probe for the streaming sweep (no ADMM arithmetic): what HBM
// bandwidth does the sweep's access pattern reach by itself?
//   rows of n = 1000 doubles (n_pad = 1000), q rows per stream, 12 read streams
//   (x0, x1, a2_0, a2_1, a1_0, a1_1, b2_0, b2_1, b1_0, b1_1, y, v) + lo/hi
//   (2 x 2 rows shared by all scenarios) and 3 written streams (x0, x1, v).
// Variants: (0) item = row per CTA of 512 threads x 2 cells, block barrier per item,
// (1) same without the barrier, (2) 256 threads x 4 cells, 2 CTAs/SM, barrier,
// (3) flat grid-stride over all cells (no rows), 2 cells per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/stream_probe.cu -o tools/stream_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NS = 12;
struct P {
    const double* in[NS];
    double* out[3];
    const double *lo, *hi;
    long long q;
    int n;
};

template <int U, bool BAR>
__global__ void item_kernel(P p) {
    const int tid = threadIdx.x;
    const int k = U * tid;
    const bool inb = k < p.n;
    for (long long j = blockIdx.x; j < p.q; j += gridDim.x) {
        double acc[U] = {};
        double o0[U], o1[U], o2[U];
        if (inb) {
            const long long e = j * p.n + k;
#pragma unroll
            for (int s = 0; s < NS; ++s)
#pragma unroll
                for (int h = 0; h < U; h += 2) {
                    const double2 t = __ldg(reinterpret_cast<const double2*>(p.in[s] + e + h));
                    acc[h] += t.x;
                    acc[h + 1] += t.y;
                }
#pragma unroll
            for (int h = 0; h < U; h += 2) {
                const double2 l = __ldg(reinterpret_cast<const double2*>(p.lo + k + h));
                const double2 u = __ldg(reinterpret_cast<const double2*>(p.hi + k + h));
                acc[h] += l.x * u.x;
                acc[h + 1] += l.y * u.y;
            }
#pragma unroll
            for (int h = 0; h < U; ++h) {
                o0[h] = acc[h];
                o1[h] = acc[h] * 0.5;
                o2[h] = acc[h] * 0.25;
            }
#pragma unroll
            for (int h = 0; h < U; h += 2) {
                *reinterpret_cast<double2*>(p.out[0] + e + h) = make_double2(o0[h], o0[h + 1]);
                *reinterpret_cast<double2*>(p.out[1] + e + h) = make_double2(o1[h], o1[h + 1]);
                *reinterpret_cast<double2*>(p.out[2] + e + h) = make_double2(o2[h], o2[h + 1]);
            }
        }
        if (BAR) __syncthreads();
    }
}

__global__ void flat_kernel(P p) {
    const long long N = p.q * p.n;
    for (long long c = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x); c < N;
         c += 2LL * gridDim.x * blockDim.x) {
        double a0 = 0, a1 = 0;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const double2 t = __ldg(reinterpret_cast<const double2*>(p.in[s] + c));
            a0 += t.x;
            a1 += t.y;
        }
        const int k = (int)(c % p.n);
        const double2 l = __ldg(reinterpret_cast<const double2*>(p.lo + k));
        a0 += l.x;
        a1 += l.y;
        *reinterpret_cast<double2*>(p.out[0] + c) = make_double2(a0, a1);
        *reinterpret_cast<double2*>(p.out[1] + c) = make_double2(a0 * .5, a1 * .5);
        *reinterpret_cast<double2*>(p.out[2] + c) = make_double2(a0 * .25, a1 * .25);
    }
}

int main(int argc, char** argv) {
    const long long q = argc > 1 ? atoll(argv[1]) : 10000;
    const int n = 1000;
    P p{};
    p.q = q;
    p.n = n;
    const size_t B = (size_t)q * n * 8;
    for (int s = 0; s < NS; ++s) {
        double* d;
        cudaMalloc(&d, B);
        cudaMemset(d, 0, B);
        p.in[s] = d;
    }
    for (int s = 0; s < 3; ++s) cudaMalloc(&p.out[s], B);
    double *lo, *hi;
    cudaMalloc(&lo, n * 8 * 2);
    cudaMalloc(&hi, n * 8 * 2);
    cudaMemset(lo, 0, n * 16);
    cudaMemset(hi, 0, n * 16);
    p.lo = lo;
    p.hi = hi;
    char* flush;
    cudaMalloc(&flush, 512 << 20);
    const double bytes = (double)B * (NS + 3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[] = {"item 512x2 barrier", "item 512x2 no-barrier", "item 256x4 barrier (2/SM)",
                           "item 256x2 barrier (4/SM, 64 regs)", "flat grid-stride 2 cells"};
    for (int v = 0; v < 5; ++v) {
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            cudaMemset(flush, rep, 512 << 20);
            cudaEventRecord(e0);
            if (v == 0) item_kernel<2, true><<<148, 512>>>(p);
            if (v == 1) item_kernel<2, false><<<148, 512>>>(p);
            if (v == 2) item_kernel<4, true><<<296, 256>>>(p);
            if (v == 3) item_kernel<2, true><<<592, 512>>>(p);
            if (v == 4) flat_kernel<<<148 * 4, 512>>>(p);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        printf("%-40s q=%lld  %.3f ms  %.0f GB/s\n", names[v], q, best, bytes / best / 1e6);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
