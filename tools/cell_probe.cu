// Dependent-chain latency (cycles, one warp) of the Algorithm-1 pieces and of one
// two-source Gauss-Seidel cell in its two arrangements (gs_cell_prep, gs_cell_lat).
// The Estrin / latency-arranged variants below were measured and NOT adopted: on sm_100a
// they are not faster (profiles/r02f/cell_probe.txt; an FMA takes one constant-bank operand,
// so Estrin's two-constant pairs cost extra moves, and the fp64 chains are short enough
// that Horner's fewer instructions win).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1903_10041_b200/csrc tools/cell_probe.cu -o /tmp/cellp
#include <cstdio>
#include "admm_kernels.cuh"
using namespace admm_dev;
namespace admm_dev {
// ----------------------------------------------------------------------------
// Latency-shortened evaluation of the trigonometric branch (the on-chip engines,
// whose iteration time is one cell's dependent fp64 chain): the same
// polynomials evaluated by Estrin's scheme (atan: depth 6 instead of 11 in s; cos /
// sin: 4 instead of 7 in w), the two candidate Vieta fixes of G5 computed side by side
// instead of select-then-divide, and 2 sqrt(-Q) supplied by the caller (it does not
// depend on the Gauss-Seidel predecessor).  Same closed form; the rounding differs from
// trig_pick by a few ulp (different association of the same sums).

// atan(y/x)-style angle theta = atan2(y, x) in [0, pi] for y >= 0, (x, y) != (0, 0)
__device__ __forceinline__ double atan2_upper_est(double y, double x) {
    const double ax = fabs(x);
    const bool yb = y > ax;
    const double mx = yb ? y : ax, mn = yb ? ax : y;
    const double r = mn * rcp_nr(mx);  // in [0, 1]
    const double s = r * r, s2 = s * s, s4 = s2 * s2, s8 = s4 * s4, s16 = s8 * s8;
#define A_(k) c_atan_pa[20 - (k)]
    const double p0 = fma(A_(1), s, A_(0)), p1 = fma(A_(3), s, A_(2)), p2 = fma(A_(5), s, A_(4));
    const double p3 = fma(A_(7), s, A_(6)), p4 = fma(A_(9), s, A_(8)), p5 = fma(A_(11), s, A_(10));
    const double p6 = fma(A_(13), s, A_(12)), p7 = fma(A_(15), s, A_(14)), p8 = fma(A_(17), s, A_(16));
    const double p9 = fma(A_(19), s, A_(18));
    const double q0 = fma(p1, s2, p0), q1 = fma(p3, s2, p2), q2 = fma(p5, s2, p4), q3 = fma(p7, s2, p6);
    const double q4 = fma(p9, s2, p8);
    const double r0 = fma(q1, s4, q0), r1 = fma(q3, s4, q2), r2 = fma(A_(20), s4, q4);
    const double pa = fma(r2, s16, fma(r1, s8, r0));
#undef A_
    double a = fma(r * s, pa, r);  // atan(min/max)
    if (yb) a = (1.5707963267948966 - a) + 6.123233995736766e-17;
    if (x < 0.0) a = (3.141592653589793 - a) + 1.2246467991473532e-16;
    return a;
}

// sin, cos of phi in [0, pi/3]
__device__ __forceinline__ void sincos_third_est(double phi, double* sn, double* cs) {
    const double w = phi * phi, w2 = w * w, w4 = w2 * w2;
#define C_(k) c_cos_pc[7 - (k)]
#define S_(k) c_sin_ps[6 - (k)]
    const double pc = fma(fma(fma(C_(7), w, C_(6)), w2, fma(C_(5), w, C_(4))), w4,
                          fma(fma(C_(3), w, C_(2)), w2, fma(C_(1), w, C_(0))));
    const double ps = fma(fma(S_(6), w2, fma(S_(5), w, S_(4))), w4,
                          fma(fma(S_(3), w, S_(2)), w2, fma(S_(1), w, S_(0))));
#undef C_
#undef S_
    *cs = fma(w, pc, 1.0);
    *sn = fma(phi * w, ps, phi);
}

// trig_pick with the shortened chains; t2 = 2 sqrt(-Q)
template <int MODE>
__device__ __forceinline__ double trig_pick_lat(double b, double c, double d, double t2, double R, double Delta,
                                                double lo, double hi) {
    const double b3 = b * (1.0 / 3.0);
    const double phi = atan2_upper_est(sqrt_pos(-Delta), R) * (1.0 / 3.0);
    double sn, cs;
    sincos_third_est(phi, &sn, &cs);
    const double h = 0.86602540378443864676 * sn;
    double xa = fma(t2, cs, -b3);                 // largest
    double xb = fma(t2, fma(-0.5, cs, -h), -b3);  // smallest
    const double xc = fma(t2, fma(-0.5, cs, h), -b3);
    // G5 as in trig_pick, both candidate fixes evaluated side by side
    const double aa = fabs(xa), ab = fabs(xb), ac = fabs(xc);
    const bool pa = (aa <= ab) && (aa <= ac);
    const bool pb = !pa && (ab <= ac);
    const double da = xb * xc, db = xa * xc;
    const double fa = -d * rcp_nr(da != 0.0 ? da : 1.0), fb = -d * rcp_nr(db != 0.0 ? db : 1.0);
    xa = (pa && da != 0.0) ? fa : xa;
    xb = (pb && db != 0.0) ? fb : xb;
    if (MODE == BOX_EXACT) {
        const double u = clampd(xb, lo, hi), w = clampd(xa, lo, hi);
        return right_well_lower(b, c, d, u, w) ? w : u;
    } else {
        const double xs = right_well_lower(b, c, d, xb, xa) ? xa : xb;
        return clampd(xs, lo, hi);
    }
}

// gs_cell_prep arranged for latency (the on-chip engines, where an iteration waits on
// one cell's chain): everything of source i that does not depend on the new x of the
// sources before it -- e, C, the normalised b and c, Q, b(9c - 2b^2)/54, Q^3 and
// 2 sqrt(-Q) -- is computed for all sources up front (independent chains the scheduler
// overlaps with source 0), so the Gauss-Seidel step from x^{(i-1)} to the cubic of
// source i is five dependent operations (phi, D, d, R, Delta) before Algorithm 1, whose
// trigonometric branch runs the shortened trig_pick_lat.  Same arithmetic up to the
// association of a few sums (R = b(9c - 2b^2)/54 - d/2, D = -rho3 phi + (a1/q - rho1 b1 e
// [- rho4 (x1 - nu)])), i.e. rounding-level differences from gs_cell_prep.
template <int M, int MODE>
__device__ __forceinline__ void gs_cell_lat(const double* a2q, const double* a1q, const double* cb2,
                                            const double* cb1, const double* bq, const double* ib2s,
                                            const double* clo, const double* chi, const double* xo,
                                            double* xn, double y, double s_e, double mu_e,
                                            const double* zl, const double* R, bool k0,
                                            const double* x1nu) {
    double K2[M], cn[M], hd[M], Qv[M], Q3[M], bP[M], t2[M], base[M], Cq[M];
    const double sym = (s_e + y) + mu_e;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const double xoi = xo[i];
        const double b2 = cb2[i], b1 = cb1[i];
        const double e = fma(fma(b2, xoi, b1), xoi, zl[i]);
        double C = fma(0.5 * R[0], fma(b1, b1, -2.0 * b2 * e), a2q[i] + 0.5 * R[1]);
        double k2 = fma(-R[0] * b1, e, a1q[i]);
        if (k0) {
            C += 0.5 * R[2];
            k2 += -R[2] * x1nu[i];
        }
        Cq[i] = C;
        K2[i] = k2;
        const double ia2 = ib2s[i] * R[3];  // 1 / 2A = 1 / (rho1 b2^2)
        const double b = bq[i];
        const double c = C * ia2;
        cn[i] = c;
        hd[i] = 0.5 * ia2;
        const double bb = b * b;
        const double Q = fma(3.0, c, -bb) * (1.0 / 9.0);
        Qv[i] = Q;
        Q3[i] = (Q * Q) * Q;
        bP[i] = (b * fma(9.0, c, -2.0 * bb)) * (1.0 / 54.0);
        t2[i] = 2.0 * sqrt_pos(fmax(-Q, 0.0));
        // phi minus the new x of the sources before i: the old x of the sources after i
        double later = 0.0;
#pragma unroll
        for (int l = i + 1; l < M; ++l) later += xo[l];
        base[i] = sym - later;
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double before = 0.0;
#pragma unroll
        for (int l = 0; l < i; ++l) before += xn[l];
        const double phi = base[i] - before;
        const double D = fma(-R[1], phi, K2[i]);
        if (cb2[i] != 0.0) {
            const double d = D * hd[i];
            const double Rr = fma(-0.5, d, bP[i]);
            const double De = fma(Rr, Rr, Q3[i]);
            const bool trig = isfinite(De) && !(De > 0.0) && !(Qv[i] == 0.0 && Rr == 0.0);
            xn[i] = trig ? trig_pick_lat<MODE>(bq[i], cn[i], d, t2[i], Rr, De, clo[i], chi[i])
                         : quartic_core<MODE>(bq[i], cn[i], d, Cq[i], D, clo[i], chi[i]);
        } else {
            xn[i] = clampd(-D * rcp_nr(2.0 * Cq[i]), clo[i], chi[i]);  // A = B = 0: quadratic
        }
    }
}

}  // namespace admm_dev

#define CHAIN 128
template <int OP>
__global__ void lat(double seed, double* out, long long* cyc) {
    double x = seed;
    // a PHEV-like cell: engine (a2 > 0, b2 = 0: quadratic in g) and battery sources
    double a2q[2] = {2e-4, 1e-4}, a1q[2] = {1e-2, 0.0}, cb2[2] = {1e-4, 2e-4}, cb1[2] = {1.0, 1.1};
    double bq[2], ib[2], lo[2] = {0.0, -30.0}, hi[2] = {60.0, 30.0}, xo[2] = {20.0, 3.0}, xn[2];
    double zl[2] = {-0.01, 0.02}, R[4] = {1e-2, 1e-2, 1e-2, 100.0}, x1nu[2] = {0, 0};
    for (int i = 0; i < 2; ++i) {
        bq[i] = 1.5 * cb1[i] / cb2[i];
        ib[i] = 1.0 / (cb2[i] * cb2[i]);
    }
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < CHAIN; ++it) {
        const double y = 25.0 + 1e-12 * x;
        if (OP == 0) gs_cell_prep<2, 0>(a2q, a1q, cb2, cb1, bq, ib, lo, hi, xo, xn, y, 0.0, 0.0, zl, R, false, x1nu);
        if (OP == 1) gs_cell_lat<2, 0>(a2q, a1q, cb2, cb1, bq, ib, lo, hi, xo, xn, y, 0.0, 0.0, zl, R, false, x1nu);
        if (OP == 2) { xn[0] = quartic_core<0>(bq[0], 0.3 + 1e-12 * x, -50.0, 1.0, 1.0, -1e5, 1e5); xn[1] = 0; }
        if (OP == 3) {
            const double b = bq[0], c = 0.3 + 1e-12 * x, d = -50.0;
            const double bb = b * b, Q = fma(3.0, c, -bb) * (1.0 / 9.0);
            const double Rr = fma(b, fma(9.0, c, -2.0 * bb), -27.0 * d) * (1.0 / 54.0);
            const double De = fma(Q * Q, Q, Rr * Rr);
            xn[0] = trig_pick_lat<0>(b, c, d, 2.0 * sqrt_pos(-Q), Rr, De, -1e5, 1e5);
            xn[1] = 0;
        }
        if (OP == 4) { xn[0] = atan2_upper(0.5 + 1e-12 * x, 0.3); xn[1] = 0; }
        if (OP == 5) { xn[0] = atan2_upper_est(0.5 + 1e-12 * x, 0.3); xn[1] = 0; }
        if (OP == 6) { double s, c; sincos_third(0.5 + 1e-12 * x, &s, &c); xn[0] = s + c; xn[1] = 0; }
        if (OP == 7) { double s, c; sincos_third_est(0.5 + 1e-12 * x, &s, &c); xn[0] = s + c; xn[1] = 0; }
        if (OP == 8) { xn[0] = rcp_nr(3.0 + 1e-12 * x); xn[1] = 0; }
        if (OP == 9) { xn[0] = sqrt_pos(3.0 + 1e-12 * x); xn[1] = 0; }
        x = x + (xn[0] + xn[1]) * 1e-30;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x + xn[0];
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* d; long long* c; cudaMalloc(&d, 1024 * 8); cudaMalloc(&c, 8);
    const char* names[] = {"cell gs_cell_prep", "cell gs_cell_lat", "quartic_core trig", "trig_pick_lat",
                           "atan2_upper", "atan2_upper_est", "sincos_third", "sincos_third_est", "rcp_nr", "sqrt_pos"};
    void (*k[])(double, double*, long long*) = {lat<0>, lat<1>, lat<2>, lat<3>, lat<4>, lat<5>, lat<6>, lat<7>, lat<8>, lat<9>};
    for (int o = 0; o < 10; ++o) {
        long long h = 0;
        for (int rep = 0; rep < 3; ++rep) {
            k[o]<<<1, 32>>>(0.7, d, c);
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-20s %8.1f cycles/op (1 warp)\n", names[o], (double)h / CHAIN);
    }
    return 0;
}
