/*
 * oracle.c -- plain CPU oracle (TEST INFRASTRUCTURE ONLY; see oracle.h).
 *
 * Compiled with -O2 -ffp-contract=off, fp64, single thread.  Each function
 * cites the PAPER.md passage it follows.  No blocking, fusion or reordering
 * beyond the printed algorithm; the only deviations are the readings listed
 * in DESIGN.md §Readings, cited where they apply.
 */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdlib.h>
#include <string.h>

/* OpenMP build (liboracle_omp.so, the "CPU-parallel" baseline of bench.py):
   the loops over independent (j,k) cells and (i,j) rows are shared out over
   threads; every sum stays serial inside its row and every max is
   order-independent, so the results are bitwise those of the serial build.
   orc_set_threads is a no-op in the serial build. */
int orc_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* ------------------------------------------------------------------------- */
/* small helpers                                                             */
/* ------------------------------------------------------------------------- */

static double clampd(double v, double lo, double hi)
{
    /* projection onto [lo, hi] (Pi_I) */
    if (v < lo) return lo;
    if (v > hi) return hi;
    return v;
}

/* Neumaier compensated sum: the oracle's sums over k and j are near-exact and
   independent of any blocking (SURVEY.md §8(c) "Sums"). */
typedef struct { double s, comp; } nsum;
static void nsum_add(nsum *a, double v)
{
    double t = a->s + v;
    if (fabs(a->s) >= fabs(v)) a->comp += (a->s - t) + v;
    else a->comp += (v - t) + a->s;
    a->s = t;
}
static double nsum_val(const nsum *a) { return a->s + a->comp; }

/* quartic value J(x) = A x^4 + B x^3 + C x^2 + D x (E dropped: irrelevant to argmin) */
static double quartic_val(double A, double B, double C, double D, double x)
{
    return (((A * x + B) * x + C) * x + D) * x;
}

static double cubic_val(double b, double c, double d, double x)
{
    return ((x + b) * x + c) * x + d;
}

/* Guarded Newton polish of one cubic root: oracle-only (SURVEY.md §8(c)
   "BOXMIN (oracle version)"; the GPU path never iterates).  A step is kept
   only if it strictly reduces |p(x)|. */
static double polish(double b, double c, double d, double x)
{
    double px = cubic_val(b, c, d, x);
    for (int it = 0; it < 8 && px != 0.0; ++it) {
        double dp = (3.0 * x + 2.0 * b) * x + c;
        if (dp == 0.0 || !isfinite(dp)) break;
        double xn = x - px / dp;
        double pn = cubic_val(b, c, d, xn);
        if (!(fabs(pn) < fabs(px))) break;
        x = xn;
        px = pn;
    }
    return x;
}

/* ------------------------------------------------------------------------- */
/* Algorithm 1                                            */
/* ------------------------------------------------------------------------- */

/* Real roots of x^3 + b x^2 + c x + d, sorted ascending.
   branch: 0 = Vieta triple root (Q=R=0), 1 = Cardano (Delta>0),
           2 = trigonometric (Delta<=0).  Returns the number of roots (1 or 3). */
int orc_cubic_roots(double b, double c, double d, double roots[3], int *branch)
{
    /* PAPER.md:139-141 */
    double Q = c / 3.0 - b * b / 9.0;
    double R = b * c / 6.0 - b * b * b / 27.0 - d / 2.0;
    double Delta = Q * Q * Q + R * R;
    int nr;
    if (Delta > 0.0) {
        /* Cardano.  Reading G4: T = cbrt(R - sqrt(Delta)) is
           evaluated as -Q/S with S = cbrt(R + sign(R) sqrt(Delta)) (S*T = -Q),
           which avoids the cancellation of R - sqrt(Delta).  The polish below
           removes any remaining closed-form error. */
        double sq = sqrt(Delta);
        double S = cbrt(R >= 0.0 ? R + sq : R - sq);
        double T = (S != 0.0) ? -Q / S : 0.0;
        roots[0] = S + T - b / 3.0;
        nr = 1;
        *branch = 1;
    } else if (Q == 0.0 && R == 0.0) {
        /* Vieta triple root */
        roots[0] = -b / 3.0;
        nr = 1;
        *branch = 0;
    } else {
        /* trigonometric, PAPER.md:143-152 (Delta <= 0, so Q < 0).  The acos
           argument is clamped to [-1, 1] against rounding. */
        double sqmQ = sqrt(-Q);
        double arg = R / sqrt(-Q * Q * Q);
        arg = clampd(arg, -1.0, 1.0);
        double th = acos(arg);
        const double pi = 3.14159265358979323846;
        double xa = 2.0 * sqmQ * cos(th / 3.0) - b / 3.0;
        double xb = 2.0 * sqmQ * cos(th / 3.0 + 2.0 * pi / 3.0) - b / 3.0;
        double xc = 2.0 * sqmQ * cos(th / 3.0 + 4.0 * pi / 3.0) - b / 3.0;
        roots[0] = xa;
        roots[1] = xb;
        roots[2] = xc;
        nr = 3;
        *branch = 2;
    }
    for (int i = 0; i < nr; ++i) roots[i] = polish(b, c, d, roots[i]);
    /* "sorting the roots": plain insertion sort */
    for (int i = 1; i < nr; ++i)
        for (int j = i; j > 0 && roots[j] < roots[j - 1]; --j) {
            double t = roots[j];
            roots[j] = roots[j - 1];
            roots[j - 1] = t;
        }
    return nr;
}

/* Candidate set -> the one with the smallest J; ties go to the smaller x
   (Algorithm 1's strict "delta f > 0" test; reading G8).
   J is evaluated directly by Horner, not by the paper's delta-f shortcut.
   *tie is set when the best two distinct candidates agree within 8 eps. */
static double pick_min(double A, double B, double C, double D, const double *cand, int nc,
                       int *tie)
{
    int best = -1;
    double jb = 0.0;
    for (int i = 0; i < nc; ++i) {
        double ji = quartic_val(A, B, C, D, cand[i]);
        if (best < 0 || ji < jb || (ji == jb && cand[i] < cand[best])) {
            best = i;
            jb = ji;
        }
    }
    if (tie) {
        *tie = 0;
        for (int i = 0; i < nc; ++i) {
            if (i == best || cand[i] == cand[best]) continue;
            double ji = quartic_val(A, B, C, D, cand[i]);
            if (fabs(ji - jb) <= 8.0 * 2.220446049250313e-16 * (fabs(ji) + fabs(jb))) *tie = 1;
        }
    }
    return cand[best];
}

/* Reading G9: the quadratic formula is used only when A == 0 exactly, or when
   the reduced cubic's Q, R, Delta overflow (A so small that b, c, d are not
   representable).  In the ADMM, A == 0 implies B == 0 (A = rho1 b2^2/2,
   B = rho1 b2 b1) and C >= rho3/2 > 0. */
static int quartic_is_quadratic(double A, double B, double C, double D)
{
    if (A == 0.0) return 1;
    double b = 3.0 * B / (4.0 * A), c = C / (2.0 * A), d = D / (4.0 * A);
    double Q = c / 3.0 - b * b / 9.0;
    double R = b * c / 6.0 - b * b * b / 27.0 - d / 2.0;
    double Delta = Q * Q * Q + R * R;
    return !(isfinite(Q) && isfinite(R) && isfinite(Delta));
}

/* Global minimiser over the reals of J(x) = A x^4 + B x^3 + C x^2 + D x
   (A >= 0).  Definition: the stationary point (real root of J') with the
   smallest J.  PAPER.md:129-137 (b = 3B/4A, c = C/2A, d = D/4A). */
double orc_quartic_argmin(double A, double B, double C, double D, int *tie)
{
    if (tie) *tie = 0;
    if (quartic_is_quadratic(A, B, C, D)) {
        if (!(C > 0.0)) return NAN; /* unbounded: not a valid instance */
        return -D / (2.0 * C);
    }
    double b = 3.0 * B / (4.0 * A), c = C / (2.0 * A), d = D / (4.0 * A);
    double r[3];
    int br;
    int nr = orc_cubic_roots(b, c, d, r, &br);
    return pick_min(A, B, C, D, r, nr, tie);
}

/* Minimiser of J over [lo, hi].
   PROJECT: clamp(argmin_R J)  -- Eq. (6a) as printed.
   EXACT:   argmin over {lo, hi} U {real stationary points in (lo, hi)} -- the
            exact block minimiser of L, which contains the box indicator
            (PAPER.md:396); reading G3. */
double orc_quartic_boxmin(double A, double B, double C, double D, double lo, double hi,
                          int mode, int *tie)
{
    if (mode == ORC_BOX_PROJECT) return clampd(orc_quartic_argmin(A, B, C, D, tie), lo, hi);
    double cand[5];
    int nc = 0;
    if (isfinite(lo)) cand[nc++] = lo;
    if (isfinite(hi)) cand[nc++] = hi;
    if (quartic_is_quadratic(A, B, C, D)) {
        if (!(C > 0.0)) return NAN;
        double v = -D / (2.0 * C);
        if (v > lo && v < hi) cand[nc++] = v;
    } else {
        double b = 3.0 * B / (4.0 * A), c = C / (2.0 * A), d = D / (4.0 * A);
        double r[3];
        int br;
        int nr = orc_cubic_roots(b, c, d, r, &br);
        for (int i = 0; i < nr; ++i)
            if (r[i] > lo && r[i] < hi) cand[nc++] = r[i];
    }
    if (nc == 0) return clampd(0.0, lo, hi); /* unreachable for A>0 or C>0 */
    return pick_min(A, B, C, D, cand, nc, tie);
}

void orc_quartic_batch(const double *A, const double *B, const double *C, const double *D,
                       const double *lo, const double *hi, double *x, long N, int mode,
                       long *ties)
{
    long t = 0;
#pragma omp parallel for reduction(+ : t) schedule(static)
    for (long e = 0; e < N; ++e) {
        int tie = 0;
        x[e] = orc_quartic_boxmin(A[e], B[e], C[e], D[e], lo ? lo[e] : -INFINITY,
                                  hi ? hi[e] : INFINITY, mode, &tie);
        t += tie;
    }
    if (ties) *ties = t;
}

/* Coefficients of the (6a) objective in its rewritten theta/phi form
   (PAPER.md:452-463):
     J(x) = (1/q) f(x) + rho1/2 (theta - g(x))^2 + rho3/2 (phi - x)^2
            + delta_{k,1} rho4/2 (x1 - x + nu)^2
   expanded with e = theta - b0 (derivation in DESIGN.md). */
void orc_build_quartic(double a2, double a1, double b2, double b1, double b0, double theta,
                       double phi, double qd, const double rho[4], int delta, double x1,
                       double nu, double out[4])
{
    double e = theta - b0;
    double A = rho[0] * b2 * b2 / 2.0;
    double B = rho[0] * b2 * b1;
    double C = rho[0] * (b1 * b1 - 2.0 * b2 * e) / 2.0 + a2 / qd + rho[2] / 2.0;
    double D = -rho[0] * b1 * e + a1 / qd - rho[2] * phi;
    if (delta) {
        C += rho[3] / 2.0;
        D += -rho[3] * (x1 + nu);
    }
    out[0] = A;
    out[1] = B;
    out[2] = C;
    out[3] = D;
}

/* ------------------------------------------------------------------------- */
/* ADMM (Appendix A)                                                */
/* ------------------------------------------------------------------------- */

#define IX(i, j, k) (((long)(i) * q + (j)) * n + (k)) /* [m][q][n] */
#define JK(j, k) ((long)(j) * n + (k))               /* [q][n] */
#define IJ(i, j) ((long)(i) * q + (j))               /* [m][q] */
#define IK(i, k) ((long)(i) * n + (k))               /* [m][n] */

static double gfun(const orc_problem *P, long e, double x)
{
    /* g_k^{(i,j)}(x) = b2 x^2 + b1 x + b0 (Assumption 3) */
    return P->b2[e] * x * x + P->b1[e] * x + P->b0[e];
}

static double ffun(const orc_problem *P, long e, double x)
{
    /* f_k^{(i,j)}(x) = a2 x^2 + a1 x + a0 (Assumption 3) */
    return P->a2[e] * x * x + P->a1[e] * x + P->a0[e];
}

int orc_validate(const orc_problem *P, char *msg, int msglen)
{
    int m = P->m;
    long n = P->n, q = P->q;
    if (m <= 0 || n <= 0 || q <= 0 || P->q_total < q) {
        snprintf(msg, msglen, "bad dimensions");
        return ORC_INVALID;
    }
    for (int i = 0; i < m; ++i)
        for (long j = 0; j < q; ++j)
            for (long k = 0; k < n; ++k) {
                long e = IX(i, j, k);
                /* Assumption 1 under Assumption 3: convex f, g */
                if (!(P->a2[e] >= 0.0)) {
                    snprintf(msg, msglen, "nonconvex cost at (%d,%ld,%ld)", i, j, k);
                    return ORC_INVALID;
                }
                if (!(P->b2[e] >= 0.0)) {
                    snprintf(msg, msglen, "nonconvex loss at (%d,%ld,%ld)", i, j, k);
                    return ORC_INVALID;
                }
            }
    for (int i = 0; i < m; ++i)
        for (long k = 0; k < n; ++k)
            if (!(P->lo[IK(i, k)] <= P->hi[IK(i, k)])) {
                snprintf(msg, msglen, "inverted bounds at (%d,%ld)", i, k);
                return ORC_INVALID;
            }
    if (msglen > 0) msg[0] = 0;
    return ORC_OK;
}

static void reduce(orc_reduce_fn fn, void *user, double *buf, int len, int op)
{
    if (fn) fn(buf, len, op, user);
}

/* Initialisation (paper silent -> reading G19 = SPEC.md:318):
   x = clamp(midpoint(lo, hi)) (clamp(0) if a bound is infinite); z = g(x);
   lam = 0; s = max(0, sum_i x - y); mu = 0; h = min(c, 1'z); p = 0;
   x1 = mean_j x_1^{(i,j)}; nu = 0; rho = rho0. */
void orc_init(const orc_problem *P, orc_state *S, const orc_params *prm,
              orc_reduce_fn rfn, void *user)
{
    int m = P->m;
    long n = P->n, q = P->q;
    for (int i = 0; i < m; ++i)
        for (long j = 0; j < q; ++j)
            for (long k = 0; k < n; ++k) {
                long e = IX(i, j, k);
                double lo = P->lo[IK(i, k)], hi = P->hi[IK(i, k)];
                double mid = (isfinite(lo) && isfinite(hi)) ? 0.5 * (lo + hi) : 0.0;
                S->x[e] = clampd(mid, lo, hi);
                S->z[e] = gfun(P, e, S->x[e]);
                S->lam[e] = 0.0;
            }
    for (long j = 0; j < q; ++j)
        for (long k = 0; k < n; ++k) {
            double sx = 0.0;
            for (int i = 0; i < m; ++i) sx += S->x[IX(i, j, k)];
            S->s[JK(j, k)] = fmax(0.0, sx - P->y[JK(j, k)]);
            S->mu[JK(j, k)] = 0.0;
        }
    const int hz = P->n_total > 0;       /* horizon-sharded */
    const int own_k1 = !hz || P->k_off == 0; /* this process holds the k = 1 cell */
    double *rs = (double *)calloc((size_t)m * q, sizeof(double));
    for (int i = 0; i < m; ++i)
        for (long j = 0; j < q; ++j) {
            nsum a = {0, 0};
            for (long k = 0; k < n; ++k) nsum_add(&a, S->z[IX(i, j, k)]);
            rs[IJ(i, j)] = nsum_val(&a);
        }
    if (hz) reduce(rfn, user, rs, (int)(m * q), 0); /* 1'z over the horizon blocks */
    for (int i = 0; i < m; ++i)
        for (long j = 0; j < q; ++j) {
            S->h[IJ(i, j)] = fmin(P->c[i], rs[IJ(i, j)]);
            S->p[IJ(i, j)] = 0.0;
            S->nu[IJ(i, j)] = 0.0;
        }
    free(rs);
    double *buf = (double *)calloc((size_t)m, sizeof(double));
    for (int i = 0; i < m; ++i) {
        nsum a = {0, 0};
        if (own_k1)
            for (long j = 0; j < q; ++j) nsum_add(&a, S->x[IX(i, j, 0)]);
        buf[i] = nsum_val(&a);
    }
    reduce(rfn, user, buf, m, 0);
    for (int i = 0; i < m; ++i) S->x1[i] = buf[i] / (double)P->q_total;
    free(buf);
    for (int l = 0; l < 4; ++l) S->rho[l] = prm->rho0[l];
    S->iter = 0;
}

double orc_objective(const orc_problem *P, const double *x, orc_reduce_fn rfn, void *user)
{
    /* (1/q) sum_{i,j,k} f(x), Eq. (2) objective, reading G20 */
    int m = P->m;
    long n = P->n, q = P->q;
    nsum a = {0, 0};
    for (int i = 0; i < m; ++i)
        for (long j = 0; j < q; ++j)
            for (long k = 0; k < n; ++k) {
                long e = IX(i, j, k);
                nsum_add(&a, ffun(P, e, x[e]));
            }
    double v = nsum_val(&a);
    reduce(rfn, user, &v, 1, 0);
    return v / (double)P->q_total;
}

int orc_run(const orc_problem *P, orc_state *S, const orc_params *prm, long iters,
            int stop_on_converge, orc_info *info, double *hist, long hist_cap,
            orc_reduce_fn rfn, void *user)
{
    int m = P->m;
    long n = P->n, q = P->q;
    double qd = (double)P->q_total;
    size_t NE = (size_t)m * q * n, NC = (size_t)q * n, NR = (size_t)m * q;
    double *zt = (double *)malloc(NE * sizeof(double));  /* z~ */
    double *xt = (double *)malloc(NE * sizeof(double));  /* x~ */
    double *st = (double *)malloc(NC * sizeof(double));  /* s~ */
    double *ht = (double *)malloc(NR * sizeof(double));  /* h~ */
    double *W = (double *)malloc(NR * sizeof(double));
    double *sz = (double *)malloc(NR * sizeof(double));  /* 1'z */
    double *buf = (double *)malloc((size_t)(m + 8) * sizeof(double));
    const int hz = P->n_total > 0;                 /* horizon-sharded */
    const int own_k1 = !hz || P->k_off == 0;       /* this process holds the k = 1 cell */
    const double nd = hz ? (double)P->n_total : (double)n; /* horizon length in (6b) */
    int status = ORC_NOT_CONVERGED;
    long ties = 0, rows = 0, done = 0;
    double r = NAN, sigma = NAN;

    for (long it = 0; it < iters; ++it) {
        const double *rho = S->rho;
        /* tilde = value at the start of the current iteration (reading G13) */
        memcpy(zt, S->z, NE * sizeof(double));
        memcpy(xt, S->x, NE * sizeof(double));
        memcpy(st, S->s, NC * sizeof(double));
        memcpy(ht, S->h, NR * sizeof(double));

        /* (6a) PAPER.md:423-429 in the theta/phi form :452-463.  "For each i
           ... in parallel for k and j": sources in order, with
           the latest values of the other sources (Gauss-Seidel, reading G2).
           theta uses lambda^{(i,j)}_k (erratum E5). */
        for (int i = 0; i < m; ++i)
#pragma omp parallel for reduction(+ : ties) schedule(static)
            for (long j = 0; j < q; ++j)
                for (long k = 0; k < n; ++k) {
                    long e = IX(i, j, k);
                    double theta = S->z[e] + S->lam[e];
                    double others = 0.0;
                    for (int l = 0; l < m; ++l)
                        if (l != i) others += S->x[IX(l, j, k)];
                    double phi = S->s[JK(j, k)] - others + P->y[JK(j, k)] + S->mu[JK(j, k)];
                    double cf[4];
                    orc_build_quartic(P->a2[e], P->a1[e], P->b2[e], P->b1[e], P->b0[e], theta,
                                      phi, qd, rho, own_k1 && k == 0, S->x1[i], S->nu[IJ(i, j)], cf);
                    int tie = 0;
                    S->x[e] = orc_quartic_boxmin(cf[0], cf[1], cf[2], cf[3], P->lo[IK(i, k)],
                                                 P->hi[IK(i, k)], prm->box_mode, &tie);
                    ties += tie;
                }

        /* (6b) PAPER.md:431-434: z = w + rho2/(rho1 + n rho2) 1 (h + p - 1'w),
           w = g(x) - lambda */
        double kap = rho[1] / (rho[0] + nd * rho[1]);
#pragma omp parallel for collapse(2) schedule(static)
        for (int i = 0; i < m; ++i)
            for (long j = 0; j < q; ++j) {
                nsum a = {0, 0};
                for (long k = 0; k < n; ++k) {
                    long e = IX(i, j, k);
                    nsum_add(&a, gfun(P, e, S->x[e]) - S->lam[e]);
                }
                W[IJ(i, j)] = nsum_val(&a);
            }
        if (hz) reduce(rfn, user, W, (int)NR, 0); /* 1'w over the horizon blocks */
#pragma omp parallel for collapse(2) schedule(static)
        for (int i = 0; i < m; ++i)
            for (long j = 0; j < q; ++j) {
                double corr = kap * (S->h[IJ(i, j)] + S->p[IJ(i, j)] - W[IJ(i, j)]);
                for (long k = 0; k < n; ++k) {
                    long e = IX(i, j, k);
                    S->z[e] = gfun(P, e, S->x[e]) - S->lam[e] + corr;
                }
            }

        /* (6c) PAPER.md:436 with the mean (erratum E4 / reading G1):
           x1^{(i)} = (1/q) sum_j (x_1^{(i,j)} - nu^{(i,j)}).  nu is the value
           before (6h).  The sum over j crosses shards: rfn (sum). */
        for (int i = 0; i < m; ++i) {
            nsum a = {0, 0};
            if (own_k1)
                for (long j = 0; j < q; ++j) nsum_add(&a, S->x[IX(i, j, 0)] - S->nu[IJ(i, j)]);
            buf[i] = nsum_val(&a);
        }
        reduce(rfn, user, buf, m, 0);
        for (int i = 0; i < m; ++i) S->x1[i] = buf[i] / qd;

        /* (6d) PAPER.md:438: h = min(c, 1'z - p) */
#pragma omp parallel for collapse(2) schedule(static)
        for (int i = 0; i < m; ++i)
            for (long j = 0; j < q; ++j) {
                nsum a = {0, 0};
                for (long k = 0; k < n; ++k) nsum_add(&a, S->z[IX(i, j, k)]);
                sz[IJ(i, j)] = nsum_val(&a);
            }
        if (hz) reduce(rfn, user, sz, (int)NR, 0); /* 1'z over the horizon blocks */
        for (int i = 0; i < m; ++i)
            for (long j = 0; j < q; ++j)
                S->h[IJ(i, j)] = fmin(P->c[i], sz[IJ(i, j)] - S->p[IJ(i, j)]);

        /* (6e) PAPER.md:440: s = max(0, sum_i x - y - mu);
           (6f) PAPER.md:442: mu = mu + s - sum_i x + y */
#pragma omp parallel for schedule(static)
        for (long j = 0; j < q; ++j)
            for (long k = 0; k < n; ++k) {
                double sx = 0.0;
                for (int i = 0; i < m; ++i) sx += S->x[IX(i, j, k)];
                long c = JK(j, k);
                S->s[c] = fmax(0.0, sx - P->y[c] - S->mu[c]);
            }
#pragma omp parallel for schedule(static)
        for (long j = 0; j < q; ++j)
            for (long k = 0; k < n; ++k) {
                double sx = 0.0;
                for (int i = 0; i < m; ++i) sx += S->x[IX(i, j, k)];
                long c = JK(j, k);
                S->mu[c] = S->mu[c] + S->s[c] - sx + P->y[c];
            }
        /* (6g) PAPER.md:444: lambda = lambda + z - g(x) */
#pragma omp parallel for schedule(static)
        for (size_t e = 0; e < NE; ++e) S->lam[e] = S->lam[e] + S->z[e] - gfun(P, (long)e, S->x[e]);
        /* (6h) PAPER.md:446: nu = nu + x1 - x_1^{(i,j)} */
        if (own_k1)
            for (int i = 0; i < m; ++i)
                for (long j = 0; j < q; ++j)
                    S->nu[IJ(i, j)] = S->nu[IJ(i, j)] + S->x1[i] - S->x[IX(i, j, 0)];
        /* (6i) PAPER.md:448: p = p + h - 1'z (1'z after (6b)) */
        for (int i = 0; i < m; ++i)
            for (long j = 0; j < q; ++j)
                S->p[IJ(i, j)] = S->p[IJ(i, j)] + S->h[IJ(i, j)] - sz[IJ(i, j)];

        S->iter += 1;
        done += 1;

        /* residual check every check_every iterations */
        if (prm->check_every > 0 && S->iter % prm->check_every == 0) {
            double t[7] = {0, 0, 0, 0, 0, 0, 0};
            double t0 = 0.0, t1 = 0.0, t4 = 0.0, t6 = 0.0;
            /* r, erratum E6 / reading G14: max over all indices */
#pragma omp parallel for reduction(max : t0, t6) schedule(static)
            for (long j = 0; j < q; ++j)
                for (long k = 0; k < n; ++k) {
                    double sx = 0.0, dx = 0.0;
                    for (int i = 0; i < m; ++i) {
                        sx += S->x[IX(i, j, k)];
                        dx += S->x[IX(i, j, k)] - xt[IX(i, j, k)];
                    }
                    long c = JK(j, k);
                    t0 = fmax(t0, fabs(S->s[c] - sx + P->y[c]));
                    /* sigma 3rd term: ||(s - s~) - sum_i (x - x~)|| */
                    t6 = fmax(t6, fabs((S->s[c] - st[c]) - dx));
                }
#pragma omp parallel for reduction(max : t1, t4) schedule(static)
            for (size_t e = 0; e < NE; ++e) {
                t1 = fmax(t1, fabs(S->z[e] - gfun(P, (long)e, S->x[e])));
                t4 = fmax(t4, fabs(S->z[e] - zt[e]));
            }
            t[0] = t0;
            t[1] = t1;
            t[4] = t4;
            t[6] = t6;
            for (int i = 0; i < m; ++i)
                for (long j = 0; j < q; ++j) {
                    t[2] = fmax(t[2], fabs(S->h[IJ(i, j)] - sz[IJ(i, j)]));
                    if (own_k1) t[3] = fmax(t[3], fabs(S->x[IX(i, j, 0)] - S->x1[i]));
                    t[5] = fmax(t[5], fabs(S->h[IJ(i, j)] - ht[IJ(i, j)]));
                }
            reduce(rfn, user, t, 7, 1);
            /* sigma with the rho of this iteration */
            double s1 = rho[0] * t[4], s2 = rho[1] * t[5], s3 = rho[2] * t[6];
            r = fmax(fmax(t[0], t[1]), fmax(t[2], t[3]));
            sigma = fmax(s1, fmax(s2, s3));
            int conv = (r < prm->r_bar) && (sigma < prm->sigma_bar);
            double fac = 1.0;
            double rho_used[4] = {rho[0], rho[1], rho[2], rho[3]};
            if (!conv && prm->adapt_rho) {
                /* PAPER.md:318-324; reading G12 for sigma = 0 */
                double thr_hi = prm->hi_ratio * prm->r_bar / prm->sigma_bar;
                double thr_lo = prm->lo_ratio * prm->r_bar / prm->sigma_bar;
                double ratio = (sigma > 0.0) ? r / sigma : INFINITY;
                int dir = 0;
                if (ratio > thr_hi) dir = 1;
                else if (ratio < thr_lo) dir = -1;
                if (dir != 0) {
                    double old[4];
                    for (int l = 0; l < 4; ++l) {
                        old[l] = S->rho[l];
                        S->rho[l] = dir > 0 ? S->rho[l] * prm->tau : S->rho[l] / prm->tau;
                    }
                    fac = dir > 0 ? prm->tau : 1.0 / prm->tau;
                    if (prm->rescale_duals) {
                        /* scaled duals follow their penalty (reading G11):
                           lambda<->rho1, p<->rho2, mu<->rho3, nu<->rho4 */
                        double f1 = old[0] / S->rho[0], f2 = old[1] / S->rho[1];
                        double f3 = old[2] / S->rho[2], f4 = old[3] / S->rho[3];
                        for (size_t e = 0; e < NE; ++e) S->lam[e] *= f1;
                        for (size_t e = 0; e < NR; ++e) S->p[e] *= f2;
                        for (size_t e = 0; e < NC; ++e) S->mu[e] *= f3;
                        for (size_t e = 0; e < NR; ++e) S->nu[e] *= f4;
                    }
                }
            }
            if (hist && rows < hist_cap) {
                double *h = hist + rows * ORC_HIST_COLS;
                h[0] = (double)S->iter;
                h[1] = r;
                h[2] = sigma;
                for (int l = 0; l < 4; ++l) h[3 + l] = rho_used[l];
                for (int l = 0; l < 4; ++l) h[7 + l] = t[l];
                h[11] = s1;
                h[12] = s2;
                h[13] = s3;
                h[14] = conv;
                h[15] = fac;
            }
            rows++;
            if (conv) {
                status = ORC_OK;
                if (stop_on_converge) break;
            } else {
                status = ORC_NOT_CONVERGED;
            }
        }
    }
    if (info) {
        info->iterations = done;
        info->r = r;
        info->sigma = sigma;
        info->objective = orc_objective(P, S->x, rfn, user);
        for (int l = 0; l < 4; ++l) info->rho[l] = S->rho[l];
        info->status = status;
        info->ties = ties;
        info->hist_rows = rows;
    }
    free(zt);
    free(xt);
    free(st);
    free(ht);
    free(W);
    free(sz);
    free(buf);
    return status;
}
