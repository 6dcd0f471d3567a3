/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle for the ADMM hot path
 * of arXiv 1903.10041 (Appendix A, Eq. (6a)-(6i); §III-B Algorithm 1).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load, call or link this
 * library.  The product (paper_1903_10041_b200/, libadmm_b200.so) never does;
 * the two share no code, headers, helpers or constants.
 *
 * Everything is fp64, single thread, literal arrays, in the paper's printed
 * update order.  Readings of the paper where it is silent / garbled are listed
 * in DESIGN.md §"Readings" (G1..G21 of SURVEY.md §8(c)) and cited inline.
 *
 * Layouts (row-major, k fastest):
 *   a2,a1,a0,b2,b1,b0, x,z,lam : [m][q][n]    lo,hi : [m][n]
 *   y, s, mu : [q][n]      h, p, nu : [m][q]      c, x1 : [m]
 */
#ifndef ORACLE_H
#define ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_BOX_PROJECT 0 /* x <- clamp(argmin_R J)  (Eq. (6a) literally) */
#define ORC_BOX_EXACT 1   /* x <- argmin_[lo,hi] J   (block minimiser of L) */

#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_NOT_CONVERGED 2

/* history row layout (doubles), one row per residual check */
#define ORC_HIST_COLS 16
/* iter, r, sigma, rho1..rho4 (values used in this iteration), r1..r4, s1..s3,
   converged flag, rho factor applied after the check (tau, 1/tau or 1) */

typedef struct {
    int m;
    long n, q;       /* q = local scenario count */
    long q_total;    /* total scenario count (the 1/q in Eq. (2) and (6c)); = q unsharded */
    const double *a2, *a1, *a0, *b2, *b1, *b0;
    const double *lo, *hi;
    const double *y;
    const double *c;
    /* horizon-block sharding ("in parallel for k and
       j"): this process holds steps [k_off, k_off + n) of an n_total-step horizon
       and every scenario; the per-row sums over k ((6b) 1'w, (6d) 1'z, the
       initial 1'z) are summed over the processes with the reduce callback, and
       only the process with k_off = 0 owns the k = 1 consensus cell.
       n_total = 0: unsharded horizon (n_total = n, k_off = 0). */
    long n_total, k_off;
} orc_problem;

typedef struct {
    double *x, *z, *lam;
    double *s, *mu;
    double *h, *p, *nu;
    double *x1;
    double rho[4];
    long iter; /* iterations done so far (checks happen when iter % check_every == 0) */
} orc_state;

typedef struct {
    double rho0[4];
    double tau, hi_ratio, lo_ratio;
    double r_bar, sigma_bar;
    int check_every, adapt_rho, rescale_duals, box_mode;
} orc_params;

typedef struct {
    long iterations;
    double r, sigma, objective;
    double rho[4];
    int status;
    long ties;       /* x-updates whose two wells tied within 8 eps (G8) */
    long hist_rows;
} orc_info;

/* op: 0 = sum, 1 = max.  In-place over buf[0..len).  NULL = single process. */
typedef void (*orc_reduce_fn)(double *buf, int len, int op, void *user);

/* Algorithm 1 building blocks */
int orc_cubic_roots(double b, double c, double d, double roots[3], int *branch);
double orc_quartic_argmin(double A, double B, double C, double D, int *tie);
double orc_quartic_boxmin(double A, double B, double C, double D, double lo, double hi,
                          int mode, int *tie);
void orc_quartic_batch(const double *A, const double *B, const double *C, const double *D,
                       const double *lo, const double *hi, double *x, long N, int mode,
                       long *ties);
/* Eq. (6a) quartic J(x) = f/q + rho1/2 (theta - g)^2 + rho3/2 (phi - x)^2
   + delta rho4/2 (x1 - x + nu)^2, expanded. out = {A,B,C,D}. */
void orc_build_quartic(double a2, double a1, double b2, double b1, double b0, double theta,
                       double phi, double qd, const double rho[4], int delta, double x1,
                       double nu, double out[4]);

/* ADMM */
int orc_validate(const orc_problem *P, char *msg, int msglen);
/* OpenMP build only: threads for the parallel loops (returns the count in use;
   the serial build returns 1) */
int orc_set_threads(int n);
void orc_init(const orc_problem *P, orc_state *S, const orc_params *prm,
              orc_reduce_fn reduce, void *user);
int orc_run(const orc_problem *P, orc_state *S, const orc_params *prm, long iters,
            int stop_on_converge, orc_info *info, double *hist, long hist_cap,
            orc_reduce_fn reduce, void *user);
double orc_objective(const orc_problem *P, const double *x, orc_reduce_fn reduce, void *user);

#ifdef __cplusplus
}
#endif
#endif
