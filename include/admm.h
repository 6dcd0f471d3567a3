/*
 * admm.h -- C ABI of libadmm_b200.so: the per-iteration ADMM hot path of
 * arXiv 1903.10041 (Appendix A, Eq. (5)-(6); §III-B Algorithm 1) on
 * NVIDIA B200 (sm_100a), fp64.
 *
 * Problem (Eq. (2)), with Assumption 3 quadratics
 * (PAPER.md:93-101):
 *   min_{x1, x}  (1/q) sum_{i,j,k} f_k^{(i,j)}(x_k^{(i,j)})
 *   s.t. sum_i x_k^{(i,j)} >= y_k^{(j)},   sum_k g_k^{(i,j)}(x_k^{(i,j)}) <= c^{(i)},
 *        x_1^{(i,j)} = x1^{(i)},           lo_k^{(i)} <= x_k^{(i,j)} <= hi_k^{(i)}
 *   f = a2 x^2 + a1 x + a0,  g = b2 x^2 + b1 x + b0   (a2, b2 >= 0: Assumption 1)
 * solved by the ADMM iteration (6a)-(6i) with residuals
 * r, sigma, termination checked every check_every
 * iterations and adaptive rho.
 * Readings of the paper where it is silent or garbled: DESIGN.md §Readings.
 *
 * Indices: i = source (m), j = scenario (q), k = step (n).  0-based; k = 0 is
 * the paper's k = 1 (the consensus step).
 *
 * Layouts of caller arrays (row-major, k fastest, no padding):
 *   f, g coefficient blocks : [3][m][q][n] doubles  (f: a2,a1,a0; g: b2,b1,b0)
 *   x, z, lam               : [m][q][n]
 *   lo, hi                  : [m][n]      (shared by all scenarios)
 *   y, s, mu                : [q][n]
 *   h, p, nu                : [m][q]
 *   c, x1                   : [m]         (c = +INFINITY: no capacity constraint)
 * Under scenario sharding "q" in these layouts is the LOCAL count q_local.
 *
 * Ownership: every input is copied during the call (the caller may free it on
 * return); outputs are caller-allocated.  The context owns all device state,
 * inside a caller-provided device workspace (e.g. a torch tensor) or, when
 * workspace == NULL, memory it allocates itself.  `on_device` = 1 means the
 * pointer arguments of that call are device pointers, 0 means host pointers.
 *
 * Errors: every function returns admm_status and never throws across the ABI;
 * admm_last_error(ctx) gives the first violation with its index path, e.g.
 * "nonconvex loss at (i=1,j=3,k=17)".  A CUDA failure returns ADMM_ERR_CUDA.
 *
 * Threading / streams: a context is not thread safe; all work is ordered on
 * the CUDA stream given at create.  Calls that return results to the host
 * synchronise that stream.  Multi-GPU calls are collective: every rank calls
 * iterate/solve/get_solution with the same arguments.
 *
 * Determinism: same inputs, parameters, device model and world size give
 * bitwise-identical results (fixed-order reductions, no fp atomics on sums).
 */
#ifndef ADMM_B200_H
#define ADMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct admm_ctx admm_ctx; /* opaque */

typedef enum {
    ADMM_OK = 0,
    ADMM_ERR_INVALID = 1,     /* bad argument / problem data (Assumption 1, bounds, NaN) */
    ADMM_NOT_CONVERGED = 2,   /* admm_solve hit max_iter (SPEC.md:505 exit code 2) */
    ADMM_ERR_NONCONVEX = 3,   /* a2 < 0 or b2 < 0 (Assumption 1) */
    ADMM_ERR_NUMERICAL = 4,   /* NaN / Inf in r or sigma */
    ADMM_ERR_CUDA = 5,
    ADMM_ERR_NCCL = 6,
    ADMM_ERR_STATE = 7        /* call-order misuse, or a state that is not representable */
} admm_status;

typedef enum {
    ADMM_BOX_PROJECT = 0, /* x <- Pi_box(argmin_R J): Eq. (6a) as printed */
    ADMM_BOX_EXACT = 1    /* x <- argmin_box J: block minimiser of L */
} admm_box_mode;

typedef enum {
    ADMM_EXEC_AUTO = 0,       /* persistent when the state fits on chip, else streaming */
    ADMM_EXEC_STREAMING = 1,  /* one fused sweep kernel per iteration, CUDA-graph while loop */
    ADMM_EXEC_PERSISTENT = 2  /* one kernel per call, state in shared memory (cluster-row
                                 engine, else grid-barrier engine); ADMM_ERR_INVALID if the
                                 problem does not fit on chip */
} admm_exec_mode;

/* Engine that ran the last admm_iterate / admm_solve (admm_get_engine). */
typedef enum {
    ADMM_ENGINE_NONE = 0,
    ADMM_ENGINE_STREAM = 1,      /* sweep_kernel: one launch per iteration (graph while loop) */
    ADMM_ENGINE_GRID = 2,        /* persist_kernel: one cooperative launch per call */
    ADMM_ENGINE_CLUSTER = 3,     /* persist_cluster_kernel: one cluster launch per call (barrier protocol, ADMM_CLUSTER_V=1) */
    ADMM_ENGINE_STREAM_TMA = 4,  /* sweep2_kernel: TMA-fed streaming sweep, one launch per iteration (default for finite boxes) */
    ADMM_ENGINE_CLUSTER_MSG = 5  /* persist_cluster2_kernel: one cluster launch per call, message-passing protocol
                                    (default on-chip engine: PHEV-sized problems) */
} admm_engine;

/* Multi-GPU partition (one process per GPU; the method is
   "parallel for k and j").  nccl_id comes from admm_nccl_unique_id
   on rank 0, broadcast by the caller (torch.distributed).  A non-NULL admm_dist
   always runs the collective path, also at world = 1 (a one-rank communicator:
   the same graph, exchanges and finalisation as world > 1).
   mode = ADMM_SHARD_SCENARIOS: rank r owns the scenarios j in [j_begin, j_end) of
     q_total and every step; per iteration the ranks all-gather 32 doubles
     (consensus sums of (6c), residual maxima).  k_begin / k_end are ignored.
   mode = ADMM_SHARD_HORIZON: rank r owns the steps k in [k_begin, k_end) of the
     n-step horizon and every scenario (j_begin = 0, j_end = q_total); the
     per-row sums over k of (6b)/(6d) (exact 64-bit fixed point, m q values)
     and their dg extrema are all-reduced every iteration, every rank finalises
     every row identically, and the rank with k_begin = 0 owns the consensus
     cell k = 1 (horizon length must not grow the time per
     iteration).  Needs finite boxes; the problem arrays passed to
     admm_set_problem are the rank's [k_begin, k_end) slices. */
typedef enum { ADMM_SHARD_SCENARIOS = 0, ADMM_SHARD_HORIZON = 1 } admm_shard_mode;
typedef struct {
    int32_t rank, world;
    int64_t j_begin, j_end;
    unsigned char nccl_id[128];
    int64_t k_begin, k_end;  /* ADMM_SHARD_HORIZON only */
    int32_t mode;            /* admm_shard_mode */
    int32_t reserved;
} admm_dist;

/* Parameters; admm_default_params() fills the paper's values (PAPER.md:317-324,
   :353): rho = (1e-4, 2e-6, 5e-6, 5e-6), tau = 1.1, band 1.2 / 0.8,
   sigma_bar = 1e-2, check_every = 10, adapt on, dual rescale on, PROJECT,
   exec_mode AUTO. */
typedef struct {
    double rho[4];          /* rho1..rho4 used from the next iteration on */
    double tau, hi_ratio, lo_ratio;
    double r_bar, sigma_bar;
    int32_t check_every;    /* residual check period (>= 1) */
    int32_t adapt_rho;      /* adapt rho at each check */
    int32_t rescale_duals;  /* scaled duals *= rho_old/rho_new on adaptation (reading G11) */
    int32_t box_mode;       /* admm_box_mode */
    int32_t exec_mode;      /* admm_exec_mode (execution engine; results agree to rounding) */
} admm_params;

typedef struct {
    int64_t iterations;     /* total iterations done on this context */
    double r, sigma;        /* residuals at the last check (NaN before the first) */
    double objective;       /* (1/q) sum f(x) incl. a0 (filled by get_solution / solve) */
    double rho[4];          /* current rho */
    int32_t status;         /* ADMM_OK if the last check met r < r_bar and sigma < sigma_bar */
    int32_t checks;         /* residual checks done */
} admm_info;

/* One history row per residual check (admm_get_history). */
#define ADMM_HIST_COLS 16
/* iter, r, sigma, rho1..rho4 (of that iteration), r1..r4, sigma1..sigma3,
   converged flag, factor applied to rho after the check (tau, 1/tau or 1). */

void admm_default_params(admm_params* out);

/* Device workspace needed for a context (bytes).  device = CUDA ordinal. */
size_t admm_workspace_bytes(int32_t m, int64_t n, int64_t q_local, int32_t device);

/* NCCL unique id for a multi-GPU context (call on rank 0 only). */
admm_status admm_nccl_unique_id(unsigned char out[128]);

/* Create a context for m sources, n steps, q_total scenarios of the robust
   problem Eq. (2) (variables and multipliers of its ADMM form
   Eq. (5)).  dist = NULL: single GPU, all scenarios local.
   Errors: ADMM_ERR_INVALID for m not in 1..4, n or q_total <= 0, a bad shard;
   ADMM_ERR_CUDA / ADMM_ERR_NCCL if the device or communicator cannot be set
   up (*ctx is then NULL).  The caller owns the workspace; the context owns
   everything it creates and frees it in admm_destroy.  workspace: device buffer of at least
   admm_workspace_bytes bytes (NULL: the library allocates).  cuda_stream:
   cudaStream_t to order all work on (NULL = the legacy default stream). */
admm_status admm_create(admm_ctx** ctx, int32_t m, int64_t n, int64_t q_total,
                        const admm_dist* dist, int32_t device, void* workspace,
                        size_t workspace_bytes, void* cuda_stream);

/* Problem data (Eq. (2) + Assumption 3).  f = [3][m][q_local][n] (a2,a1,a0),
   g = [3][m][q_local][n] (b2,b1,b0), lo/hi = [m][n], y = [q_local][n], c = [m].
   Validates (ADMM_ERR_NONCONVEX for a2 or b2 < 0, ADMM_ERR_INVALID for lo > hi,
   NaN, or non-finite coefficients / y) and then initialises the state
   (reading G19): x = clamp(midpoint(lo,hi)) (clamp(0) if a bound
   is infinite), z = g(x), lam = 0, s = max(0, sum_i x - y), mu = 0,
   h = min(c, 1'z), p = 0, x1 = mean_j x_1^{(i,j)}, nu = 0, rho = params.rho. */
admm_status admm_set_problem(admm_ctx* ctx, const double* f, const double* g, const double* lo,
                             const double* hi, const double* y, const double* c, int32_t on_device);

/* Re-initialise the state from the current problem data exactly as
   admm_set_problem does (reading G19), with rho = params.rho and the
   iteration counter, checks and history cleared.  No host<->device copies of
   problem data. */
admm_status admm_reset(admm_ctx* ctx);

/* Replace the parameters.  rho takes effect on the next iteration. */
admm_status admm_set_params(admm_ctx* ctx, const admm_params* params);
admm_status admm_get_params(const admm_ctx* ctx, admm_params* out);

/* Exactly `iters` ADMM iterations, each the updates (6a)-(6i) of PAPER.md:421-450
   in printed order (readings G1-G21): the per-element quartic of
   (6a) minimised in closed form by Algorithm 1 and boxed,
   the capacity sums (6b)/(6d)/(6g)/(6i), the consensus (6c)/(6h), the demand
   slack (6e)/(6f).  At every multiple of check_every (counted over the
   context's lifetime) the residuals r and sigma are
   evaluated and rho adapted by the 1.2 / 0.8 band rule (PAPER.md:318-324,
   checked every 10 iterations :353); never stops early.  Asynchronous with
   respect to the host only up to one device->host read of the iteration
   counter at the end of the call.  ADMM_ERR_STATE before admm_set_problem,
   ADMM_ERR_NUMERICAL if a check saw NaN/Inf (the state then stops changing). */
admm_status admm_iterate(admm_ctx* ctx, int64_t iters);

/* Iterate as admm_iterate until a check finds r < r_bar and sigma < sigma_bar
   (the termination rule of PAPER.md:353, :464-479; thresholds r_bar = 1e-6 dE,
   sigma_bar = 1e-2 in the paper's experiments) -> ADMM_OK, or
   max_iter more iterations are done -> ADMM_NOT_CONVERGED.  The whole loop
   runs on the device (CUDA-graph WHILE node; no host round trip per
   iteration).  info may be NULL. */
admm_status admm_solve(admm_ctx* ctx, double r_bar, double sigma_bar, int64_t max_iter,
                       admm_info* info);

/* Solution of the ADMM iterate: x = x_k^{(i,j)} [m][q_local][n] (row-major,
   k fastest) and the consensus first move x1^{(i)} [m] of (6c) (PAPER.md:436,
   mean reading G1), either may be NULL; info (may be NULL) with the objective
   (1/q) sum_{i,j,k} f(x) of Eq. (2) (reading G20).  Outputs are
   caller-allocated; on_device = 1 for device pointers.  Synchronous. */
admm_status admm_get_solution(admm_ctx* ctx, double* x, double* x1, admm_info* info,
                              int32_t on_device);

/* Literal state arrays, materialised from the
   reduced device representation.  Any pointer
   may be NULL. */
admm_status admm_get_state(admm_ctx* ctx, double* x, double* z, double* lam, double* s,
                           double* mu, double* h, double* p, double* nu, double* x1,
                           int32_t on_device);

/* Warm start (Algorithm 2 re-solves).  All pointers
   required.  The state must be representable: lam constant over k and
   z - g(x) constant over k per (i,j) (identity I1), and s * mu = 0 (I2), to a
   relative 1e-12; otherwise ADMM_ERR_STATE. */
admm_status admm_set_state(admm_ctx* ctx, const double* x, const double* z, const double* lam,
                           const double* s, const double* mu, const double* h, const double* p,
                           const double* nu, const double* x1, int32_t on_device);

/* Residual-check history (host buffer of rows x ADMM_HIST_COLS doubles); returns
   the number of rows written (the most recent rows if more were recorded). */
int64_t admm_get_history(admm_ctx* ctx, double* out, int64_t max_rows);

/* Average device time (ms) of each kernel class over the last solve/iterate
   call, measured with CUDA events; out[0] = sweep kernel, out[1] = whole call. */
admm_status admm_get_timing(admm_ctx* ctx, double out[2]);

/* Engine of the last iterate/solve call (admm_engine) and the number of CUDA
   kernels this context has launched since admm_create (cumulative; resets,
   sweeps, graph condition kernels, objective).  Either pointer may be NULL.
   ADMM_ERR_INVALID on a NULL context. */
admm_status admm_get_engine(const admm_ctx* ctx, int32_t* engine, int64_t* launches);

/* F2 mixed precision (the paper ran in fp32).
   Storage precision of the per-element cost coefficients a2, a1 (f) and b2, b1 (g)
   that admm_set_problem applies: bits = 64 (default: stored as given) or 32 (each
   is rounded to the nearest fp32 value; the streaming sweep then reads 16 instead
   of 32 bytes of coefficients per element).  Every operation and every state
   array stays fp64, and every engine solves the same problem -- the one whose
   a2, a1, b2, b1 are the rounded inputs (a0, b0, bounds, demand, c unchanged);
   admm_get_state/objective refer to that problem.  Changing the precision
   discards the loaded problem (call admm_set_problem again; iterate/solve
   return ADMM_ERR_STATE until then).  ADMM_ERR_INVALID for bits not in {32, 64}
   or a NULL context. */
admm_status admm_set_coeff_precision(admm_ctx* ctx, int32_t bits);
admm_status admm_get_coeff_precision(const admm_ctx* ctx, int32_t* bits);

const char* admm_last_error(const admm_ctx* ctx);
void admm_destroy(admm_ctx* ctx);

/* Algorithm 1 of PAPER.md:170-198 (closed-form minimiser of a quartic through the
   roots of its derivative cubic: Cardano / trigonometric / Vieta branches,
   PAPER.md:129-165, with the stable forms G4-G9 of DESIGN.md §3) on a batch:
   x[e] = the minimiser of A x^4 + B x^3 + C x^2 + D x, then the box step of
   (6a) (box_mode PROJECT = clamp of the global minimiser,
   EXACT = minimiser over [lo[e], hi[e]], reading G3).  A >= 0 (A = 0: the
   convex quadratic).  All arrays are DEVICE pointers of length N (caller
   owned); lo/hi may be NULL (unbounded).  Asynchronous on cuda_stream (a 4-byte
   stream-ordered allocation per call from a library-owned memory pool): one CTA
   classifies a strided sample of 4096 quartics and picks, on the device, the
   one-quartic-per-lane kernel (one branch dominates) or the warp-compacted one
   (both common: trigonometric-branch quartics are queued per warp so each branch
   runs with all lanes); results are bit-identical either way.
   ADMM_ERR_INVALID for N < 0, NULL A..D / x or a bad box_mode. */
admm_status quartic_minimize_batch(const double* A, const double* B, const double* C,
                                   const double* D, const double* lo, const double* hi,
                                   double* x, int64_t N, int32_t box_mode, void* cuda_stream);

/* Library version / build info string. */
const char* admm_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* ADMM_B200_H */
