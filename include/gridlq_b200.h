/*
 * gridlq_b200 -- C ABI of the B200-native PCGM hot path (arXiv 2304.04980).
 *
 * Drop-in boundary for the reference package `gridlq` (Python, /root/reference/pkg/src).
 * The reference has no FFI of its own: its hot path is the duck-typed operator /
 * preconditioner protocol consumed by `pcg_solve`.  Each entry point below replaces one
 * member of that protocol (reference file:line in brackets):
 *
 *   gq_create            build_stacked + build_schur + NestedJacobiPreconditioner.__init__
 *                        (factor_all)          [kkt_assembly.py:204,487,695; nested_jacobi.py:31-43]
 *   gq_apply_delta       SchurOperator.apply / apply_delta        [kkt_assembly.py:389-403,547]
 *   gq_apply_outer_coupling  SchurOperator.apply_outer_coupling   [kkt_assembly.py:414-425]
 *   gq_apply_inner_coupling  PairSplitting.apply_inner_coupling   [kkt_assembly.py:645-662]
 *   gq_pair_solve        NestedJacobiPreconditioner._pair_solves  [nested_jacobi.py:65-77]
 *   gq_apply_precond     NestedJacobiPreconditioner.apply         [nested_jacobi.py:105-122]
 *   gq_nbjm_solve        NestedJacobiPreconditioner.solve / nbjm_solve
 *                                                                 [nested_jacobi.py:124-159]
 *   gq_pcg_start / gq_pcg_run / gq_pcg_read / gq_pcg_history / gq_pcg
 *                        pcg_solve / cg_solve                     [pcg.py:50-156]
 *
 * Conventions
 *   - Vectors are fp64 in the reference's global order (t, j, i, k): element
 *     t*K*N*n + (j*K + i)*n + k  [grid_problem.py:143-144].  Vector pointers may be host
 *     (pageable or pinned) or device pointers; the library detects which.
 *   - Problem arrays in gq_problem_desc are HOST pointers, copied at gq_create.
 *   - All functions return a gq_status; gq_last_error() gives the message of the most
 *     recent failure on the calling thread.
 *   - A context is not thread-safe; one solve at a time per context.
 */
#ifndef GRIDLQ_B200_H
#define GRIDLQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gq_status {
  GQ_OK = 0,
  GQ_MAX_ITER = 1,        /* MaxIterationsExceeded        [pcg.py:141-148]  */
  GQ_BREAKDOWN = 2,       /* BreakdownError               [pcg.py:103-107]  */
  GQ_DIM_MISMATCH = 3,    /* DimensionMismatchError       [pcg.py:63-64]    */
  GQ_INVALID_ARG = 4,     /* ValueError (odd L, tol<=0, non-finite rhs, ...) */
  GQ_NOT_SPD = 5,         /* NotPositiveDefiniteError     [block_linalg.py:54-60] */
  GQ_CUDA_ERROR = 6,
  GQ_UNSUPPORTED = 7      /* e.g. state dimension without a compiled kernel */
} gq_status;

enum { GQ_VEC_X = 0, GQ_VEC_R = 1 };

/* Dense, stage-class-deduplicated problem description (see GridArrays in problem.py).
 * Node axes are [N][K] (column j, then row i).  Stage t < T uses dynamics set
 * dyn_class[t]; stage t <= T uses state-cost set cost_class[t]. */
typedef struct gq_problem_desc {
  int32_t K, N, T, n, m;
  int32_t n_dyn, n_cost;
  const int32_t* dyn_class;   /* [T]   */
  const int32_t* cost_class;  /* [T+1] */
  const double* A;            /* [n_dyn][N][K][n][n] */
  const double* B;            /* [n_dyn][N][K][n][m] */
  const double* R;            /* [n_dyn][N][K][m][m] */
  const double* C;            /* [n_dyn][4][N][K][n][n]  west, east, north, south */
  const double* Q;            /* [n_cost][N][K][n][n] */
} gq_problem_desc;

typedef struct gq_ctx gq_ctx;

const char* gq_last_error(void);
const char* gq_version(void);

int gq_create(const gq_problem_desc* desc, int32_t inner_sweeps, int32_t outer_sweeps,
              gq_ctx** out);
void gq_destroy(gq_ctx* ctx);
int64_t gq_dim(const gq_ctx* ctx);
int gq_set_stream(gq_ctx* ctx, void* cuda_stream);
int gq_synchronize(gq_ctx* ctx);
/* change the nested-Jacobi budgets L (inner) and S (outer); factors are independent of them */
int gq_set_sweeps(gq_ctx* ctx, int32_t inner_sweeps, int32_t outer_sweeps);

int gq_apply_delta(gq_ctx* ctx, const double* x, double* y);
int gq_apply_outer_coupling(gq_ctx* ctx, const double* x, double* y);
int gq_apply_inner_coupling(gq_ctx* ctx, const double* x, double* y);
int gq_pair_solve(gq_ctx* ctx, const double* rhs, double* out);
int gq_apply_precond(gq_ctx* ctx, const double* r, double* q);

/* Standalone nested block Jacobi solve with the context's inner budget (any L >= 1):
 * outer sweeps, inner sweeps warm-started from the outer iterate, until
 * max|new - prev| < tol [nested_jacobi.py:124-151].  Returns GQ_OK with the solution and
 * the outer sweep count, or GQ_MAX_ITER with the last iterate in x_out and
 * *outers = max_outer.  Resets any PCG solve in progress on the context. */
int gq_nbjm_solve(gq_ctx* ctx, const double* rhs, double tol, int64_t max_outer,
                  double* x_out, int64_t* outers);

/* Stateful PCG: start (r = rhs - Delta x0, d = P r, mu = d.r), then run until convergence
 * (||r||_inf < tol, absolute), breakdown or max_steps total steps. */
int gq_pcg_start(gq_ctx* ctx, const double* rhs, const double* x0, int32_t use_precond);
int gq_pcg_run(gq_ctx* ctx, double tol, int64_t max_steps, int64_t* steps_done,
               int32_t* converged);
int gq_pcg_read(gq_ctx* ctx, int32_t which, double* out);
int gq_pcg_history(gq_ctx* ctx, double* out, int64_t count);
int gq_pcg_scalars(gq_ctx* ctx, double* mu, double* curvature, double* alpha, double* beta);
/* one-shot: start + run + read x + history; returns GQ_OK / GQ_MAX_ITER / GQ_BREAKDOWN */
int gq_pcg(gq_ctx* ctx, const double* rhs, const double* x0, double tol, int64_t max_steps,
           int32_t use_precond, double* x_out, double* hist_out, int64_t hist_capacity,
           int64_t* steps, int32_t* converged);

/* Stage-slab mode (pcg.py:50-149 split at its reductions).
 * The context holds the stage window of one slab: owned stages [own_lo, own_hi) plus at most
 * one halo stage per side (own_lo in {0, 1}, own_hi in {T, T+1} of the window).  A solve is
 *   gq_slab_start(r0 = the slab's initial residual, zero on halo stages; x0 or NULL)
 *   init:  for s < S: INIT_OUTER(s) [exchange DL(s%2) if s < S-1]; reduce MU (sum); INIT_FINISH
 *   step:  exchange D; DELTA; reduce CURV (sum); UPDATE;
 *          for s < S: OUTER(s) [exchange DL(s%2) if s < S-1];
 *          reduce RES (max) and MU (sum) -- one collective; DIRECTION
 * (the max|r| kernels only record max|r| in stage-slab mode; DIRECTION decides convergence
 * on the global value, so a converged step computes its q = P r for nothing)
 * (CG: S = 1).  "exchange v" = every slab packs its owned boundary stages of v
 * (gq_slab_pack) and unpacks the neighbours' into its halo stages (gq_slab_unpack); a halo
 * buffer holds K*N*n doubles in (column, row, state) order.  "reduce" = combine the device
 * scalar gq_slab_scalar_ptr(ctx, which) over all slabs and write the result back into each.
 * All calls enqueue on the context stream and return without synchronising, except
 * gq_slab_status.  Replaces nothing in the reference (it has no multi-process path). */
enum { GQ_SLAB_INIT_OUTER = 0, GQ_SLAB_INIT_FINISH = 1, GQ_SLAB_DELTA = 2, GQ_SLAB_UPDATE = 3,
       GQ_SLAB_OUTER = 4, GQ_SLAB_DIRECTION = 5 };
enum { GQ_SLAB_VEC_D = 0, GQ_SLAB_VEC_DL0 = 1, GQ_SLAB_VEC_DL1 = 2 };
enum { GQ_SLAB_CURV = 0, GQ_SLAB_RES = 1, GQ_SLAB_MU = 2 };
int gq_slab_enable(gq_ctx* ctx, int32_t own_lo, int32_t own_hi);
int gq_slab_start(gq_ctx* ctx, const double* r0, const double* x0, int32_t use_precond,
                  double tol, int64_t max_steps);
int gq_slab_phase(gq_ctx* ctx, int32_t kind, int32_t outer);
int gq_slab_pack(gq_ctx* ctx, int32_t which, int32_t stage, double* buf);
int gq_slab_unpack(gq_ctx* ctx, int32_t which, int32_t stage, const double* buf);
void* gq_slab_scalar_ptr(gq_ctx* ctx, int32_t which);
int gq_slab_status(gq_ctx* ctx, int64_t* step, int32_t* done, int32_t* converged,
                   int32_t* breakdown);

/* Primal recovery and first-order optimality residuals (recovery.py:50-80).
 *   gq_recover:      x = -Qinv (A~' lam), u = -Rinv (B~' lam), objective 0.5 (x'Qx + u'Ru)
 *                    [recovery.py:50-65; kkt_assembly.py:84-160]
 *   gq_kkt_residual: res3 = {||Qx + A~'lam||_inf, ||Ru + B~'lam||_inf,
 *                            ||A~x + B~u + omega~||_inf}      [recovery.py:68-80]
 * lam, x and omega~ have gq_dim entries in the reference order (t, j, i, k); u has
 * gq_input_dim entries in the order (t, j, i, c) of GridLayout.stage_u_slice. */
int64_t gq_input_dim(const gq_ctx* ctx);
int gq_recover(gq_ctx* ctx, const double* lam, double* x_out, double* u_out, double* objective);
int gq_kkt_residual(gq_ctx* ctx, const double* lam, const double* x, const double* u,
                    const double* offset, double* res3);

/* Reduced right-hand side omega~ built on the device (replaces the offset loop of
 * build_stacked, kkt_assembly.py:275-301): out[stage 0] = init, out[stage t+1] (edge nodes) =
 * sum over the off-grid directions d with a declared trajectory of C_d(t) sigma_d(t), added in
 * the reference's order north, south, west, east.  All pointers are device pointers:
 *   init   [N][K][n]                initial states, node order (j, i) as in the vectors
 *   blocks [4][L][ncls][n][n]       coupling blocks of edge node e of direction d (west,
 *                                   east, north, south; L = max(K, N); e = row i for
 *                                   west/east, column j for north/south), row-major
 *   cls    [4][L][T]  int32         block class of (d, e, t), or -1: no term
 *   traj   [4][L][T][n]             boundary trajectories sigma_d(e, t)
 *   out    [gq_dim]                 omega~ in the reference order (t, j, i, k)
 * No context is needed; `stream` is a cudaStream_t (or null). */
int gq_build_offset(int32_t K, int32_t N, int32_t T, int32_t n, int32_t ncls,
                    const double* init, const double* blocks, const int32_t* cls,
                    const double* traj, double* out, void* stream);

/* Host helper of the solver API (no reference counterpart: numpy's pcg_solve returns a fresh
 * array, pcg.py:83): fault in the pages of a fresh host result buffer from several threads
 * while the device iterates, so the device-to-host copy does not wait for the page faults. */
void gq_touch_pages(void* p, int64_t bytes);

/* Page-locked host memory for result arrays (same place in the API: the array pcg_solve
 * returns, pcg.py:83).  The device-to-host copy of a result lands in it directly at PCIe speed
 * instead of through the staging vector and a host copy; the Python side keeps freed buffers
 * in a small pool, because page-locking 211 MB takes longer than a 100-step solve.
 * gq_host_alloc returns NULL when the allocation fails (callers fall back to pageable memory). */
void* gq_host_alloc(int64_t bytes);
void gq_host_free(void* p);

/* Measurement helpers (bench.py): run `steps` PCG steps as individual launches with CUDA
 * events around every kernel; per-kernel total milliseconds go to ms_out[0..count) in the
 * order gq_kernel_name(ctx, i) reports.  Returns the number of kernels per step. */
int gq_profile_steps(gq_ctx* ctx, int32_t steps, float* ms_out, int32_t count);
const char* gq_kernel_name(gq_ctx* ctx, int32_t i);
/* kernels launched per PCG step (graph nodes) */
int gq_launches_per_step(gq_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* GRIDLQ_B200_H */
