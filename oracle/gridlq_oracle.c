/*
 * C restatement of the gridlq PCGM step -- TEST INFRASTRUCTURE ONLY (CPU oracle / CPU
 * baseline).  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs use it.
 *
 * It consumes the operator arrays assembled by oracle/gridlq_oracle.py (Psi/Xi blocks and
 * pair factors, themselves restating build_schur / PairSplitting / block_tridiag_factor)
 * and restates the per-step algorithm of the reference:
 *   orc_delta        SchurOperator.apply                   kkt_assembly.py:379-403
 *   orc_outer        SchurOperator.apply_outer_coupling    kkt_assembly.py:414-425
 *   orc_inner        PairSplitting.apply_inner_coupling    kkt_assembly.py:645-662
 *   orc_pair_solve   BlockTridiagCholesky.solve per chain  block_linalg.py:336-358
 *   orc_precond      NestedJacobiPreconditioner.apply      nested_jacobi.py:79-122
 *   orc_pcg          pcg_solve                             pcg.py:50-149
 * Vectors are in the reference order (t, j, i, k).  OpenMP parallel loops with static
 * schedules; dot products accumulate per-thread partials summed in thread order.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int K, N, T, n, V, nb, q;
  const int* psi_cls;   /* [T+1] */
  const int* xi_cls;    /* [T]   */
  const double* psi;    /* [npc][N][K][13][n][n] */
  const double* xi;     /* [nxc][N][K][5][n][n]  Xi(a, a+u) */
  const double* xit;    /* [nxc][N][K][5][n][n]  Xi(a+u, a)' */
  const double* linv;   /* [npc][nb][V][q][q] */
  const double* sub;    /* [npc][nb][V][q][q] */
} orc_t;

static const int ODI[13] = {0, -1, 1, 0, 0, -2, 2, 0, 0, -1, -1, 1, 1};
static const int ODJ[13] = {0, 0, 0, -1, 1, 0, 0, -2, 2, -1, 1, -1, 1};

static inline long vi(const orc_t* o, int t, int j, int i) {
  return (((long)t * o->N + j) * o->K + i) * o->n;
}

/* acc += M x (n x n row-major) */
static inline void mv_add(int n, const double* M, const double* x, double* acc) {
  for (int a = 0; a < n; ++a) {
    double s = 0.0;
    for (int b = 0; b < n; ++b) s += M[a * n + b] * x[b];
    acc[a] += s;
  }
}

static inline int in_grid(const orc_t* o, int j, int i) {
  return j >= 0 && j < o->N && i >= 0 && i < o->K;
}

/* mode 0: Delta, 1: outer coupling (Xi~), 2: inner coupling (Omega~) */
static void stencil(const orc_t* o, int mode, const double* x, double* y) {
  const int n = o->n, T1 = o->T + 1, B2 = n * n;
  const long nk = (long)o->N * o->K;
#pragma omp parallel for schedule(static)
  for (long tj = 0; tj < (long)T1 * o->N; ++tj) {
    const int t = (int)(tj / o->N), j = (int)(tj % o->N);
    const int pc = o->psi_cls[t];
    double acc[8], e[8];
    for (int i = 0; i < o->K; ++i) {
      const long node = (long)j * o->K + i;
      for (int k = 0; k < n; ++k) acc[k] = 0.0;
      if (mode == 0 || mode == 2) {
        const double* P = o->psi + ((long)pc * nk + node) * 13 * B2;
        for (int s = 0; s < 13; ++s) {
          const int jj = j + ODJ[s], ii = i + ODI[s];
          if (!in_grid(o, jj, ii)) continue;
          if (mode == 2 && ((jj >> 1) == (j >> 1))) continue;   /* same pair: not Omega */
          mv_add(n, P + s * B2, x + vi(o, t, jj, ii), acc);
        }
        if (mode == 2)
          for (int k = 0; k < n; ++k) acc[k] = -acc[k];
      }
      if (mode == 0 || mode == 1) {
        const double sg = (mode == 0) ? 1.0 : -1.0;
        if (t >= 1) {
          const double* X = o->xi + ((long)o->xi_cls[t - 1] * nk + node) * 5 * B2;
          for (int k = 0; k < n; ++k) e[k] = 0.0;
          for (int u = 0; u < 5; ++u) {
            const int jj = j + ODJ[u], ii = i + ODI[u];
            if (in_grid(o, jj, ii)) mv_add(n, X + u * B2, x + vi(o, t - 1, jj, ii), e);
          }
          for (int k = 0; k < n; ++k) acc[k] += sg * e[k];
        }
        if (t < o->T) {
          const double* X = o->xit + ((long)o->xi_cls[t] * nk + node) * 5 * B2;
          for (int k = 0; k < n; ++k) e[k] = 0.0;
          for (int u = 0; u < 5; ++u) {
            const int jj = j + ODJ[u], ii = i + ODI[u];
            if (in_grid(o, jj, ii)) mv_add(n, X + u * B2, x + vi(o, t + 1, jj, ii), e);
          }
          for (int k = 0; k < n; ++k) acc[k] += sg * e[k];
        }
      }
      double* yo = y + vi(o, t, j, i);
      for (int k = 0; k < n; ++k) yo[k] = acc[k];
    }
  }
}

void orc_delta(const orc_t* o, const double* x, double* y) { stencil(o, 0, x, y); }
void orc_outer(const orc_t* o, const double* x, double* y) { stencil(o, 1, x, y); }
void orc_inner(const orc_t* o, const double* x, double* y) { stencil(o, 2, x, y); }

void orc_pair_solve(const orc_t* o, const double* b, double* out) {
  const int n = o->n, q = o->q, T1 = o->T + 1, nb = o->nb, V = o->V;
#pragma omp parallel
  {
    double* work = (double*)malloc(sizeof(double) * (size_t)nb * q);
    double seg[32], acc[32];
#pragma omp for schedule(static)
    for (long tv = 0; tv < (long)T1 * V; ++tv) {
      const int t = (int)(tv / V), v = (int)(tv % V);
      const int pc = o->psi_cls[t];
      const double* Lb = o->linv + (long)pc * nb * V * q * q;
      const double* Sb = o->sub + (long)pc * nb * V * q * q;
      for (int k = 0; k < nb; ++k) {
        for (int p = 0; p < q; ++p) {
          const int s = p / n, kk = p % n, i = 2 * k + (s >> 1), j = 2 * v + (s & 1);
          seg[p] = in_grid(o, j, i) ? b[vi(o, t, j, i) + kk] : 0.0;
        }
        if (k) {
          const double* C = Sb + ((long)k * V + v) * q * q;
          const double* wp = work + (long)(k - 1) * q;
          for (int p = 0; p < q; ++p) {
            double s = 0.0;
            for (int c = 0; c < q; ++c) s += C[p * q + c] * wp[c];
            acc[p] = s;
          }
          for (int p = 0; p < q; ++p) seg[p] -= acc[p];
        }
        const double* Li = Lb + ((long)k * V + v) * q * q;
        double* w = work + (long)k * q;
        for (int p = 0; p < q; ++p) {
          double s = 0.0;
          for (int c = 0; c <= p; ++c) s += Li[p * q + c] * seg[c];
          w[p] = s;
        }
      }
      for (int k = nb - 1; k >= 0; --k) {
        double* w = work + (long)k * q;
        for (int p = 0; p < q; ++p) seg[p] = w[p];
        if (k + 1 < nb) {
          const double* C = Sb + ((long)(k + 1) * V + v) * q * q;
          const double* xn = work + (long)(k + 1) * q;
          for (int p = 0; p < q; ++p) {
            double s = 0.0;
            for (int c = 0; c < q; ++c) s += C[c * q + p] * xn[c];
            seg[p] -= s;
          }
        }
        const double* Li = Lb + ((long)k * V + v) * q * q;
        for (int p = 0; p < q; ++p) {
          double s = 0.0;
          for (int c = p; c < q; ++c) s += Li[c * q + p] * seg[c];
          w[p] = s;
        }
        for (int p = 0; p < q; ++p) {
          const int s = p / n, kk = p % n, i = 2 * k + (s >> 1), j = 2 * v + (s & 1);
          if (in_grid(o, j, i)) out[vi(o, t, j, i) + kk] = w[p];
        }
      }
    }
    free(work);
  }
}

static long dimof(const orc_t* o) { return (long)(o->T + 1) * o->N * o->K * o->n; }

static void vadd(long d, const double* a, const double* b, double* out) {
#pragma omp parallel for schedule(static)
  for (long e = 0; e < d; ++e) out[e] = a[e] + b[e];
}

/* theta = inner_sweep(rhs) from the zero start (nested_jacobi.py:79-103) */
static void inner_sweep(const orc_t* o, int L, const double* rhs, double* theta, double* w1,
                        double* w2) {
  const long d = dimof(o);
  orc_pair_solve(o, rhs, theta);
  for (int l = 1; l < L; ++l) {
    orc_inner(o, theta, w1);
    vadd(d, rhs, w1, w2);
    orc_pair_solve(o, w2, theta);
  }
}

/* q = P r (nested_jacobi.py:105-122); work: 4 vectors */
void orc_precond(const orc_t* o, int L, int S, const double* r, double* q, double* work) {
  const long d = dimof(o);
  double *w1 = work, *w2 = work + d, *w3 = work + 2 * d, *dl = work + 3 * d;
  inner_sweep(o, L, r, dl, w1, w2);
  for (int s = 1; s < S; ++s) {
    orc_outer(o, dl, w1);
    vadd(d, r, w1, w3);
    inner_sweep(o, L, w3, dl, w1, w2);
  }
  memcpy(q, dl, sizeof(double) * d);
}

static double dot(long d, const double* a, const double* b) {
  int nt = 1;
#ifdef _OPENMP
  nt = omp_get_max_threads();
#endif
  double* part = (double*)calloc(nt, sizeof(double));
#pragma omp parallel
  {
    int id = 0;
#ifdef _OPENMP
    id = omp_get_thread_num();
#endif
    double s = 0.0;
#pragma omp for schedule(static)
    for (long e = 0; e < d; ++e) s += a[e] * b[e];
    part[id] = s;
  }
  double s = 0.0;
  for (int k = 0; k < nt; ++k) s += part[k];
  free(part);
  return s;
}

/* pcg_solve control flow (pcg.py:50-149).  Returns 0 ok/converged-or-budget, 2 breakdown.
 * work: 7 vectors.  `step_seconds` (optional, length max_steps) gets cumulative wall time
 * at the end of each step. */
int orc_pcg(const orc_t* o, int L, int S, int use_precond, const double* rhs, double tol,
            long max_steps, double* x, double* hist, long* steps_out, int* converged,
            double* work, double* step_seconds) {
  const long d = dimof(o);
  double *r = work, *dv = work + d, *y = work + 2 * d, *qv = work + 3 * d, *pw = work + 4 * d;
  /* pw needs 4 vectors: work must hold 8 */
  memset(x, 0, sizeof(double) * d);
  memcpy(r, rhs, sizeof(double) * d);
  if (use_precond) orc_precond(o, L, S, r, dv, pw);
  else memcpy(dv, r, sizeof(double) * d);
  double mu = dot(d, dv, r);
  long steps = 0;
  *converged = 0;
#ifdef _OPENMP
  const double t0 = omp_get_wtime();
#endif
  for (long it = 0; it < max_steps; ++it) {
    orc_delta(o, dv, y);
    const double curv = dot(d, y, dv);
    if (curv <= 0.0) {
      *steps_out = steps;
      return 2;
    }
    const double alpha = mu / curv;
    double res = 0.0;
    int nan = 0;
#pragma omp parallel for schedule(static) reduction(max : res) reduction(| : nan)
    for (long e = 0; e < d; ++e) {
      x[e] += alpha * dv[e];
      r[e] = r[e] - alpha * y[e];
      const double a = fabs(r[e]);
      if (a != a) nan = 1;
      if (a > res) res = a;
    }
    if (nan) res = NAN;
    hist[steps++] = res;
#ifdef _OPENMP
    if (step_seconds) step_seconds[steps - 1] = omp_get_wtime() - t0;
#endif
    if (res < tol) {
      *converged = 1;
      break;
    }
    const double* qq = r;
    if (use_precond) {
      orc_precond(o, L, S, r, qv, pw);
      qq = qv;
    }
    const double mu_next = dot(d, qq, r);
    const double beta = mu_next / mu;
#pragma omp parallel for schedule(static)
    for (long e = 0; e < d; ++e) dv[e] = qq[e] + beta * dv[e];
    mu = mu_next;
  }
  *steps_out = steps;
  return 0;
}

int orc_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
