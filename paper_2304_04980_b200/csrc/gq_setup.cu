// Setup kernels, run once per problem: cost inverses, the reduced-operator blocks Psi / Xi
// per stage class, and the block Cholesky factors of every column-pair chain.
//
// Reference formulas:
//   spd_inverse (column Cholesky, pivot <= 1e-14*max diag -> not SPD, forward-substitution
//     inverse, Linv' Linv symmetrised)              gridlq/block_linalg.py:43-85
//   Psi_0 = Qinv_0 ; Psi_t = Qinv_t + Ahat Qinv_{t-1} Ahat' + sym(B R^-1 B'), diagonal
//     blocks symmetrised                            gridlq/kkt_assembly.py:493-533
//   Xi_t = -Ahat_t Qinv_t                           gridlq/kkt_assembly.py:535-543
//   pair extraction (row-interleaved, rows paired)  kkt_assembly.py:579-641, block_linalg.py:277-301
//   block tri-diagonal Cholesky                     gridlq/block_linalg.py:371-398
// Psi is made exactly symmetric by computing every off-diagonal block once, at its
// canonical owner (the later node in the (j, i) order), and transposing for the mirror,
// as the reference's lower-triangle storage does.
#include <cmath>

#include "gq_internal.h"

namespace gq {

constexpr double kPivotRtol = 1e-14;

// ---- generic small dense helpers (runtime dim <= 8) -------------------------------------

__device__ bool dev_cholesky(const double* m, double* lower, int n, double* piv_out,
                             double* tol_out, int* col_out) {
  double mx = -INFINITY;
  for (int j = 0; j < n; ++j) mx = fmax(mx, m[j * n + j]);
  const double tol = kPivotRtol * mx;
  for (int e = 0; e < n * n; ++e) lower[e] = 0.0;
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int k = 0; k < j; ++k) s = fma(lower[j * n + k], lower[j * n + k], s);
    const double piv = m[j * n + j] - s;
    if (!(piv > tol)) {
      *piv_out = piv;
      *tol_out = tol;
      *col_out = j;
      return false;
    }
    const double ljj = sqrt(piv);
    lower[j * n + j] = ljj;
    for (int r = j + 1; r < n; ++r) {
      double a = 0.0;
      for (int k = 0; k < j; ++k) a = fma(lower[r * n + k], lower[j * n + k], a);
      lower[r * n + j] = (m[r * n + j] - a) / ljj;
    }
  }
  return true;
}

__device__ void dev_lower_inverse(const double* lower, double* inv, int n) {
  for (int e = 0; e < n * n; ++e) inv[e] = 0.0;
  for (int i = 0; i < n; ++i) {
    for (int c = 0; c < n; ++c) {
      double s = 0.0;
      for (int k = 0; k < i; ++k) s = fma(lower[i * n + k], inv[k * n + c], s);
      double row = -s;
      if (c == i) row += 1.0;
      inv[i * n + c] = row / lower[i * n + i];
    }
  }
}

__global__ void k_spd_inverse(const double* __restrict__ in, double* __restrict__ out,
                              long long count, int n, SetupErr* err) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  double m[64], lo[64], li[64];
  const double* src = in + idx * n * n;
  for (int e = 0; e < n * n; ++e) m[e] = src[e];
  double piv, tol;
  int col;
  if (!dev_cholesky(m, lo, n, &piv, &tol, &col)) {
    if (atomicCAS(&err->code, 0, 2) == 0) {
      err->cls = (int)idx;
      err->j = col;
      err->pivot = piv;
      err->tol = tol;
    }
    return;
  }
  dev_lower_inverse(lo, li, n);
  double* dst = out + idx * n * n;
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s = fma(li[k * n + r], li[k * n + c], s);
      m[r * n + c] = s;
    }
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) dst[r * n + c] = 0.5 * (m[r * n + c] + m[c * n + r]);
}

cudaError_t launch_spd_inverse(const double* in, double* out, long long count, int dim,
                               SetupErr* err, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  k_spd_inverse<<<(unsigned)((count + 127) / 128), 128, 0, s>>>(in, out, count, dim, err);
  return cudaGetLastError();
}

// brb[dc][node] = sym((B Rinv) B')
__global__ void k_brb(long long count, int n, int m, const double* __restrict__ B,
                      const double* __restrict__ rinv, double* __restrict__ brb) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  const double* b = B + idx * n * m;
  const double* ri = rinv + idx * m * m;
  double bt[64], t[64];
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < m; ++c) {
      double s = 0.0;
      for (int k = 0; k < m; ++k) s = fma(b[r * m + k], ri[k * m + c], s);
      bt[r * m + c] = s;
    }
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) {
      double s = 0.0;
      for (int k = 0; k < m; ++k) s = fma(bt[r * m + k], b[c * m + k], s);
      t[r * n + c] = s;
    }
  double* o = brb + idx * n * n;
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) o[r * n + c] = 0.5 * (t[r * n + c] + t[c * n + r]);
}

cudaError_t launch_brb(const Geo& g, int m, int n_dyn, const double* B, const double* rinv,
                       double* brb, cudaStream_t s) {
  const long long count = (long long)n_dyn * g.nk;
  k_brb<<<(unsigned)((count + 127) / 128), 128, 0, s>>>(count, g.n, m, B, rinv, brb);
  return cudaGetLastError();
}

// ---- Psi / Xi assembly (templated on n) --------------------------------------------------

template <int NS>
struct Blk {
  double a[NS * NS];
};

template <int NS>
__device__ __forceinline__ Blk<NS> ld_blk(const double* p) {
  Blk<NS> b;
#pragma unroll
  for (int e = 0; e < NS * NS; ++e) b.a[e] = p[e];
  return b;
}
template <int NS>
__device__ __forceinline__ Blk<NS> blk_zero() {
  Blk<NS> b;
#pragma unroll
  for (int e = 0; e < NS * NS; ++e) b.a[e] = 0.0;
  return b;
}
// X @ Y
template <int NS>
__device__ __forceinline__ Blk<NS> mm(const Blk<NS>& x, const Blk<NS>& y) {
  Blk<NS> o;
#pragma unroll
  for (int r = 0; r < NS; ++r)
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < NS; ++k) s = fma(x.a[r * NS + k], y.a[k * NS + c], s);
      o.a[r * NS + c] = s;
    }
  return o;
}
// X @ Y'
template <int NS>
__device__ __forceinline__ Blk<NS> mmt(const Blk<NS>& x, const Blk<NS>& y) {
  Blk<NS> o;
#pragma unroll
  for (int r = 0; r < NS; ++r)
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < NS; ++k) s = fma(x.a[r * NS + k], y.a[c * NS + k], s);
      o.a[r * NS + c] = s;
    }
  return o;
}

struct RawData {
  const double* A;      // [nd][N][K][n][n]
  const double* C;      // [nd][4][N][K][n][n]
  const double* qinv;   // [nq][N][K][n][n]
  const double* brb;    // [nd][N][K][n][n]
};

// Ahat(a, a+off5[u]) for dynamics set dc; zero if the neighbour is off-grid
template <int NS>
__device__ Blk<NS> ahat(const Geo& g, const RawData& d, int dc, int j, int i, int u) {
  const int jj = j + odj(u), ii = i + odi(u);
  if (jj < 0 || jj >= g.N || ii < 0 || ii >= g.K) return blk_zero<NS>();
  const long long node = (long long)j * g.K + i;
  if (u == 0) return ld_blk<NS>(d.A + ((long long)dc * g.nk + node) * NS * NS);
  return ld_blk<NS>(d.C + (((long long)dc * 4 + slot_dir(u)) * g.nk + node) * NS * NS);
}

template <int NS>
__device__ Blk<NS> qinv_at(const Geo& g, const RawData& d, int qc, int j, int i) {
  if (j < 0 || j >= g.N || i < 0 || i >= g.K) return blk_zero<NS>();
  return ld_blk<NS>(d.qinv + ((long long)qc * g.nk + (long long)j * g.K + i) * NS * NS);
}

template <int NS>
__global__ void k_xi(Geo g, int nxc, const int* __restrict__ keys, RawData d,
                     double* __restrict__ xi, double* __restrict__ xit) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)nxc * g.nk) return;
  const int xc = (int)(idx / g.nk);
  const long long node = idx % g.nk;
  const int j = (int)(node / g.K), i = (int)(node % g.K);
  const int dc = keys[2 * xc], qc = keys[2 * xc + 1];
  double* xo = xi + idx * 5 * NS * NS;
  double* xto = xit + idx * 5 * NS * NS;
  const Blk<NS> qa = qinv_at<NS>(g, d, qc, j, i);
  for (int u = 0; u < 5; ++u) {
    const int jj = j + odj(u), ii = i + odi(u);
    const bool in = jj >= 0 && jj < g.N && ii >= 0 && ii < g.K;
    Blk<NS> x1 = blk_zero<NS>(), x2 = blk_zero<NS>();
    if (in) {
      // Xi(a, p) = -(Ahat(a,p) Qinv(p))
      x1 = mm<NS>(ahat<NS>(g, d, dc, j, i, u), qinv_at<NS>(g, d, qc, jj, ii));
      // Xi(p, a) = -(Ahat(p,a) Qinv(a)), stored transposed
      x2 = mm<NS>(ahat<NS>(g, d, dc, jj, ii, slot_opp(u)), qa);
    }
#pragma unroll
    for (int r = 0; r < NS; ++r)
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        xo[u * NS * NS + r * NS + c] = -x1.a[r * NS + c];
        xto[u * NS * NS + r * NS + c] = -x2.a[c * NS + r];
      }
  }
}

__device__ __forceinline__ int off_index(int di, int dj) {
  for (int o = 0; o < 13; ++o)
    if (odi(o) == di && odj(o) == dj) return o;
  return -1;
}

// 5-point slots in the global (j, i) order of the node they point at
__device__ __forceinline__ int order5(int k) {
  return k == 0 ? 3 : k == 1 ? 1 : k == 2 ? 0 : k == 3 ? 2 : 4;
}

template <int NS>
__global__ void k_psi(Geo g, int npc, const int* __restrict__ keys, RawData d,
                      double* __restrict__ psi) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)npc * g.nk) return;
  const int pc = (int)(idx / g.nk);
  const long long node = idx % g.nk;
  const int j = (int)(node / g.K), i = (int)(node % g.K);
  const int qc = keys[3 * pc], dc = keys[3 * pc + 1], qp = keys[3 * pc + 2];
  double* out = psi + idx * 13 * NS * NS;
  const Blk<NS> qa = qinv_at<NS>(g, d, qc, j, i);
  if (dc < 0) {   // Psi_0 = Qinv_0
    for (int e = 0; e < 13 * NS * NS; ++e) out[e] = 0.0;
#pragma unroll
    for (int e = 0; e < NS * NS; ++e) out[e] = qa.a[e];
    return;
  }
  // pre[u] = Ahat(a, a+u) Qinv_{t-1}(a+u)
  Blk<NS> pre[5];
  for (int u = 0; u < 5; ++u)
    pre[u] = mm<NS>(ahat<NS>(g, d, dc, j, i, u), qinv_at<NS>(g, d, qp, j + odj(u), i + odi(u)));
  {  // diagonal block
    Blk<NS> acc = qa;
    for (int k = 0; k < 5; ++k) {
      const int u = order5(k);
      const Blk<NS> term = mmt<NS>(pre[u], ahat<NS>(g, d, dc, j, i, u));
#pragma unroll
      for (int e = 0; e < NS * NS; ++e) acc.a[e] = acc.a[e] + term.a[e];
    }
    const Blk<NS> bb = ld_blk<NS>(d.brb + ((long long)dc * g.nk + node) * NS * NS);
#pragma unroll
    for (int e = 0; e < NS * NS; ++e) acc.a[e] = acc.a[e] + bb.a[e];
#pragma unroll
    for (int r = 0; r < NS; ++r)
#pragma unroll
      for (int c = 0; c < NS; ++c) out[r * NS + c] = 0.5 * (acc.a[r * NS + c] + acc.a[c * NS + r]);
  }
  for (int o = 1; o < 13; ++o) {
    const int di = odi(o), dj = odj(o);
    const int jb = j + dj, ib = i + di;
    double* ob = out + o * NS * NS;
    if (jb < 0 || jb >= g.N || ib < 0 || ib >= g.K) {
      for (int e = 0; e < NS * NS; ++e) ob[e] = 0.0;
      continue;
    }
    const bool before = (dj < 0) || (dj == 0 && di < 0);
    Blk<NS> acc = blk_zero<NS>();
    for (int k = 0; k < 5; ++k) {
      const int u = order5(k);
      // common node s = a + off5[u] = b + off5[w]
      const int wdi = odi(u) - di, wdj = odj(u) - dj;
      int w = -1;
      for (int q = 0; q < 5; ++q)
        if (odi(q) == wdi && odj(q) == wdj) w = q;
      if (w < 0) continue;
      Blk<NS> term;
      if (before) {
        term = mmt<NS>(pre[u], ahat<NS>(g, d, dc, jb, ib, w));
      } else {
        const Blk<NS> pre_b =
            mm<NS>(ahat<NS>(g, d, dc, jb, ib, w), qinv_at<NS>(g, d, qp, jb + odj(w), ib + odi(w)));
        term = mmt<NS>(pre_b, ahat<NS>(g, d, dc, j, i, u));
      }
#pragma unroll
      for (int e = 0; e < NS * NS; ++e) acc.a[e] = acc.a[e] + term.a[e];
    }
#pragma unroll
    for (int r = 0; r < NS; ++r)
#pragma unroll
      for (int c = 0; c < NS; ++c) ob[r * NS + c] = before ? acc.a[r * NS + c] : acc.a[c * NS + r];
  }
}

// ---- pair-chain block Cholesky -------------------------------------------------------------
// One thread per (class, pair); matrices live in a global scratch slab (q <= 32).
template <int NS>
__global__ void k_factor(Geo g, int npc, const double* __restrict__ psi, double* __restrict__ fac,
                         double* __restrict__ scratch, SetupErr* err) {
  constexpr int Q = 4 * NS;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)npc * g.V) return;
  const int pc = (int)(idx / g.V), v = (int)(idx % g.V);
  double* mkk = scratch + idx * 5 * Q * Q;
  double* mk1 = mkk + Q * Q;
  double* sc = mk1 + Q * Q;
  double* lo = sc + Q * Q;
  double* cc = lo + Q * Q;
  const double* P = psi + (long long)pc * g.nk * 13 * NS * NS;
  double* F = fac + idx * g.nb * 2 * Q * Q;
  for (int k = 0; k < g.nb; ++k) {
    bool real[Q];
    for (int p = 0; p < Q; ++p) {
      const int s = p / NS;
      real[p] = (2 * k + (s >> 1) < g.K) && (2 * v + (s & 1) < g.N);
    }
    for (int p = 0; p < Q; ++p) {
      const int s = p / NS, kk = p % NS;
      const int i = 2 * k + (s >> 1), j = 2 * v + (s & 1);
      for (int p2 = 0; p2 < Q; ++p2) {
        const int s2 = p2 / NS, kk2 = p2 % NS;
        const int ci2 = s2 & 1, ri2 = s2 >> 1;
        // M_kk
        double val = (p == p2) ? 1.0 : 0.0;
        if (real[p] && real[p2]) {
          const int o = off_index(2 * k + ri2 - i, 2 * v + ci2 - j);
          val = P[(((long long)j * g.K + i) * 13 + o) * NS * NS + kk * NS + kk2];
        }
        mkk[p * Q + p2] = val;
        // M_{k,k-1}
        double v1 = 0.0;
        if (k > 0 && real[p]) {
          const int i2 = 2 * (k - 1) + ri2, j2 = 2 * v + ci2;
          const int di = i2 - i, dj = j2 - j;
          if (j2 < g.N && (di < 0 ? -di : di) + (dj < 0 ? -dj : dj) <= 2)
            v1 = P[(((long long)j * g.K + i) * 13 + off_index(di, dj)) * NS * NS + kk * NS + kk2];
        }
        mk1[p * Q + p2] = v1;
      }
    }
    double* Lk = F + (long long)k * 2 * Q * Q;
    double* Ck = Lk + Q * Q;
    if (k > 0) {
      const double* Lprev = F + (long long)(k - 1) * 2 * Q * Q;
      // C = M_{k,k-1} Linv_{k-1}'
      for (int p = 0; p < Q; ++p)
        for (int c = 0; c < Q; ++c) {
          double s = 0.0;
          for (int m = 0; m < Q; ++m) s = fma(mk1[p * Q + m], Lprev[c * Q + m], s);
          cc[p * Q + c] = s;
        }
      for (int p = 0; p < Q; ++p)
        for (int c = 0; c < Q; ++c) {
          double s = 0.0;
          for (int m = 0; m < Q; ++m) s = fma(cc[p * Q + m], cc[c * Q + m], s);
          sc[p * Q + c] = mkk[p * Q + c] - s;
        }
      for (int p = 0; p < Q; ++p)
        for (int c = 0; c < p; ++c) {
          const double a = 0.5 * (sc[p * Q + c] + sc[c * Q + p]);
          sc[p * Q + c] = a;
          sc[c * Q + p] = a;
        }
      for (int e = 0; e < Q * Q; ++e) Ck[e] = cc[e];
    } else {
      for (int e = 0; e < Q * Q; ++e) {
        sc[e] = mkk[e];
        Ck[e] = 0.0;
      }
    }
    // pivot threshold over real positions only (padding rows are identity)
    double mx = -INFINITY;
    for (int p = 0; p < Q; ++p)
      if (real[p]) mx = fmax(mx, sc[p * Q + p]);
    const double tol = kPivotRtol * mx;
    for (int e = 0; e < Q * Q; ++e) lo[e] = 0.0;
    for (int jc = 0; jc < Q; ++jc) {
      double s = 0.0;
      for (int m = 0; m < jc; ++m) s = fma(lo[jc * Q + m], lo[jc * Q + m], s);
      const double piv = sc[jc * Q + jc] - s;
      if (!(piv > tol)) {
        if (atomicCAS(&err->code, 0, 1) == 0) {
          err->cls = pc;
          err->v = v;
          err->k = k;
          err->j = jc;
          err->pivot = piv;
          err->tol = tol;
        }
        return;
      }
      const double ljj = sqrt(piv);
      lo[jc * Q + jc] = ljj;
      for (int r = jc + 1; r < Q; ++r) {
        double a = 0.0;
        for (int m = 0; m < jc; ++m) a = fma(lo[r * Q + m], lo[jc * Q + m], a);
        lo[r * Q + jc] = (sc[r * Q + jc] - a) / ljj;
      }
    }
    // Linv by forward substitution, straight into the factor slab
    for (int e = 0; e < Q * Q; ++e) Lk[e] = 0.0;
    for (int ii = 0; ii < Q; ++ii)
      for (int c = 0; c <= ii; ++c) {
        double s = 0.0;
        for (int m = c; m < ii; ++m) s = fma(lo[ii * Q + m], Lk[m * Q + c], s);
        double row = -s;
        if (c == ii) row += 1.0;
        Lk[ii * Q + c] = row / lo[ii * Q + ii];
      }
  }
}

template <int NS>
static cudaError_t launch_setup_n(const Geo& g, int which, int ncls, const int* keys,
                                  const RawData& d, double* o1, double* o2, double* scratch,
                                  SetupErr* err, cudaStream_t s) {
  if (which == 0) {
    const long long count = (long long)ncls * g.nk;
    k_xi<NS><<<(unsigned)((count + 127) / 128), 128, 0, s>>>(g, ncls, keys, d, o1, o2);
  } else if (which == 1) {
    const long long count = (long long)ncls * g.nk;
    k_psi<NS><<<(unsigned)((count + 127) / 128), 128, 0, s>>>(g, ncls, keys, d, o1);
  } else {
    const long long count = (long long)ncls * g.V;
    k_factor<NS><<<(unsigned)((count + 63) / 64), 64, 0, s>>>(g, ncls, o1, o2, scratch, err);
  }
  return cudaGetLastError();
}

static cudaError_t launch_setup(const Geo& g, int which, int ncls, const int* keys,
                                const RawData& d, double* o1, double* o2, double* scratch,
                                SetupErr* err, cudaStream_t s) {
  switch (g.n) {
    case 1: return launch_setup_n<1>(g, which, ncls, keys, d, o1, o2, scratch, err, s);
    case 2: return launch_setup_n<2>(g, which, ncls, keys, d, o1, o2, scratch, err, s);
    case 3: return launch_setup_n<3>(g, which, ncls, keys, d, o1, o2, scratch, err, s);
    case 4: return launch_setup_n<4>(g, which, ncls, keys, d, o1, o2, scratch, err, s);
    case 8: return launch_setup_n<8>(g, which, ncls, keys, d, o1, o2, scratch, err, s);
    default: return cudaErrorInvalidValue;
  }
}

// ---- primal recovery and KKT residuals (recovery.py:50-80) --------------------------------
// One thread per (stage t, node a); vectors in the reference order (t, j, i, k).
//   (A~' lam)_t(a) = -lam_t(a) + [t < T] sum_u Ahat_t(a+off_u, opp(u))' lam_{t+1}(a+off_u)
//   x_t(a) = -Qinv_t(a) (A~' lam)_t(a)             u_t(a) = -Rinv_t(a) B_t(a)' lam_{t+1}(a)
//   objective = 0.5 (x'Qx + u'Ru)                  (kkt_assembly.py:84-160)
//   r_x = Q x + A~' lam,  r_u = R u + B~' lam,  r_dyn = A~ x + B~ u + omega~
struct RecData {
  const double* B;      // [nd][N][K][n][m]
  const double* R;      // [nd][N][K][m][m]
  const double* rinv;   // [nd][N][K][m][m]
  const double* Q;      // [nq][N][K][n][n]
  const int* dcls;      // [T]
  const int* ccls;      // [T+1]
  int m;
};

template <int NS>
__device__ void at_lambda(const Geo& g, const RawData& d, const RecData& r, const double* lam,
                          int t, int j, int i, double* a) {
  const long long nhat = g.nk * NS;
  const long long node = (long long)j * g.K + i;
#pragma unroll
  for (int k = 0; k < NS; ++k) a[k] = -lam[t * nhat + node * NS + k];
  if (t < g.T) {
    const int dc = r.dcls[t];
    for (int u = 0; u < 5; ++u) {
      const int jj = j + odj(u), ii = i + odi(u);
      if (jj < 0 || jj >= g.N || ii < 0 || ii >= g.K) continue;
      const Blk<NS> ab = ahat<NS>(g, d, dc, jj, ii, slot_opp(u));
      const double* y = lam + (t + 1) * nhat + ((long long)jj * g.K + ii) * NS;
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        double s = 0.0;
#pragma unroll
        for (int rr = 0; rr < NS; ++rr) s = fma(ab.a[rr * NS + c], y[rr], s);
        a[c] += s;
      }
    }
  }
}

template <int NS>
__global__ void k_recover(Geo g, RawData d, RecData r, const double* __restrict__ lam,
                          double* __restrict__ xo, double* __restrict__ uo,
                          double* __restrict__ part) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double obj = 0.0;
  if (idx < (long long)g.T1 * g.nk) {
    const int t = (int)(idx / g.nk);
    const long long node = idx % g.nk;
    const int j = (int)(node / g.K), i = (int)(node % g.K);
    const long long nhat = g.nk * NS;
    double a[NS], x[NS];
    at_lambda<NS>(g, d, r, lam, t, j, i, a);
    const Blk<NS> qi = qinv_at<NS>(g, d, r.ccls[t], j, i);
    const double* Qb = r.Q + ((long long)r.ccls[t] * g.nk + node) * NS * NS;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < NS; ++c) s = fma(qi.a[k * NS + c], a[c], s);
      x[k] = -s;
      xo[t * nhat + node * NS + k] = x[k];
    }
    double xq = 0.0;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < NS; ++c) s = fma(Qb[k * NS + c], x[c], s);
      xq = fma(x[k], s, xq);
    }
    obj = xq;
    if (t < g.T) {
      const int m = r.m, dc = r.dcls[t];
      const double* Bb = r.B + ((long long)dc * g.nk + node) * NS * m;
      const double* Ri = r.rinv + ((long long)dc * g.nk + node) * m * m;
      const double* Rb = r.R + ((long long)dc * g.nk + node) * m * m;
      const double* y = lam + (t + 1) * nhat + node * NS;
      double bt[8], u[8];
      for (int c = 0; c < m; ++c) {
        double s = 0.0;
        for (int k = 0; k < NS; ++k) s = fma(Bb[k * m + c], y[k], s);
        bt[c] = s;
      }
      for (int c = 0; c < m; ++c) {
        double s = 0.0;
        for (int e = 0; e < m; ++e) s = fma(Ri[c * m + e], bt[e], s);
        u[c] = -s;
        uo[(long long)t * g.nk * m + node * m + c] = u[c];
      }
      double ur = 0.0;
      for (int c = 0; c < m; ++c) {
        double s = 0.0;
        for (int e = 0; e < m; ++e) s = fma(Rb[c * m + e], u[e], s);
        ur = fma(u[c], s, ur);
      }
      obj += ur;
    }
  }
  obj = block_reduce<false>(obj);
  if (threadIdx.x == 0) part[blockIdx.x] = obj;
}

template <int NS>
__global__ void k_kkt(Geo g, RawData d, RecData r, const double* __restrict__ lam,
                      const double* __restrict__ x, const double* __restrict__ u,
                      const double* __restrict__ off, double* __restrict__ part) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double mx = 0.0, mu = 0.0, md = 0.0;
  if (idx < (long long)g.T1 * g.nk) {
    const int t = (int)(idx / g.nk);
    const long long node = idx % g.nk;
    const int j = (int)(node / g.K), i = (int)(node % g.K);
    const long long nhat = g.nk * NS;
    const int m = r.m;
    double a[NS];
    at_lambda<NS>(g, d, r, lam, t, j, i, a);
    const double* Qb = r.Q + ((long long)r.ccls[t] * g.nk + node) * NS * NS;
    const double* xa = x + t * nhat + node * NS;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < NS; ++c) s = fma(Qb[k * NS + c], xa[c], s);
      mx = nmax(mx, fabs(s + a[k]));
    }
    if (t < g.T) {
      const int dc = r.dcls[t];
      const double* Bb = r.B + ((long long)dc * g.nk + node) * NS * m;
      const double* Rb = r.R + ((long long)dc * g.nk + node) * m * m;
      const double* y = lam + (t + 1) * nhat + node * NS;
      const double* ua = u + (long long)t * g.nk * m + node * m;
      for (int c = 0; c < m; ++c) {
        double s = 0.0, b = 0.0;
        for (int e = 0; e < m; ++e) s = fma(Rb[c * m + e], ua[e], s);
        for (int k = 0; k < NS; ++k) b = fma(Bb[k * m + c], y[k], b);
        mu = nmax(mu, fabs(s + b));
      }
    }
    // dynamics rows: stage 0 is -x_0 + omega_0; stage t is Ahat_{t-1} x_{t-1} - x_t + B u + omega
    double rd[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) rd[k] = -xa[k] + off[t * nhat + node * NS + k];
    if (t > 0) {
      const int dc = r.dcls[t - 1];
      for (int uu = 0; uu < 5; ++uu) {
        const int jj = j + odj(uu), ii = i + odi(uu);
        if (jj < 0 || jj >= g.N || ii < 0 || ii >= g.K) continue;
        const Blk<NS> ab = ahat<NS>(g, d, dc, j, i, uu);
        const double* xp = x + (t - 1) * nhat + ((long long)jj * g.K + ii) * NS;
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < NS; ++c) s = fma(ab.a[k * NS + c], xp[c], s);
          rd[k] += s;
        }
      }
      const double* Bb = r.B + ((long long)dc * g.nk + node) * NS * m;
      const double* ua = u + (long long)(t - 1) * g.nk * m + node * m;
      for (int k = 0; k < NS; ++k) {
        double s = 0.0;
        for (int c = 0; c < m; ++c) s = fma(Bb[k * m + c], ua[c], s);
        rd[k] += s;
      }
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) md = nmax(md, fabs(rd[k]));
  }
  mx = block_reduce<true>(mx);
  mu = block_reduce<true>(mu);
  md = block_reduce<true>(md);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = mx;
    part[3 * blockIdx.x + 1] = mu;
    part[3 * blockIdx.x + 2] = md;
  }
}

template <int NS>
static cudaError_t recover_n(const Geo& g, const RawData& d, const RecData& r, int which,
                             const double* lam, const double* x, const double* u,
                             const double* off, double* xo, double* uo, double* part,
                             cudaStream_t s) {
  const long long n = (long long)g.T1 * g.nk;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (which == 0)
    k_recover<NS><<<blocks, 256, 0, s>>>(g, d, r, lam, xo, uo, part);
  else
    k_kkt<NS><<<blocks, 256, 0, s>>>(g, d, r, lam, x, u, off, part);
  return cudaGetLastError();
}

int recover_blocks(const Geo& g) { return (int)(((long long)g.T1 * g.nk + 255) / 256); }

cudaError_t launch_recover(const Geo& g, int m, const double* A, const double* C,
                           const double* qinv, const double* B, const double* R,
                           const double* rinv, const double* Q, const int* dcls,
                           const int* ccls, int which, const double* lam, const double* x,
                           const double* u, const double* off, double* xo, double* uo,
                           double* part, cudaStream_t s) {
  RawData d{A, C, qinv, nullptr};
  RecData r{B, R, rinv, Q, dcls, ccls, m};
  if (m > 8) return cudaErrorInvalidValue;
  switch (g.n) {
    case 1: return recover_n<1>(g, d, r, which, lam, x, u, off, xo, uo, part, s);
    case 2: return recover_n<2>(g, d, r, which, lam, x, u, off, xo, uo, part, s);
    case 3: return recover_n<3>(g, d, r, which, lam, x, u, off, xo, uo, part, s);
    case 4: return recover_n<4>(g, d, r, which, lam, x, u, off, xo, uo, part, s);
    case 8: return recover_n<8>(g, d, r, which, lam, x, u, off, xo, uo, part, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_xi(const Geo& g, int nxc, const int* xi_keys, const double* A,
                      const double* C, const double* qinv, double* xi, double* xit,
                      cudaStream_t s) {
  if (nxc == 0) return cudaSuccess;
  RawData d{A, C, qinv, nullptr};
  return launch_setup(g, 0, nxc, xi_keys, d, xi, xit, nullptr, nullptr, s);
}

cudaError_t launch_psi(const Geo& g, int npc, const int* psi_keys, const double* A,
                       const double* C, const double* qinv, const double* brb, double* psi,
                       cudaStream_t s) {
  RawData d{A, C, qinv, brb};
  return launch_setup(g, 1, npc, psi_keys, d, psi, nullptr, nullptr, nullptr, s);
}

cudaError_t launch_factor(const Geo& g, int npc, const double* psi, double* fac,
                          double* scratch, SetupErr* err, cudaStream_t s) {
  RawData d{nullptr, nullptr, nullptr, nullptr};
  return launch_setup(g, 2, npc, nullptr, d, const_cast<double*>(psi), fac, scratch, err, s);
}

}  // namespace gq
