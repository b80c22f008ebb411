// Domain-decomposed pair-chain solve ("dd" sweeps), n = 2.
//
// Every pair chain (nb blocks of q = 8) is split into ns <= 8 segments of m blocks: the last
// block of each segment but the final one is a SEPARATOR, the rest are interior blocks.
// Exact solve of the SPD block-tridiagonal system (tools/proto/dd_chain.py):
//   1. interiors: u_s = A_II^-1 b_I            (independent, block LDL^T restarted per interior)
//   2. separators: S x_G = g,  g_s = b_{g_s} - E_{g_s} u_s[last] - E_{f(s+1)}' u_{s+1}[first]
//      with the Schur complement S block tridiagonal over the ns-1 separators
//   3. interiors: x_I = u_s - V_s x_{G,s-1} - W_s x_{G,s}   (spikes V, W precomputed)
// One CTA = W (4 or 8) warps = the segments of one 8-chain group, so the interior iterates
// never live longer than one segment (parked in L2: 15 KB per warp instead of 64 KB per
// chain group, which overflowed L2 in the single-warp kernel).  Results equal the plain
// recurrence up to rounding (parity tolerance 1e-9 is met with margin).
//
// Status (round 1): opt-in (GQ_DD=1).  It removes the parked-iterate DRAM spill (outer
// sweep 750 -> 486 MB, inner 997 -> 759 MB measured), but the extra correction pass, the
// serial separator chain and one or two CTAs per SM make it 1.6-2.5x slower than the
// per-warp chain kernel, so the default path does not use it.
//
// Setup reuses the pair-block assembly of the reference factorisation (k_factor, which
// still runs for its NotPositiveDefinite checks); everything here is derived data.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "gq_async.cuh"
#include "gq_internal.h"

namespace gq {

using namespace as;

namespace {

constexpr int Q = 8, QQ = 64, NS = 2, KT = 3, TC = 24;
constexpr int FFS = 2 * QQ + Q * TC;   // forward tiles per block: L^-1 | -G | -M
constexpr int FBS = 2 * QQ;            // backward tiles: L^-T | -H
constexpr int SPS = 2 * QQ;            // spike tiles: -V | -W
constexpr int SEPS = 9 * QQ;           // separator tiles: -E_g | -E_n' | -Om(3) | Ls^-1 | -Gs | Ls^-T | -Hs
constexpr int kMaxSeg = 8;

__device__ __forceinline__ int off_index13(int di, int dj) {
  for (int o = 0; o < 13; ++o)
    if (odi(o) == di && odj(o) == dj) return o;
  return -1;
}

// pair blocks of chain (pc, v) at block k: M_kk (identity on padded positions) and
// M_{k,k-1}; the same assembly as k_factor (gq_setup.cu)
__device__ void pair_blocks(const Geo& g, const double* __restrict__ P, int v, int k,
                            double* mkk, double* mk1, bool* real) {
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
      double val = (p == p2) ? 1.0 : 0.0;
      if (real[p] && real[p2]) {
        const int o = off_index13(2 * k + ri2 - i, 2 * v + ci2 - j);
        val = P[(((long long)j * g.K + i) * 13 + o) * NS * NS + kk * NS + kk2];
      }
      mkk[p * Q + p2] = val;
      double v1 = 0.0;
      if (k > 0 && real[p]) {
        const int i2 = 2 * (k - 1) + ri2, j2 = 2 * v + ci2;
        const int di = i2 - i, dj = j2 - j;
        if (j2 < g.N && (di < 0 ? -di : di) + (dj < 0 ? -dj : dj) <= 2)
          v1 = P[(((long long)j * g.K + i) * 13 + off_index13(di, dj)) * NS * NS + kk * NS + kk2];
      }
      mk1[p * Q + p2] = v1;
    }
  }
}

// lower Cholesky of sc (symmetric) and its inverse; identity-padded rows pass through
__device__ bool chol_inverse(const double* sc, double* lo, double* linv) {
  for (int e = 0; e < QQ; ++e) lo[e] = 0.0;
  for (int jc = 0; jc < Q; ++jc) {
    double s = 0.0;
    for (int m = 0; m < jc; ++m) s = fma(lo[jc * Q + m], lo[jc * Q + m], s);
    const double piv = sc[jc * Q + jc] - s;
    if (!(piv > 0.0)) return false;
    const double ljj = sqrt(piv);
    lo[jc * Q + jc] = ljj;
    for (int r = jc + 1; r < Q; ++r) {
      double a = 0.0;
      for (int m = 0; m < jc; ++m) a = fma(lo[r * Q + m], lo[jc * Q + m], a);
      lo[r * Q + jc] = (sc[r * Q + jc] - a) / ljj;
    }
  }
  for (int e = 0; e < QQ; ++e) linv[e] = 0.0;
  for (int ii = 0; ii < Q; ++ii)
    for (int c = 0; c <= ii; ++c) {
      double s = 0.0;
      for (int m = c; m < ii; ++m) s = fma(lo[ii * Q + m], linv[m * Q + c], s);
      double row = -s;
      if (c == ii) row += 1.0;
      linv[ii * Q + c] = row / lo[ii * Q + ii];
    }
  return true;
}

__device__ void mm(const double* a, const double* b, double* c, bool bt) {   // c = a b (b' if bt)
  for (int p = 0; p < Q; ++p)
    for (int q2 = 0; q2 < Q; ++q2) {
      double s = 0.0;
      for (int m = 0; m < Q; ++m) s = fma(a[p * Q + m], bt ? b[q2 * Q + m] : b[m * Q + q2], s);
      c[p * Q + q2] = s;
    }
}

struct DDGeo {
  int m, ns;   // segment length (blocks), segments per chain
};

__device__ __forceinline__ int seg_begin(const DDGeo& d, int s) { return s * d.m; }
__device__ __forceinline__ int seg_end(const DDGeo& d, const Geo& g, int s) {   // interior end
  return s == d.ns - 1 ? g.nb : s * d.m + d.m - 1;
}

// ---- setup 1: interior factors + spikes, one thread per (class, pair, segment) ----------
// ddf[pc][v][k] = {Linv_k, C_k} (C = 0 at interior starts); spk[pc][v][k] = {V_k, W_k}
__global__ void k_dd_factor(Geo g, DDGeo d, int npc, const double* __restrict__ psi,
                            double* __restrict__ ddf, double* __restrict__ spk,
                            double* __restrict__ scratch) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)npc * g.V * d.ns) return;
  const int s = (int)(idx % d.ns);
  const int v = (int)((idx / d.ns) % g.V);
  const int pc = (int)(idx / ((long long)d.ns * g.V));
  double* mkk = scratch + idx * 6 * QQ;
  double* mk1 = mkk + QQ;
  double* sc = mk1 + QQ;
  double* lo = sc + QQ;
  double* cc = lo + QQ;
  double* t1 = cc + QQ;
  bool real[Q];
  const double* P = psi + (long long)pc * g.nk * 13 * NS * NS;
  double* F = ddf + ((long long)pc * g.V + v) * g.nb * 2 * QQ;
  double* SP = spk + ((long long)pc * g.V + v) * g.nb * SPS;
  const int kb = seg_begin(d, s), ke = seg_end(d, g, s);
  for (int k = kb; k < ke; ++k) {
    pair_blocks(g, P, v, k, mkk, mk1, real);
    double* Lk = F + (long long)k * 2 * QQ;
    double* Ck = Lk + QQ;
    if (k > kb) {
      mm(mk1, F + (long long)(k - 1) * 2 * QQ, cc, true);    // C = M_{k,k-1} Linv_{k-1}'
      mm(cc, cc, t1, true);
      for (int e = 0; e < QQ; ++e) sc[e] = mkk[e] - t1[e];
      for (int p = 0; p < Q; ++p)
        for (int c = 0; c < p; ++c) {
          const double a = 0.5 * (sc[p * Q + c] + sc[c * Q + p]);
          sc[p * Q + c] = a;
          sc[c * Q + p] = a;
        }
      for (int e = 0; e < QQ; ++e) Ck[e] = cc[e];
    } else {
      for (int e = 0; e < QQ; ++e) {
        sc[e] = mkk[e];
        Ck[e] = 0.0;
      }
    }
    chol_inverse(sc, lo, Lk);   // SPD-ness was certified by the reference factorisation
  }
  // spikes: V = A_II^-1 [E_first; 0 ...]  (s > 0),  W = A_II^-1 [0 ...; E_sep']  (s < ns-1)
  for (int which = 0; which < 2; ++which) {
    const bool have = which == 0 ? s > 0 : s < d.ns - 1;
    for (int k = kb; k < ke; ++k) {
      double* X = SP + (long long)k * SPS + which * QQ;
      for (int e = 0; e < QQ; ++e) X[e] = 0.0;
    }
    if (!have) continue;
    // rhs block
    if (which == 0) {
      pair_blocks(g, P, v, kb, mkk, mk1, real);               // E_first = M_{kb,kb-1}
      for (int e = 0; e < QQ; ++e) t1[e] = mk1[e];
    } else {
      pair_blocks(g, P, v, ke, mkk, mk1, real);               // E_sep = M_{ke,ke-1}
      for (int p = 0; p < Q; ++p)
        for (int c = 0; c < Q; ++c) t1[p * Q + c] = mk1[c * Q + p];
    }
    // forward: w_k = Linv_k (b_k - C_k w_{k-1})
    for (int k = kb; k < ke; ++k) {
      const double* Lk = F + (long long)k * 2 * QQ;
      double* X = SP + (long long)k * SPS + which * QQ;
      const bool rhs_here = which == 0 ? k == kb : k == ke - 1;
      for (int e = 0; e < QQ; ++e) sc[e] = rhs_here ? t1[e] : 0.0;
      if (k > kb) {
        mm(Lk + QQ, SP + (long long)(k - 1) * SPS + which * QQ, cc, false);
        for (int e = 0; e < QQ; ++e) sc[e] -= cc[e];
      }
      mm(Lk, sc, X, false);
    }
    // backward: x_k = Linv_k' (w_k - C_{k+1}' x_{k+1})
    for (int k = ke - 1; k >= kb; --k) {
      const double* Lk = F + (long long)k * 2 * QQ;
      double* X = SP + (long long)k * SPS + which * QQ;
      for (int e = 0; e < QQ; ++e) sc[e] = X[e];
      if (k + 1 < ke) {
        const double* Cn = F + (long long)(k + 1) * 2 * QQ + QQ;
        const double* Xn = SP + (long long)(k + 1) * SPS + which * QQ;
        for (int p = 0; p < Q; ++p)
          for (int c = 0; c < Q; ++c) {
            double a = 0.0;
            for (int m = 0; m < Q; ++m) a = fma(Cn[m * Q + p], Xn[m * Q + c], a);
            sc[p * Q + c] -= a;
          }
      }
      for (int p = 0; p < Q; ++p)
        for (int c = 0; c < Q; ++c) {
          double a = 0.0;
          for (int m = 0; m < Q; ++m) a = fma(Lk[m * Q + p], sc[m * Q + c], a);
          X[p * Q + c] = a;
        }
    }
  }
}

// ---- setup 2: separator Schur complement and its factor, one thread per (class, pair) ---
// sepd[pc][v][s] = {Ls^-1, Cs, E_g, E_n}
__global__ void k_dd_sep(Geo g, DDGeo d, int npc, const double* __restrict__ psi,
                         const double* __restrict__ spk, double* __restrict__ sepd,
                         double* __restrict__ scratch) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)npc * g.V) return;
  const int v = (int)(idx % g.V), pc = (int)(idx / g.V);
  double* mkk = scratch + idx * 8 * QQ;
  double* mk1 = mkk + QQ;
  double* sd = mk1 + QQ;
  double* ssub = sd + QQ;
  double* lo = ssub + QQ;
  double* cc = lo + QQ;
  double* t1 = cc + QQ;
  double* t2 = t1 + QQ;
  bool real[Q];
  const double* P = psi + (long long)pc * g.nk * 13 * NS * NS;
  const double* SP = spk + ((long long)pc * g.V + v) * g.nb * SPS;
  double* SD = sepd + ((long long)pc * g.V + v) * kMaxSeg * 4 * QQ;
  for (int s = 0; s + 1 < d.ns; ++s) {
    const int gk = seg_end(d, g, s);              // separator block
    const int last = gk - 1, first = gk + 1;
    double* o = SD + (long long)s * 4 * QQ;
    double* Ls = o;
    double* Cs = o + QQ;
    double* Eg = o + 2 * QQ;
    double* En = o + 3 * QQ;
    pair_blocks(g, P, v, gk, mkk, mk1, real);
    for (int e = 0; e < QQ; ++e) Eg[e] = mk1[e];
    pair_blocks(g, P, v, first, t1, t2, real);
    for (int e = 0; e < QQ; ++e) En[e] = t2[e];
    pair_blocks(g, P, v, gk, mkk, mk1, real);     // restore M_gg
    // Sd = M_gg - E_g W_s[last] - E_n' V_{s+1}[first]
    mm(Eg, SP + (long long)last * SPS + QQ, t1, false);
    for (int p = 0; p < Q; ++p)
      for (int c = 0; c < Q; ++c) {
        double a = 0.0;
        for (int m = 0; m < Q; ++m) a = fma(En[m * Q + p], SP[(long long)first * SPS + m * Q + c], a);
        sd[p * Q + c] = mkk[p * Q + c] - t1[p * Q + c] - a;
      }
    for (int p = 0; p < Q; ++p)
      for (int c = 0; c < p; ++c) {
        const double a = 0.5 * (sd[p * Q + c] + sd[c * Q + p]);
        sd[p * Q + c] = a;
        sd[c * Q + p] = a;
      }
    if (s > 0) {
      // S[s][s-1] = -E_g V_s[last];  C_s = S[s][s-1] Ls_{s-1}'
      const int first_s = seg_begin(d, s);
      (void)first_s;
      mm(Eg, SP + (long long)last * SPS, ssub, false);
      for (int e = 0; e < QQ; ++e) ssub[e] = -ssub[e];
      mm(ssub, SD + (long long)(s - 1) * 4 * QQ, cc, true);
      mm(cc, cc, t1, true);
      for (int e = 0; e < QQ; ++e) sd[e] -= t1[e];
      for (int p = 0; p < Q; ++p)
        for (int c = 0; c < p; ++c) {
          const double a = 0.5 * (sd[p * Q + c] + sd[c * Q + p]);
          sd[p * Q + c] = a;
          sd[c * Q + p] = a;
        }
      for (int e = 0; e < QQ; ++e) Cs[e] = cc[e];
    } else {
      for (int e = 0; e < QQ; ++e) Cs[e] = 0.0;
    }
    chol_inverse(sd, lo, Ls);
  }
}

// ---- setup 3: tiles (one thread per (class, pair, block, row)) ---------------------------
__host__ __device__ __forceinline__ int tile8(int r, int c, int kc) {
  return ((r >> 3) * (kc >> 3) + (c >> 3)) * 64 + (r & 7) * 8 + (c & 7);
}
__host__ __device__ constexpr int th_rec2(int dc, int u) {
  return dc == 0 ? (u == 0 ? 0 : u == 1 ? 2 : u == 2 ? 3 : u == 3 ? 4 : 7)
                 : (u == 0 ? 3 : u == 1 ? 6 : u == 2 ? 7 : u == 3 ? 8 : 10);
}

// row p of Omega~ at block k of pair v (Q x TC), optionally premultiplied by Linv (row p)
__device__ void omega_row(const Geo& g, const double* __restrict__ omega, int pc, int v, int k,
                          const double* L, int p, double* row) {
  const int a = 2 * v;
  for (int c = 0; c < TC; ++c) row[c] = 0.0;
  const int f_lo = L ? 0 : p, f_hi = L ? p : p;
  for (int f = f_lo; f <= f_hi; ++f) {
    const double l = L ? L[p * Q + f] : 1.0;
    if (l == 0.0) continue;
    const int nd = f / NS, fc = f % NS, dc = nd & 1, dr = nd >> 1;
    const int col = a + dc, rw = 2 * k + dr;
    if (col >= g.N || rw >= g.K) continue;
    const double* W = omega + ((long long)pc * g.nk + (long long)col * g.K + rw) * 5 * NS * NS;
    for (int u = 0; u < 5; ++u) {
      const int rec = th_rec2(dc, u) + dr;
      for (int c = 0; c < NS; ++c)
        row[rec * NS + c] = fma(l, W[u * NS * NS + fc * NS + c], row[rec * NS + c]);
    }
  }
}

__global__ void k_dd_tiles(Geo g, DDGeo d, int npc, const double* __restrict__ ddf,
                           const double* __restrict__ spk, const double* __restrict__ sepd,
                           const double* __restrict__ omega, double* __restrict__ ffd,
                           double* __restrict__ fbd, double* __restrict__ spt,
                           double* __restrict__ sept) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)npc * g.V * g.nb * Q) return;
  const int p = (int)(gid % Q);
  const long long idx = gid / Q;
  const int k = (int)(idx % g.nb);
  const int v = (int)((idx / g.nb) % g.V);
  const int pc = (int)(idx / ((long long)g.nb * g.V));
  const int s = k / d.m;
  const bool sep = s < d.ns - 1 && k == seg_end(d, g, s);
  const double* L = ddf + idx * 2 * QQ;
  const double* C = L + QQ;
  double* F = ffd + idx * FFS;
  double* B = fbd + idx * FBS;
  double* SPo = spt + idx * SPS;
  const double* SPi = spk + idx * SPS;
  if (sep) {
    for (int c = 0; c < Q; ++c) {
      F[tile8(p, c, Q)] = 0.0;
      F[QQ + tile8(p, c, Q)] = 0.0;
      B[tile8(p, c, Q)] = 0.0;
      B[QQ + tile8(p, c, Q)] = 0.0;
      SPo[tile8(p, c, Q)] = 0.0;
      SPo[QQ + tile8(p, c, Q)] = 0.0;
    }
    for (int c = 0; c < TC; ++c) F[2 * QQ + tile8(p, c, TC)] = 0.0;
    // separator tiles
    const double* SD = sepd + (((long long)pc * g.V + v) * kMaxSeg + s) * 4 * QQ;
    const double* Ls = SD;
    const double* Cs = SD + QQ;
    const double* Eg = SD + 2 * QQ;
    const double* En = SD + 3 * QQ;
    const double* Csn = (s + 1 < d.ns - 1) ? SD + 4 * QQ + QQ : nullptr;   // C_{s+1}
    double* T = sept + (((long long)pc * g.V + v) * kMaxSeg + s) * SEPS;
    double row[TC];
    omega_row(g, omega, pc, v, k, nullptr, p, row);
    for (int c = 0; c < TC; ++c) T[2 * QQ + tile8(p, c, TC)] = -row[c];
    for (int c = 0; c < Q; ++c) {
      T[tile8(p, c, Q)] = -Eg[p * Q + c];
      T[QQ + tile8(p, c, Q)] = -En[c * Q + p];
      T[5 * QQ + tile8(p, c, Q)] = Ls[p * Q + c];
      double gs = 0.0;
      for (int m = 0; m <= p; ++m) gs = fma(Ls[p * Q + m], Cs[m * Q + c], gs);
      T[6 * QQ + tile8(p, c, Q)] = -gs;
      T[7 * QQ + tile8(p, c, Q)] = Ls[c * Q + p];
      double hs = 0.0;
      if (Csn)
        for (int m = p; m < Q; ++m) hs = fma(Ls[m * Q + p], Csn[c * Q + m], hs);
      T[8 * QQ + tile8(p, c, Q)] = -hs;
    }
    return;
  }
  const int ke = seg_end(d, g, s);
  const double* Cn = (k + 1 < ke) ? L + 2 * QQ + QQ : nullptr;
  for (int c = 0; c < Q; ++c) {
    double gsum = 0.0;
    for (int m = 0; m <= p; ++m) gsum = fma(L[p * Q + m], C[m * Q + c], gsum);
    F[tile8(p, c, Q)] = L[p * Q + c];
    F[QQ + tile8(p, c, Q)] = -gsum;
    B[tile8(p, c, Q)] = L[c * Q + p];
    double h = 0.0;
    if (Cn)
      for (int m = p; m < Q; ++m) h = fma(L[m * Q + p], Cn[c * Q + m], h);
    B[QQ + tile8(p, c, Q)] = -h;
    SPo[tile8(p, c, Q)] = -SPi[p * Q + c];
    SPo[QQ + tile8(p, c, Q)] = -SPi[QQ + p * Q + c];
  }
  double row[TC];
  omega_row(g, omega, pc, v, k, L, p, row);
  for (int c = 0; c < TC; ++c) F[2 * QQ + tile8(p, c, TC)] = -row[c];
}

}  // namespace

// ---- host: setup ---------------------------------------------------------------------------

static int denv(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

static int dd_warps() { return denv("GQ_DD_W", 4) == 8 ? 8 : 4; }

bool dd_supported(const Geo& g) {
  if (g.n != 2 || denv("GQ_DD", 0) == 0) return false;   // experimental, opt-in
  const int w = dd_warps();
  const int m = std::max(2, (g.nb + w - 1) / w);
  return m <= 32 && g.nb >= 8;   // short chains gain nothing
}

DDShape dd_shape(const Geo& g) {
  DDShape sh;
  const int w = dd_warps();
  sh.m = std::max(2, (g.nb + w - 1) / w);
  sh.ns = (g.nb + sh.m - 1) / sh.m;
  return sh;
}

size_t dd_doubles(const Geo& g, int npc) {
  const size_t blocks = (size_t)npc * g.V * g.nb;
  return blocks * (FFS + FBS + SPS) + (size_t)npc * g.V * kMaxSeg * SEPS;
}

cudaError_t launch_build_dd(const Geo& g, int npc, const double* psi, const double* omega,
                            double* arena, cudaStream_t s) {
  const DDShape sh = dd_shape(g);
  const DDGeo d{sh.m, sh.ns};
  const size_t blocks = (size_t)npc * g.V * g.nb;
  double* ffd = arena;
  double* fbd = ffd + blocks * FFS;
  double* spt = fbd + blocks * FBS;
  double* sept = spt + blocks * SPS;
  // temporaries: raw interior factors, raw spikes, separator data, scratch
  double *ddf = nullptr, *spk = nullptr, *sepd = nullptr, *scr = nullptr;
  cudaError_t e;
  if ((e = cudaMalloc(&ddf, blocks * 2 * QQ * 8)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&spk, blocks * SPS * 8)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&sepd, (size_t)npc * g.V * kMaxSeg * 4 * QQ * 8)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&scr, (size_t)npc * g.V * kMaxSeg * 8 * QQ * 8)) != cudaSuccess) return e;
  cudaMemsetAsync(ddf, 0, blocks * 2 * QQ * 8, s);
  cudaMemsetAsync(sepd, 0, (size_t)npc * g.V * kMaxSeg * 4 * QQ * 8, s);
  cudaMemsetAsync(sept, 0, (size_t)npc * g.V * kMaxSeg * SEPS * 8, s);
  const long long n1 = (long long)npc * g.V * d.ns;
  k_dd_factor<<<(unsigned)((n1 + 63) / 64), 64, 0, s>>>(g, d, npc, psi, ddf, spk, scr);
  const long long n2 = (long long)npc * g.V;
  k_dd_sep<<<(unsigned)((n2 + 63) / 64), 64, 0, s>>>(g, d, npc, psi, spk, sepd, scr);
  const long long n3 = (long long)blocks * Q;
  k_dd_tiles<<<(unsigned)((n3 + 127) / 128), 128, 0, s>>>(g, d, npc, ddf, spk, sepd, omega, ffd,
                                                          fbd, spt, sept);
  e = cudaStreamSynchronize(s);
  cudaFree(ddf);
  cudaFree(spk);
  cudaFree(sepd);
  cudaFree(scr);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace gq
