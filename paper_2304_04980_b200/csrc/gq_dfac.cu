// Factored Delta apply for time-invariant problems, n = 2 ("dfac" kernel).
//
// The reference assembles Psi_t / Xi_t (kkt_assembly.py:487-544) and applies the 23-block
// stencil (Delta x)_t = Psi_t x_t + Xi_{t-1} x_{t-1} + Xi_t' x_{t+1} (kkt_assembly.py:389-403).
// With Psi_t = Q^-1 + Ahat Q^-1 Ahat' + B R^-1 B' (t >= 1), Psi_0 = Q^-1 and Xi_t = -Ahat Q^-1
// the same product factors as
//
//     w_t = Q^-1 (x_t - Ahat' x_{t+1})                   (w_T = Q^-1 x_T)
//     (Delta x)_t = w_t - Ahat w_{t-1} + B R^-1 B' x_t   ((Delta x)_0 = w_0)
//
// i.e. two 5-point stencils and two block-diagonal products: 48 multiply-adds per node-stage
// instead of 92, with 48 operator doubles per node instead of 92.  The catch is that the
// output of column j needs w of columns j-1 and j+1, so w is shared through shared memory:
// a CTA of NW warps owns NW adjacent columns (one per warp, lane = stage, 30 useful stages
// per 32 lanes as in gq_grid.cu), computes w for all of them and Delta x for the NW-2 inner
// ones, walking a strip of rows with ONE barrier per row step:
//
//   step s:  wait x/op row s; barrier; issue row s+P (cp.async); w(s-1) -> smem; y(s-3).
//
// The x ring holds NW+2 columns (the edge warps also stage the outer columns) and RX = P+4
// rows; w has a 4-row ring.  The shifts in t are lane shuffles: u = Ahat' x at the lane's own
// stage, shuffled down; v = Ahat w at the lane's own stage, shuffled up.  Rounding differs from
// the assembled operator at the 1e-16 level (the reference symmetrises Psi's diagonal blocks).
#include <algorithm>
#include <cstdlib>

#include "gq_async.cuh"
#include "gq_internal.h"

namespace gq {

namespace {

using namespace as;

constexpr int kRec = 48;   // op record doubles: row blocks (5x4) | col blocks^T (5x4) | Qinv | BRB

// acc += M x, M 2x2 row-major in shared memory (broadcast loads)
__device__ __forceinline__ void mv2(double2& acc, const double* m, double2 x) {
  const double2 r0 = lds2(m), r1 = lds2(m + 2);
  acc.x = fma(r0.x, x.x, acc.x);
  acc.y = fma(r1.x, x.x, acc.y);
  acc.x = fma(r0.y, x.y, acc.x);
  acc.y = fma(r1.y, x.y, acc.y);
}

}  // namespace

template <int NW, int P>
__global__ void __launch_bounds__(32 * NW) k_dfac(Geo g, const double* __restrict__ ops,
                                                  const double* __restrict__ x,
                                                  double* __restrict__ y, int ngrp, int nchunk,
                                                  int nstrip, int rows, int n_items,
                                                  double* partials, PcgState* st, int dotmode) {
  constexpr int RX = P + 4;            // x / op ring rows
  constexpr int XC = NW + 2;           // staged x columns
  constexpr int W = NW - 2;            // output columns per CTA
  extern __shared__ __align__(16) double sm[];
  double* xs = sm;                                   // [RX][XC][32][2]
  double* os = xs + RX * XC * 64;                    // [RX][NW][48]
  double* ws = os + RX * NW * kRec;                  // [4][NW][32][2]
  if (st != nullptr) {
    if (dotmode == kDotStep) {
      const bool stop = st->done || st->step >= st->max_steps;
      if (blockIdx.x == 0 && threadIdx.x == 0) st->skip = stop ? 1 : 0;
      if (stop) return;
    } else if (halted(st)) {
      return;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = g.K, N = g.N;
  const long long rs = (long long)g.T1 * 2, cs = (long long)K * rs;
  double dot = 0.0;
  const unsigned xs_u = smem_u32(xs), os_u = smem_u32(os);

#pragma unroll 1
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int strip = item % nstrip;
    const int rest = item / nstrip;
    const int chunk = rest % nchunk;
    const int grp = rest / nchunk;
    const int j0 = grp * W;                 // first output column
    const int q = j0 - 1 + warp;            // my column
    const int t = chunk * kHaloChunk + lane - 1;
    const bool tv = t >= 0 && t < g.T1;
    const bool useful = tv && lane >= 1 && lane <= kHaloChunk;
    const bool out_col = warp >= 1 && warp <= W && q < N;
    const long long toff = (long long)(tv ? t : 0) * 2;
    const int i0 = strip * rows, i1 = min(K, i0 + rows);
    // staged x columns for this warp: its own (slot warp+1) and, for the edge warps, the
    // outer one (slot 0 / XC-1)
    const int xq0 = q, xs0 = warp + 1;
    const int xq1 = warp == 0 ? q - 1 : (warp == NW - 1 ? q + 1 : -1);
    const int xs1 = warp == 0 ? 0 : XC - 1;
    const bool ok0 = tv && xq0 >= 0 && xq0 < N;
    const bool ok1 = tv && xq1 >= 0 && xq1 < N;
    const double* xb0 = ok0 ? x + (long long)xq0 * cs + toff : x;
    const double* xb1 = ok1 ? x + (long long)xq1 * cs + toff : x;
    const bool opq = q >= 0 && q < N;
    const double* ob = ops + (long long)(opq ? q : 0) * K * kRec;

    auto issue = [&](int r) {
      const int slot = ((r % RX) + RX) % RX;
      const bool rok = r >= 0 && r < K;
      const unsigned xd = xs_u + (unsigned)(((slot * XC + xs0) * 32 + lane) * 16);
      ldgsts(lane_opaque(xd), (ok0 && rok) ? xb0 + (long long)r * rs : x, (ok0 && rok) ? 16 : 0, 0);
      if (warp == 0 || warp == NW - 1) {
        const unsigned xd1 = xs_u + (unsigned)(((slot * XC + xs1) * 32 + lane) * 16);
        ldgsts(lane_opaque(xd1), (ok1 && rok) ? xb1 + (long long)r * rs : x,
               (ok1 && rok) ? 16 : 0, 0);
      }
      // lane_opaque is a full-warp shuffle: compute it on every lane, copy on lanes < 24
      const int ol = lane < kRec / 2 ? lane : 0;
      const unsigned od = lane_opaque(os_u + (unsigned)(((slot * NW + warp) * kRec + 2 * ol) * 8));
      if (lane < kRec / 2) {
        const bool ook = opq && rok;
        ldgsts(od, ook ? ob + (long long)r * kRec + 2 * lane : ops, ook ? 16 : 0, 0);
      }
    };
    auto xat = [&](int r, int col_slot) -> double2 {
      const int slot = ((r % RX) + RX) % RX;
      return lds2(xs + ((slot * XC + col_slot) * 32 + lane) * 2);
    };
    auto opat = [&](int r) -> const double* {
      const int slot = ((r % RX) + RX) % RX;
      return os + (slot * NW + warp) * kRec;
    };
    auto wat = [&](int r, int w_) -> double2 {
      return lds2(ws + (((r & 3) * NW + w_) * 32 + lane) * 2);
    };

    // prologue: rows i0-2 .. i0+P-1
    __syncthreads();   // the previous item's readers are done with the rings
#pragma unroll 1
    for (int r = i0 - 2; r < i0 + P; ++r) {
      issue(r);
      commit();
    }

#pragma unroll 1
    for (int s = i0; s <= i1 + 2; ++s) {
      wait_groups<P - 1>();
      __syncthreads();
      issue(s + P);
      commit();
      // ---- w(s-1): all columns ----
      if (s - 1 <= i1) {
        const int r = s - 1;
        const double* op = opat(r);
        const double2 xc = xat(r, xs0);
        double2 u0 = make_double2(0.0, 0.0), u1 = u0;
        mv2(u0, op + 20 + 0 * 4, xc);              // A(q)' x(q)
        mv2(u1, op + 20 + 1 * 4, xat(r - 1, xs0));  // from the north neighbour
        mv2(u0, op + 20 + 2 * 4, xat(r + 1, xs0));  // from the south neighbour
        mv2(u1, op + 20 + 3 * 4, xat(r, xs0 - 1));  // from the west neighbour
        mv2(u0, op + 20 + 4 * 4, xat(r, xs0 + 1));  // from the east neighbour
        const double2 u = add2(u0, u1);
        double2 ud;
        ud.x = __shfl_down_sync(0xffffffffu, u.x, 1);
        ud.y = __shfl_down_sync(0xffffffffu, u.y, 1);
        const double2 z = make_double2(xc.x - ud.x, xc.y - ud.y);
        double2 w = make_double2(0.0, 0.0);
        mv2(w, op + 40, z);                          // Q^-1 z
        if (!tv) w = make_double2(0.0, 0.0);
        *reinterpret_cast<double2*>(ws + (((r & 3) * NW + warp) * 32 + lane) * 2) = w;
      }
      // ---- y(s-3): inner columns; needs w rows s-4..s-2 (written in earlier steps) ----
      const int p = s - 3;
      if (p >= i0 && p < i1 && out_col) {
        const double* op = opat(p);
        const double2 wc = wat(p, warp);
        double2 v0 = make_double2(0.0, 0.0), v1 = v0;
        mv2(v0, op + 0 * 4, wc);                   // Ahat(p,p) w(p)
        mv2(v1, op + 1 * 4, wat(p - 1, warp));      // north
        mv2(v0, op + 2 * 4, wat(p + 1, warp));      // south
        mv2(v1, op + 3 * 4, wat(p, warp - 1));      // west
        mv2(v0, op + 4 * 4, wat(p, warp + 1));      // east
        const double2 v = add2(v0, v1);
        double2 vu;
        vu.x = __shfl_up_sync(0xffffffffu, v.x, 1);
        vu.y = __shfl_up_sync(0xffffffffu, v.y, 1);
        double2 acc = make_double2(wc.x - vu.x, wc.y - vu.y);
        const double2 xp = xat(p, xs0);
        if (t >= 1) mv2(acc, op + 44, xp);         // B R^-1 B' x (stages t >= 1)
        if (useful) {
          *reinterpret_cast<double2*>(y + (long long)q * cs + (long long)p * rs + toff) = acc;
          if (dotmode != kDotNone) {
            dot = fma(acc.x, xp.x, dot);
            dot = fma(acc.y, xp.y, dot);
          }
        }
      }
    }
    wait_groups<0>();
  }
  if (dotmode != kDotNone) {
    double c;
    if (grid_reduce<false>(dot, partials, &st->counter[0], c) && threadIdx.x == 0) {
      st->curv = c;                        // pcg.py:101-108
      if (c <= 0.0) {
        st->breakdown = 1;
        st->done = 1;
      } else {
        st->alpha = st->mu / c;
      }
    }
  }
}

// ---- setup: per-node operator records (one dynamics set, one cost set) ----------------------
// rec[j][i] = Ahat row blocks (self, N, S, W, E) | Ahat column blocks transposed, i.e. the
// blocks A(s, q)' of the neighbours s that multiply x(q) (self, N, S, W, E) | Qinv | B R^-1 B'
__global__ void k_build_dfac(Geo g, const double* __restrict__ A, const double* __restrict__ C,
                             const double* __restrict__ qinv, const double* __restrict__ brb,
                             double* __restrict__ rec) {
  const long long node = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= g.nk) return;
  const int j = (int)(node / g.K), i = (int)(node % g.K);
  double* o = rec + node * kRec;
  // Ahat(j, i, u): u = 0 self, 1 north, 2 south, 3 west, 4 east (gq_setup.cu ahat)
  auto ahat = [&](int jj, int ii, int u, double* b) {
    const int j2 = jj + odj(u), i2 = ii + odi(u);
    const bool in = jj >= 0 && jj < g.N && ii >= 0 && ii < g.K && j2 >= 0 && j2 < g.N &&
                    i2 >= 0 && i2 < g.K;
    const long long nd = (long long)jj * g.K + ii;
    for (int e = 0; e < 4; ++e)
      b[e] = !in ? 0.0 : (u == 0 ? A[nd * 4 + e] : C[((long long)slot_dir(u) * g.nk + nd) * 4 + e]);
  };
  for (int u = 0; u < 5; ++u) {
    double b[4];
    ahat(j, i, u, b);
    for (int e = 0; e < 4; ++e) o[u * 4 + e] = b[e];
    // the neighbour s = (i, j) + off(u) multiplies x(i, j) with its block toward slot opp(u)
    ahat(j + odj(u), i + odi(u), slot_opp(u), b);
    o[20 + u * 4 + 0] = b[0];
    o[20 + u * 4 + 1] = b[2];
    o[20 + u * 4 + 2] = b[1];
    o[20 + u * 4 + 3] = b[3];
  }
  for (int e = 0; e < 4; ++e) o[40 + e] = qinv[node * 4 + e];
  for (int e = 0; e < 4; ++e) o[44 + e] = brb[node * 4 + e];
}

// ---- host side -----------------------------------------------------------------------------

static int denv(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

// opt-in (GQ_DFAC=1): parity-green, but at the headline it measured 592-594 steps/s against
// 595 with the assembled-operator grid stencil (tools/steptime.py)
bool dfac_supported(const Geo& g, int n_dyn, int n_cost) {
  return g.n == 2 && n_dyn == 1 && n_cost == 1 && g.T1 >= 2 && denv("GQ_DFAC", 0) == 1;
}

cudaError_t launch_build_dfac(const Geo& g, const double* A, const double* C, const double* qinv,
                              const double* brb, double* rec, cudaStream_t s) {
  k_build_dfac<<<(unsigned)((g.nk + 127) / 128), 128, 0, s>>>(g, A, C, qinv, brb, rec);
  return cudaGetLastError();
}

template <int NW, int P>
static cudaError_t dfac_launch(const Geo& g, const double* ops, const double* x, double* y,
                               double* partials, PcgState* st, int dotmode, int sm_count,
                               cudaStream_t s) {
  constexpr int RX = P + 4, XC = NW + 2;
  constexpr size_t smem = (size_t)(RX * XC * 64 + RX * NW * kRec + 4 * NW * 64) * sizeof(double);
  static int cache[64] = {0};
  int per_sm = 1;
  cudaError_t e = kernel_occupancy(k_dfac<NW, P>, 32 * NW, smem, cache, per_sm);
  if (e != cudaSuccess) return e;
  const int W = NW - 2;
  const int ngrp = (g.N + W - 1) / W;
  const int nchunk = (g.T1 + kHaloChunk - 1) / kHaloChunk;
  // strips: enough items for every resident CTA, strips of at least 24 rows
  const long long slots = (long long)per_sm * sm_count;
  const long long base = (long long)ngrp * nchunk;
  int nstrip = (int)std::max<long long>(1, std::min<long long>((slots + base - 1) / base, g.K / 24));
  nstrip = std::max(1, denv("GQ_DFAC_STRIPS", nstrip));
  const int rows = (g.K + nstrip - 1) / nstrip;
  nstrip = (g.K + rows - 1) / rows;
  const int n_items = (int)(base * nstrip);
  const int blocks = (int)std::min<long long>(n_items, slots);
  k_dfac<NW, P><<<blocks, 32 * NW, smem, s>>>(g, ops, x, y, ngrp, nchunk, nstrip, rows, n_items,
                                             partials, st, dotmode);
  return cudaGetLastError();
}

cudaError_t launch_dfac(const Geo& g, const double* ops, const double* x, double* y,
                        double* partials, PcgState* st, int dotmode, int sm_count, cudaStream_t s) {
  const int nw = denv("GQ_DFAC_NW", 8);
  if (nw == 16) return dfac_launch<16, 2>(g, ops, x, y, partials, st, dotmode, sm_count, s);
  if (nw == 6) return dfac_launch<6, 2>(g, ops, x, y, partials, st, dotmode, sm_count, s);
  return dfac_launch<8, 2>(g, ops, x, y, partials, st, dotmode, sm_count, s);
}

long long dfac_max_blocks(int sm_count) { return 32LL * sm_count; }

}  // namespace gq
