// Lean grid stencils for n = 2 (the headline block size): y = Delta x (+ y.x, curvature) and
// the outer-sweep right-hand side y = r + Xi~ x.
//
// Mapping (unchanged from the v2 stencil): a warp owns one grid column j, 30 useful stages
// (lanes 1..30; lanes 0 and 31 are the t-1 / t+1 halo of the Xi coupling, exchanged by
// shuffles) and walks a strip of rows.  Per row-step it needs five NEW x records (column j
// row i+2, columns j+-1 row i+1, columns j+-2 row i); the rest of the 13-point diamond is a
// register window.  The window lives in three 5-entry register rings (columns j-1, j, j+1)
// and the row loop is unrolled by 5, so sliding the window is pure register renaming.
//
// The five records and the node's operator row (Psi 13 | Xi 5 | Xi' 5 blocks, warp-uniform,
// one or two stage classes) are staged by cp.async P rows ahead into a per-warp shared ring;
// operators are read back as broadcast LDS.128.  Accumulation is split over four partial
// sums so the 92 DFMAs of a row-step form short dependency chains.
//
// Reference: gridlq/operators.py (apply_delta), nested_jacobi.py:119-121 (outer rhs).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "gq_async.cuh"
#include "gq_internal.h"

namespace gq {

using namespace as;

template <int MODE>
struct Gd {
  static constexpr int B2 = 4;
  static constexpr int OPOFF = MODE == kDelta ? 0 : 13 * B2;  // doubles into an oprow
  static constexpr int OPN = 23 * B2 - OPOFF;                   // doubles staged per class
  static constexpr int OPC = OPN / 2;                           // 16-byte chunks
  static constexpr int OPI = (OPC + 31) / 32;                   // copy instructions per class
  static constexpr int OPS = OPI * 64;                          // doubles reserved per class
  static constexpr int NREC = MODE == kDelta ? 5 : 4;           // new records per row-step
  static constexpr int REC = 64;                                // 32 lanes x 2 doubles
  static constexpr int SLOT = NREC * REC + 2 * OPS;
};

// acc += M x for a 2x2 row-major block at p (broadcast shared loads)
__device__ __forceinline__ void mac2(double2& acc, const double* p, double2 x) {
  const double2 m0 = lds2(p), m1 = lds2(p + 2);
  acc.x = fma(m0.x, x.x, acc.x);
  acc.y = fma(m1.x, x.x, acc.y);
  acc.x = fma(m0.y, x.y, acc.x);
  acc.y = fma(m1.y, x.y, acc.y);
}

__device__ bool warp_grid_sum2(double v, double* partials, unsigned int* counter, double& out) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int last = 0;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return false;
  __threadfence();
  double acc = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) acc += __ldcg(partials + b);
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  out = acc;
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

template <int MODE, int P>
__device__ __forceinline__ void grid_body(const Geo& g, const FastOps& fo,
                                          const double* __restrict__ x,
                                          const double* __restrict__ rin,
                                          double* __restrict__ y, int nchunk, int nstrip,
                                          int rows, int n_items, double* partials,
                                          PcgState* st, int dotmode) {
  using C = Gd<MODE>;
  constexpr int R = P + 1, REC = C::REC, OPS = C::OPS;
  extern __shared__ __align__(128) double ring[];
  if (st != nullptr) {
    if (dotmode == kDotStep) {
      const bool stop = st->done || st->step >= st->max_steps;
      if (blockIdx.x == 0 && threadIdx.x == 0) st->skip = stop ? 1 : 0;
      if (stop) return;
    } else if (halted(st)) {
      return;
    }
  }
  const int lane = threadIdx.x;
  const uint64_t pol_s = pol_first(), pol_k = pol_last();
  const unsigned ring_u = lane_opaque(smem_u32(ring) + 16 * lane) - 16 * lane;
  double dot = 0.0;
#pragma unroll 1
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
  const int strip = item % nstrip;
  const int rest = item / nstrip;
  const int chunk = rest % nchunk;
  const int j = rest / nchunk;
  const int K = g.K;
  const int t = chunk * kHaloChunk + lane - 1;
  const bool tv = t >= 0 && t < g.T1;
  const bool useful = tv && lane >= 1 && lane <= kHaloChunk &&
                      (MODE != kDelta || slab_owned(g, t));
  const unsigned vmask = __ballot_sync(0xffffffffu, tv);
  const int pc = tv ? fo.psi_cls[t] : 0;
  const int cA = __shfl_sync(0xffffffffu, pc, vmask ? __ffs(vmask) - 1 : 0);
  const int cB = __shfl_sync(0xffffffffu, pc, vmask ? 31 - __clz(vmask) : 0);
  const bool two = cA != cB;
  const int psel = (tv && pc != cA) ? 1 : 0;
  const bool ke = tv && t < g.T;    // e_t exists (Xi_t, t < T)
  const bool kf = tv && t >= 1;     // f_t exists (Xi_{t-1})
  const bool ku = t >= 1;           // receives e_{t-1}
  const bool kd = t < g.T;          // receives f_{t+1}
  const long long rs = (long long)g.TS * 2;
  const long long cs = (long long)K * rs;
  const long long toff = (long long)(tv ? t : 0) * 2;
  auto colp = [&](const double* base, int jj) { return base + (long long)jj * cs + toff; };
  const bool okm1 = tv && j >= 1, okp1 = tv && j + 1 < g.N;
  const bool okm2 = tv && j >= 2, okp2 = tv && j + 2 < g.N;
  const double* xj = colp(x, j);
  const double* xm1 = okm1 ? colp(x, j - 1) : x;
  const double* xp1 = okp1 ? colp(x, j + 1) : x;
  const double* xm2 = okm2 ? colp(x, j - 2) : x;
  const double* xp2 = okp2 ? colp(x, j + 2) : x;
  const double* rj = MODE == kOuterRhs ? colp(rin, j) : x;
  const double* opA = fo.oprow + ((long long)cA * g.nk + (long long)j * K) * 23 * 4 + C::OPOFF;
  const double* opB = fo.oprow + ((long long)cB * g.nk + (long long)j * K) * 23 * 4 + C::OPOFF;

  const int i0 = strip * rows;
  const int i1 = min(K, i0 + rows);

  // records of row-step ii -> ring slot
  auto issue = [&](int ii, int slot) {
    const unsigned so = lane_opaque((unsigned)(slot * C::SLOT * 8));
    const unsigned sb = ring_u + so + lane * 16;
    if (MODE == kDelta) {
      const bool r2 = ii + 2 < K, r1 = ii + 1 < K;
      ldgsts(sb + 0 * REC * 8, (tv && r2) ? xj + (ii + 2) * rs : x, (tv && r2) ? 16 : 0, pol_s);
      ldgsts(sb + 1 * REC * 8, (okm1 && r1) ? xm1 + (ii + 1) * rs : x, (okm1 && r1) ? 16 : 0, pol_s);
      ldgsts(sb + 2 * REC * 8, (okp1 && r1) ? xp1 + (ii + 1) * rs : x, (okp1 && r1) ? 16 : 0, pol_s);
      ldgsts(sb + 3 * REC * 8, okm2 ? xm2 + ii * rs : x, okm2 ? 16 : 0, pol_s);
      ldgsts(sb + 4 * REC * 8, okp2 ? xp2 + ii * rs : x, okp2 ? 16 : 0, pol_s);
    } else {
      const bool r1 = ii + 1 < K;
      ldgsts(sb + 0 * REC * 8, (tv && r1) ? xj + (ii + 1) * rs : x, (tv && r1) ? 16 : 0, pol_s);
      ldgsts(sb + 1 * REC * 8, okm1 ? xm1 + ii * rs : x, okm1 ? 16 : 0, pol_s);
      ldgsts(sb + 2 * REC * 8, okp1 ? xp1 + ii * rs : x, okp1 ? 16 : 0, pol_s);
      ldgsts(sb + 3 * REC * 8, tv ? rj + ii * rs : x, tv ? 16 : 0, pol_s);
    }
    const unsigned ob = ring_u + so + (unsigned)(C::NREC * REC * 8);
    // every lane issues OPI copies per class (chunks past the row zero-fill the padding):
    // no guard predicates on LDGSTS
    const double* oa = opA + (long long)ii * 92;
#pragma unroll
    for (int u = 0; u < C::OPI; ++u) {
      const bool in = 32 * u + lane < C::OPC;
      ldgsts(ob + (32 * u + lane) * 16, in ? oa + 2 * (32 * u + lane) : oa, in ? 16 : 0, pol_k);
    }
    if (two) {
      const double* ob2 = opB + (long long)ii * 92;
#pragma unroll
      for (int u = 0; u < C::OPI; ++u) {
        const bool in = 32 * u + lane < C::OPC;
        ldgsts(ob + OPS * 8 + (32 * u + lane) * 16, in ? ob2 + 2 * (32 * u + lane) : ob2,
               in ? 16 : 0, pol_k);
      }
    }
  };
  auto ldx = [&](const double* base, bool ok, int row) -> double2 {
    if (ok && row >= 0 && row < K) return __ldg(reinterpret_cast<const double2*>(base + row * rs));
    return make_double2(0.0, 0.0);
  };

  // register windows: entry (r - i0 + 2) % 5 holds row r
  double2 X[5], W[5], E[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) X[q] = W[q] = E[q] = make_double2(0.0, 0.0);
  if (i0 < i1) {
    if (MODE == kDelta) {
      X[0] = ldx(xj, tv, i0 - 2);
      X[1] = ldx(xj, tv, i0 - 1);
      X[2] = ldx(xj, tv, i0);
      X[3] = ldx(xj, tv, i0 + 1);
      W[1] = ldx(xm1, okm1, i0 - 1);
      W[2] = ldx(xm1, okm1, i0);
      E[1] = ldx(xp1, okp1, i0 - 1);
      E[2] = ldx(xp1, okp1, i0);
    } else {
      X[1] = ldx(xj, tv, i0 - 1);
      X[2] = ldx(xj, tv, i0);
    }
    const int pro = min(P, i1 - i0);
#pragma unroll 1
    for (int p = 0; p < pro; ++p) {
      issue(i0 + p, p);
      commit();
    }
#pragma unroll 1
    for (int p = pro; p < P; ++p) commit();
  }
  int cslot = 0, islot = P % R;
  double* yj = y + (long long)j * cs + toff;

  // one row-step; S = (i - i0) % 5 is static so every window index is a register name
  auto stepS = [&](auto Sc, int i) {
    constexpr int S = decltype(Sc)::value;
    if (i + P < i1) issue(i + P, islot);
    commit();
    islot = islot + 1 == R ? 0 : islot + 1;
    wait_groups<P>();
    __syncwarp();
    const double* sl = ring + cslot * C::SLOT;
    cslot = cslot + 1 == R ? 0 : cslot + 1;
    const double* op = sl + C::NREC * REC + psel * OPS;
    double2 x0 = X[(S + 2) % 5];                   // self
    double2 eacc = make_double2(0.0, 0.0), facc = eacc;
    double2 acc = eacc;
    if (MODE == kDelta) {
      X[(S + 4) % 5] = lds2(sl + 0 * REC + 2 * lane);   // col j,   row i+2
      W[(S + 3) % 5] = lds2(sl + 1 * REC + 2 * lane);   // col j-1, row i+1
      E[(S + 3) % 5] = lds2(sl + 2 * REC + 2 * lane);   // col j+1, row i+1
      const double2 xmm = lds2(sl + 3 * REC + 2 * lane);
      const double2 xpp = lds2(sl + 4 * REC + 2 * lane);
      const double2 xn = X[(S + 1) % 5], xs = X[(S + 3) % 5];
      const double2 xw = W[(S + 2) % 5], xe = E[(S + 2) % 5];
      double2 a1 = eacc, a2 = eacc, a3 = eacc;
      mac2(acc, op + 0 * 4, x0);
      mac2(a1, op + 1 * 4, xn);
      mac2(a2, op + 2 * 4, xs);
      mac2(a3, op + 3 * 4, xw);
      mac2(acc, op + 4 * 4, xe);
      mac2(a1, op + 5 * 4, X[S % 5]);               // (-2, 0)
      mac2(a2, op + 6 * 4, X[(S + 4) % 5]);         // (+2, 0)
      mac2(a3, op + 7 * 4, xmm);                    // (0, -2)
      mac2(acc, op + 8 * 4, xpp);                   // (0, +2)
      mac2(a1, op + 9 * 4, W[(S + 1) % 5]);         // (-1, -1)
      mac2(a2, op + 10 * 4, E[(S + 1) % 5]);        // (-1, +1)
      mac2(a3, op + 11 * 4, W[(S + 3) % 5]);        // (+1, -1)
      mac2(acc, op + 12 * 4, E[(S + 3) % 5]);       // (+1, +1)
      acc = add2(add2(acc, a1), add2(a2, a3));
      const double* xo = op + 13 * 4;
      double2 e1 = eacc, f1 = eacc;
      mac2(eacc, xo + 0 * 4, x0);
      mac2(e1, xo + 1 * 4, xn);
      mac2(eacc, xo + 2 * 4, xs);
      mac2(e1, xo + 3 * 4, xw);
      mac2(eacc, xo + 4 * 4, xe);
      mac2(facc, xo + 5 * 4, x0);
      mac2(f1, xo + 6 * 4, xn);
      mac2(facc, xo + 7 * 4, xs);
      mac2(f1, xo + 8 * 4, xw);
      mac2(facc, xo + 9 * 4, xe);
      eacc = add2(eacc, e1);
      facc = add2(facc, f1);
    } else {
      X[(S + 3) % 5] = lds2(sl + 0 * REC + 2 * lane);   // col j, row i+1
      const double2 xw = lds2(sl + 1 * REC + 2 * lane);
      const double2 xe = lds2(sl + 2 * REC + 2 * lane);
      const double2 rv = lds2(sl + 3 * REC + 2 * lane);
      const double2 xn = X[(S + 1) % 5], xs = X[(S + 3) % 5];
      double2 e1 = eacc, f1 = eacc;
      mac2(eacc, op + 0 * 4, x0);
      mac2(e1, op + 1 * 4, xn);
      mac2(eacc, op + 2 * 4, xs);
      mac2(e1, op + 3 * 4, xw);
      mac2(eacc, op + 4 * 4, xe);
      mac2(facc, op + 5 * 4, x0);
      mac2(f1, op + 6 * 4, xn);
      mac2(facc, op + 7 * 4, xs);
      mac2(f1, op + 8 * 4, xw);
      mac2(facc, op + 9 * 4, xe);
      eacc = add2(eacc, e1);
      facc = add2(facc, f1);
      acc = rv;
    }
    if (!ke) eacc = make_double2(0.0, 0.0);
    if (!kf) facc = make_double2(0.0, 0.0);
    double2 eu, fd;
    eu.x = __shfl_up_sync(0xffffffffu, eacc.x, 1);
    eu.y = __shfl_up_sync(0xffffffffu, eacc.y, 1);
    fd.x = __shfl_down_sync(0xffffffffu, facc.x, 1);
    fd.y = __shfl_down_sync(0xffffffffu, facc.y, 1);
    if (!ku) eu = make_double2(0.0, 0.0);
    if (!kd) fd = make_double2(0.0, 0.0);
    if (MODE == kDelta) {
      acc.x = (acc.x + eu.x) + fd.x;
      acc.y = (acc.y + eu.y) + fd.y;
    } else {   // y = r + (-(Xi_{t-1} x_{t-1}) - Xi_t' x_{t+1})
      acc.x = acc.x + ((0.0 - eu.x) - fd.x);
      acc.y = acc.y + ((0.0 - eu.y) - fd.y);
    }
    if (useful) {
      *reinterpret_cast<double2*>(yj + (long long)i * rs) = acc;
      if (MODE == kDelta && dotmode != kDotNone) {
        dot = fma(acc.x, x0.x, dot);
        dot = fma(acc.y, x0.y, dot);
      }
    }
    __syncwarp();
  };
#pragma unroll 1
  for (int i = i0; i < i1; i += 5) {
    stepS(std::integral_constant<int, 0>{}, i);
    if (i + 1 < i1) stepS(std::integral_constant<int, 1>{}, i + 1);
    if (i + 2 < i1) stepS(std::integral_constant<int, 2>{}, i + 2);
    if (i + 3 < i1) stepS(std::integral_constant<int, 3>{}, i + 3);
    if (i + 4 < i1) stepS(std::integral_constant<int, 4>{}, i + 4);
  }
  wait_groups<0>();
  __syncwarp();
  }
  if (MODE == kDelta && dotmode != kDotNone) {
    double c;
    if (warp_grid_sum2(dot, partials, &st->counter[0], c) && threadIdx.x == 0) {
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

template <int MODE, int P>
__global__ void __launch_bounds__(32) k_grid(Geo g, FastOps fo, const double* __restrict__ x,
                                             const double* __restrict__ rin,
                                             double* __restrict__ y, int nchunk, int nstrip,
                                             int rows, int n_items, double* partials,
                                             PcgState* st, int dotmode) {
  grid_body<MODE, P>(g, fo, x, rin, y, nchunk, nstrip, rows, n_items, partials, st, dotmode);
}

// register-capped build (GQ_GRID_MAXR, default 128 for Delta): more resident warps per SM
template <int MODE, int P, int MAXR>
__global__ void __maxnreg__(MAXR) k_grid_r(Geo g, FastOps fo, const double* __restrict__ x,
                                           const double* __restrict__ rin,
                                           double* __restrict__ y, int nchunk, int nstrip,
                                           int rows, int n_items, double* partials,
                                           PcgState* st, int dotmode) {
  grid_body<MODE, P>(g, fo, x, rin, y, nchunk, nstrip, rows, n_items, partials, st, dotmode);
}

// ---- host side -----------------------------------------------------------------------------

static int genv(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

bool grid_supported(int n) { return n == 2 && genv("GQ_NO_GRID", 0) == 0; }

GridShape grid_shape(const Geo& g, int sm_count) {
  // upper bound (partials sizing); the launch picks the strip count per kernel occupancy
  GridShape sh;
  sh.nchunk = (g.T1 + kHaloChunk - 1) / kHaloChunk;
  sh.nstrip = std::max(1, std::min(8, g.K / 8));
  sh.rows = (g.K + sh.nstrip - 1) / sh.nstrip;
  sh.blocks = (int)std::min<long long>((long long)g.N * sh.nchunk * sh.nstrip, 32LL * sm_count);
  return sh;
}

template <int MODE, int P, int MAXR = 0>
static cudaError_t grid_launch(const Geo& g, const FastOps& fo, const double* x, const double* rin,
                               double* y, const GridShape& ub, double* partials, PcgState* st,
                               int dotmode, cudaStream_t s) {
  constexpr size_t smem = (size_t)(P + 1) * Gd<MODE>::SLOT * sizeof(double);
  static int cache[64] = {0};
  int per_sm = 1;
  cudaError_t e;
  if constexpr (MAXR > 0)
    e = kernel_occupancy(k_grid_r<MODE, P, MAXR>, 32, smem, cache, per_sm);
  else
    e = kernel_occupancy(k_grid<MODE, P>, 32, smem, cache, per_sm);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // equal-cost items (column, 30-stage chunk, row strip) on a persistent grid: pick the
  // strip count that minimises waves x (rows per strip + window warm-up)
  const long long cols = (long long)g.N * ub.nchunk;
  const long long slots = (long long)per_sm * sms;
  int best = 1;
  long long best_cost = -1;
  for (int ns = 1; ns <= ub.nstrip; ++ns) {
    const int rows = (g.K + ns - 1) / ns;
    const long long items = cols * ((g.K + rows - 1) / rows);
    const long long cost = ((items + slots - 1) / slots) * (rows + 4);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = ns;
    }
  }
  const int rows = (g.K + best - 1) / best;
  const int nstrip = (g.K + rows - 1) / rows;
  const int n_items = (int)(cols * nstrip);
  const int blocks = (int)std::min<long long>({(long long)n_items, slots, (long long)ub.blocks});
  if constexpr (MAXR > 0)
    k_grid_r<MODE, P, MAXR><<<blocks, 32, smem, s>>>(
        g, fo, x, rin, y, ub.nchunk, nstrip, rows, n_items, partials, st, dotmode);
  else
    k_grid<MODE, P><<<blocks, 32, smem, s>>>(g, fo, x, rin, y, ub.nchunk, nstrip, rows, n_items,
                                             partials, st, dotmode);
  return cudaGetLastError();
}

cudaError_t launch_grid(const Geo& g, const FastOps& fo, int mode, const double* x,
                        const double* rin, double* y, const GridShape& sh, double* partials,
                        PcgState* st, int dotmode, cudaStream_t s) {
  // ring depth P = 2 for both modes (round 1 sweeps: Delta P 3 / 4 and outer-rhs P 1 / 3 / 4 / 6
  // were slower or equal).  Delta capped at 128 registers (from 136): 16 resident warps per
  // SM, 592.6 -> 600.1 steps/s.
  if (mode == kDelta)
    return grid_launch<kDelta, 2, 128>(g, fo, x, rin, y, sh, partials, st, dotmode, s);
  return grid_launch<kOuterRhs, 2>(g, fo, x, rin, y, sh, partials, st, kDotNone, s);
}

}  // namespace gq
