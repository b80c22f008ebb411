// Block stencils for n = 2 on the fp64 tensor cores, 2 x 2 node groups ("st2" kernels).
//
// Same operators as gq_grid.cu / gq_stencil.cu (kkt_assembly.py:379-425):
//   Delta:      (Delta x)_t = Psi_t x_t + Xi_{t-1} x_{t-1} + Xi_t' x_{t+1}
//   outer rhs:  y_t = r_t - (Xi_{t-1} x_{t-1} + Xi_t' x_{t+1})
// A warp owns one 2 x 2 group of nodes (rows 2kb, 2kb+1 of columns 2v, 2v+1 -- the pair-chain
// blocks) and walks its class-pure stage chunks (8 stages on M).  The group's 8 outputs
// (4 nodes x 2 states) are one DMMA N-tile; its inputs are the union of the four stencils:
// 24 same-stage nodes (13-point diamonds), 12 nodes at t-1 and 12 at t+1 (5-point), i.e.
// 48 records = 12 k-pairs of 4 records (one per lane quad) x 2 states.  The coefficient
// matrix (96 x 8 per group and stage class, built at setup) lives in registers as 12 B
// fragments; A fragments are single 16-byte loads of the stage-inner records (stage shifted
// by -1 / +1 for the Xi terms), so a chunk is 12 loads and 24 DMMAs for 64 outputs.
#include <algorithm>
#include <cstdlib>

#include "gq_async.cuh"
#include "gq_internal.h"

namespace gq {

namespace {
using namespace as;

// input record r (0..47): (row offset, column offset, stage offset) relative to the group's
// first node (2kb, 2v); k-pair p reads records 4p .. 4p+3 (lane quad qd -> record 4p + qd)
struct Rec3 {
  int di, dj, dt;
};
__host__ __device__ inline Rec3 st2_rec(int r) {
  // same stage: the 4x4 square [-1,2]^2 (16) + the 8 arms
  if (r < 16) return {r / 4 - 1, r % 4 - 1, 0};
  if (r < 24) {
    const int q = r - 16;
    const int di[8] = {-2, -2, 3, 3, 0, 1, 0, 1};
    const int dj[8] = {0, 1, 0, 1, -2, -2, 3, 3};
    return {di[q], dj[q], 0};
  }
  // t -1 (24..35) and t +1 (36..47): the 4x4 square minus its corners
  const int q = (r - 24) % 12;
  const int di[12] = {-1, -1, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2};
  const int dj[12] = {0, 1, -1, 0, 1, 2, -1, 0, 1, 2, 0, 1};
  return {di[q], dj[q], r < 36 ? -1 : 1};
}

__device__ __forceinline__ double2 ld16(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}
}  // namespace

// tiles[(cls, group)][p][o][2 qd + c]: coefficient of output o (node o/2 = 2 dr + dc, state
// o%2) on record 4p + qd, state c.  One thread per (cls, group, o).
__global__ void k_build_st2(Geo g, int npc, Ops op, double* __restrict__ tiles) {
  constexpr int B2 = 4;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long ngrp = (long long)g.V * g.nb;
  if (gid >= (long long)npc * ngrp * 8) return;
  const int o = (int)(gid % 8);
  const long long cg = gid / 8;
  const int pc = (int)(cg / ngrp);
  const long long grp = cg % ngrp;
  const int v = (int)(grp / g.nb), kb = (int)(grp % g.nb);
  const int nd = o / 2, co = o % 2, dr = nd >> 1, dc = nd & 1;
  const int i = 2 * kb + dr, j = 2 * v + dc;
  double* T = tiles + cg * 12 * 64;
  const bool in = i < g.K && j < g.N;
  const long long node = (long long)j * g.K + i;
  for (int r = 0; r < 48; ++r) {
    const Rec3 rc = st2_rec(r);
    const int di = rc.di - dr, dj = rc.dj - dc;
    double cf[2] = {0.0, 0.0};
    if (in) {
      if (rc.dt == 0) {
        for (int oo = 0; oo < 13; ++oo)
          if (odi(oo) == di && odj(oo) == dj) {
            const double* P = op.psi + (((long long)pc * g.nk + node) * 13 + oo) * B2;
            cf[0] = P[co * 2 + 0];
            cf[1] = P[co * 2 + 1];
          }
      } else {
        for (int u = 0; u < 5; ++u)
          if (odi(u) == di && odj(u) == dj) {
            const double* X = (rc.dt < 0 ? op.xi : op.xit) + ((long long)node * 5 + u) * B2;
            cf[0] = X[co * 2 + 0];
            cf[1] = X[co * 2 + 1];
          }
      }
    }
    const int p = r / 4, q = r % 4;
    T[p * 64 + o * 8 + 2 * q + 0] = cf[0];
    T[p * 64 + o * 8 + 2 * q + 1] = cf[1];
  }
}

template <int MODE>
__global__ void __launch_bounds__(32) k_st2(Geo g, const double* __restrict__ tiles,
                                            const int4* __restrict__ seg, int nseg,
                                            const double* __restrict__ x,
                                            const double* __restrict__ rin,
                                            double* __restrict__ y, double* partials,
                                            PcgState* st, int dotmode) {
  constexpr int P0 = MODE == kDelta ? 0 : 6;   // outer rhs: only the t-1 / t+1 k-pairs
  if (st != nullptr) {
    if (dotmode == kDotStep) {
      const bool stop = st->done || st->step >= st->max_steps;
      if (blockIdx.x == 0 && threadIdx.x == 0) st->skip = stop ? 1 : 0;
      if (stop) return;
    } else if (halted(st)) {
      return;
    }
  }
  const int lane = threadIdx.x, rw = lane >> 2, qd = lane & 3;
  const long long rs = (long long)g.T1 * 2, cs = (long long)g.K * rs;
  const long long ngrp = (long long)g.V * g.nb;
  double dot = 0.0;
#pragma unroll 1
  for (long long grp = blockIdx.x; grp < ngrp; grp += gridDim.x) {
    const int v = (int)(grp / g.nb), kb = (int)(grp % g.nb);
    const int i0 = 2 * kb, j0 = 2 * v;
    // my record per k-pair: base pointer (stage 0) and in-grid flag
    const double* rb[12];
    bool rok[12];
    int rdt[12];
#pragma unroll
    for (int p = P0; p < 12; ++p) {
      const Rec3 rc = st2_rec(4 * p + qd);
      const int ii = i0 + rc.di, jj = j0 + rc.dj;
      rok[p] = ii >= 0 && ii < g.K && jj >= 0 && jj < g.N;
      rb[p] = x + (rok[p] ? (long long)jj * cs + (long long)ii * rs : 0);
      rdt[p] = rc.dt;
    }
    // my output node (qd) and its record
    const int oi = i0 + (qd >> 1), oj = j0 + (qd & 1);
    const bool ook = oi < g.K && oj < g.N;
    const long long oofs = (long long)oj * cs + (long long)oi * rs;
    double2 bt[12];
    int cur = -1;
#pragma unroll 1
    for (int sgi = 0; sgi < nseg; ++sgi) {
      const int4 sg = seg[sgi];
      const int t0 = sg.x, nvalid = sg.y, pc = sg.z;
      if (pc != cur) {
        const double* T = tiles + ((long long)pc * ngrp + grp) * 12 * 64 + rw * 8 + 2 * qd;
#pragma unroll
        for (int p = P0; p < 12; ++p) bt[p] = ld16(T + p * 64);
        cur = pc;
      }
      const int t = t0 + rw;
      const bool tv = rw < nvalid;
      double2 acc[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) acc[a] = make_double2(0.0, 0.0);
#pragma unroll
      for (int p = P0; p < 12; ++p) {
        const int ts = t + rdt[p];
        const double2 a = (rok[p] && tv && ts >= 0 && ts < g.T1) ? ld16(rb[p] + (long long)ts * 2)
                                                                : make_double2(0.0, 0.0);
        dmma(acc[p & 3], a.x, bt[p].x);
        dmma(acc[p & 3], a.y, bt[p].y);
      }
      const double2 s = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
      if (tv && ook) {
        double2 out;
        if (MODE == kDelta) {
          out = s;
          if (dotmode != kDotNone) {
            const double2 xs = ld16(x + oofs + (long long)t * 2);
            dot = fma(out.x, xs.x, dot);
            dot = fma(out.y, xs.y, dot);
          }
        } else {   // y = r + (0 - (Xi_{t-1} x_{t-1} + Xi_t' x_{t+1}))
          const double2 rv = ld16(rin + oofs + (long long)t * 2);
          out.x = rv.x + (0.0 - s.x);
          out.y = rv.y + (0.0 - s.y);
        }
        *reinterpret_cast<double2*>(y + oofs + (long long)t * 2) = out;
      }
    }
  }
  if (MODE == kDelta && dotmode != kDotNone) {
#pragma unroll
    for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    int last = 0;
    if (lane == 0) {
      partials[blockIdx.x] = dot;
      __threadfence();
      last = atomicAdd(&st->counter[0], 1u) == gridDim.x - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence();
      double acc = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) acc += __ldcg(partials + b);
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        st->counter[0] = 0u;
        st->curv = acc;                      // pcg.py:101-108
        if (acc <= 0.0) {
          st->breakdown = 1;
          st->done = 1;
        } else {
          st->alpha = st->mu / acc;
        }
      }
    }
  }
}

static int s2env(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

bool st2_supported(const Geo& g, int nxc) {
  return g.n == 2 && nxc == 1 && s2env("GQ_ST2", 0) == 1;
}

size_t st2_doubles(const Geo& g, int npc) { return (size_t)npc * g.V * g.nb * 12 * 64; }

cudaError_t launch_build_st2(const Geo& g, int npc, const Ops& op, double* tiles, cudaStream_t s) {
  const long long n = (long long)npc * g.V * g.nb * 8;
  k_build_st2<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(g, npc, op, tiles);
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t st2_launch(const Geo& g, const double* tiles, const int4* seg, int nseg,
                              const double* x, const double* rin, double* y, int sm_count,
                              double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  static int cache[64] = {0};
  int per_sm = 1;
  cudaError_t e = kernel_occupancy(k_st2<MODE>, 32, 0, cache, per_sm);
  if (e != cudaSuccess) return e;
  const long long blocks = std::min<long long>((long long)g.V * g.nb, (long long)per_sm * sm_count);
  k_st2<MODE><<<(unsigned)blocks, 32, 0, s>>>(g, tiles, seg, nseg, x, rin, y, partials, st, dotmode);
  return cudaGetLastError();
}

cudaError_t launch_st2(const Geo& g, const double* tiles, const int4* seg, int nseg, int mode,
                       const double* x, const double* rin, double* y, int sm_count,
                       double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  if (mode == kDelta)
    return st2_launch<kDelta>(g, tiles, seg, nseg, x, rin, y, sm_count, partials, st, dotmode, s);
  return st2_launch<kOuterRhs>(g, tiles, seg, nseg, x, rin, y, sm_count, partials, st, kDotNone, s);
}

long long st2_max_blocks(int sm_count) { return 64LL * sm_count; }

}  // namespace gq
