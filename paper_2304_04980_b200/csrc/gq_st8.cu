// Block stencils for n = 8 on the fp64 tensor cores ("st8" kernels).
//
// Same operators as the generic stencils of gq_stencil.cu (kkt_assembly.py:379-425):
//   Delta:      (Delta x)_t = Psi_t x_t + Xi_{t-1} x_{t-1} + Xi_t' x_{t+1}
//   outer rhs:  y_t = r_t - (Xi_{t-1} x_{t-1} + Xi_t' x_{t+1})        (r + Xi~ x)
// At n = 8 every block is 8 x 8, i.e. exactly one m8n8k4 fp64 DMMA pair with the 8 stages of
// a class-pure stage chunk on M: D[stage][out] += x_nbr[stage][feat] * B[feat][out] with
// B[f][o] = block[o][f].  With features interleaved across the two k-steps (lane quad qd
// holds features 2qd and 2qd+1), the A fragment is ONE 16-byte load of the neighbour's
// record (stage-inner layout), the B fragment ONE 16-byte load of the row-major block and
// the D fragment the lane's 16 bytes of the output record -- no staging, no shuffles.
// A warp owns one node and walks its stage chunks (the chain kernel's class-pure segments);
// the node's operator blocks stay in L1 across chunks.  23 (Delta) or 10 (outer rhs) blocks
// are spread over 8 independent accumulators to keep the DMMA dependency chains short.
#include <algorithm>
#include <cstdlib>

#include "gq_async.cuh"
#include "gq_internal.h"

namespace gq {

namespace {
using namespace as;
__device__ __forceinline__ double2 ld16(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}
}  // namespace

template <int MODE>
__device__ __forceinline__ void st8_body(const Geo& g, const Ops& op, const int4* __restrict__ seg,
                                        int nseg, const double* __restrict__ x,
                                        const double* __restrict__ rin,
                                        double* __restrict__ y, double* partials,
                                        PcgState* st, int dotmode) {
  constexpr int NS = 8, B2 = 64;
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
  const long long rs = (long long)g.TS * NS, cs = (long long)g.K * rs;
  double dot = 0.0;
#pragma unroll 1
  for (long long node = blockIdx.x; node < g.nk; node += gridDim.x) {
    const int j = (int)(node / g.K), i = (int)(node % g.K);
    // neighbour record bases (stage 0) and validity for the 13-point diamond
    const double* nb[13];
    bool ok[13];
#pragma unroll
    for (int o = 0; o < 13; ++o) {
      const int jj = j + odj(o), ii = i + odi(o);
      ok[o] = jj >= 0 && jj < g.N && ii >= 0 && ii < g.K;
      nb[o] = x + (ok[o] ? (long long)jj * cs + (long long)ii * rs : 0) + 2 * qd;
    }
    const double* xi = op.xi + (long long)node * 5 * B2 + rw * 8 + 2 * qd;    // nxc == 1
    const double* xit = op.xit + (long long)node * 5 * B2 + rw * 8 + 2 * qd;
#pragma unroll 1
    for (int sgi = 0; sgi < nseg; ++sgi) {
      const int4 sg = seg[sgi];
      const int t0 = sg.x, nvalid = sg.y, pc = sg.z;
      const int t = t0 + rw;
      const bool tv = rw < nvalid;
      double2 acc[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) acc[a] = make_double2(0.0, 0.0);
      double2 xself = make_double2(0.0, 0.0);
      if (MODE == kDelta) {
        const double* P = op.psi + ((long long)pc * g.nk + node) * 13 * B2 + rw * 8 + 2 * qd;
#pragma unroll
        for (int o = 0; o < 13; ++o) {
          const double2 a = (ok[o] && tv) ? ld16(nb[o] + (long long)t * NS) : make_double2(0.0, 0.0);
          if (o == 0) xself = a;
          const double2 b = ld16(P + o * B2);
          dmma(acc[o & 7], a.x, b.x);
          dmma(acc[o & 7], a.y, b.y);
        }
      } else {
        xself = make_double2(0.0, 0.0);
      }
      // Xi_{t-1} x_{t-1} (t >= 1) and Xi_t' x_{t+1} (t + 1 <= T): 5-point neighbours
      const bool tm = tv && t >= 1, tp = tv && t + 1 < g.T1;
      double2 e[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
#pragma unroll
      for (int u = 0; u < 5; ++u) {
        const double2 am = (ok[u] && tm) ? ld16(nb[u] + (long long)(t - 1) * NS) : make_double2(0.0, 0.0);
        const double2 ap = (ok[u] && tp) ? ld16(nb[u] + (long long)(t + 1) * NS) : make_double2(0.0, 0.0);
        const double2 bm = ld16(xi + u * B2), bp = ld16(xit + u * B2);
        double2& am_acc = MODE == kDelta ? acc[(u + 5) & 7] : e[0];
        double2& ap_acc = MODE == kDelta ? acc[(u + 2) & 7] : e[1];
        dmma(am_acc, am.x, bm.x);
        dmma(am_acc, am.y, bm.y);
        dmma(ap_acc, ap.x, bp.x);
        dmma(ap_acc, ap.y, bp.y);
      }
      double2 out;
      if (MODE == kDelta) {
        out = add2(add2(add2(acc[0], acc[1]), add2(acc[2], acc[3])),
                   add2(add2(acc[4], acc[5]), add2(acc[6], acc[7])));
      } else {   // y = r + (-(Xi_{t-1} x_{t-1}) - Xi_t' x_{t+1})   (gq_grid.cu convention)
        const double2 rv = tv ? ld16(rin + (long long)j * cs + (long long)i * rs + (long long)t * NS + 2 * qd)
                              : make_double2(0.0, 0.0);
        out.x = rv.x + ((0.0 - e[0].x) - e[1].x);
        out.y = rv.y + ((0.0 - e[0].y) - e[1].y);
      }
      if (tv && (MODE != kDelta || slab_owned(g, t))) {
        *reinterpret_cast<double2*>(y + (long long)j * cs + (long long)i * rs + (long long)t * NS + 2 * qd) = out;
        if (MODE == kDelta && dotmode != kDotNone) {
          dot = fma(out.x, xself.x, dot);
          dot = fma(out.y, xself.y, dot);
        }
      }
    }
  }
  if (MODE == kDelta && dotmode != kDotNone) {
    double c;
    // one-warp CTAs: warp sum + last-block pass over the per-CTA partials (fixed order)
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
      c = acc;
      if (lane == 0) {
        st->counter[0] = 0u;
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
}

// ---- n = 4: two vertically adjacent nodes per warp ------------------------------------------
// A 4 x 4 block is one k-step (K = 4 = the input node's features); the N = 8 outputs are the
// 4 features of node a1 = (i, j) and the 4 of a2 = (i + 1, j).  For every input node z of the
// union of the two stencils one DMMA computes both contributions:
//   D[stage][out] += x_z[stage][k] * B[k][out],  B[k][out] = Blk(a1, z)[out][k]  (out < 4)
//                                                           Blk(a2, z)[out-4][k] (out >= 4)
// A fragment: lane (rw, qd) holds x_z[t0 + rw][qd]; B fragment: lane (qd, rw) holds the entry
// above (zero where z is outside that node's stencil); D fragment: lane (rw, qd) holds two
// consecutive outputs of node a1 (qd < 2) or a2 (qd >= 2) at stage t0 + rw.  Union of the two
// 13-point diamonds: 18 input nodes; of the two 5-point stencils: 8 (times two stages).
namespace {
// input node z = a1 + (di, dj); o1 / o2 = its 13-point index as seen from a1 / a2, or -1
__device__ constexpr int U13_DI[18] = {-2, -1, 0, 1, 2, 3, -1, 0, 1, 2, -1, 0, 1, 2, 0, 1, 0, 1};
__device__ constexpr int U13_DJ[18] = {0, 0, 0, 0, 0, 0, -1, -1, -1, -1, 1, 1, 1, 1, -2, -2, 2, 2};
__device__ constexpr int U13_O1[18] = {5, 1, 0, 2, 6, -1, 9, 3, 11, -1, 10, 4, 12, -1, 7, -1, 8, -1};
__device__ constexpr int U13_O2[18] = {-1, 5, 1, 0, 2, 6, -1, 9, 3, 11, -1, 10, 4, 12, -1, 7, -1, 8};
// the same for the 5-point stencil (self, north, south, west, east)
__device__ constexpr int U5_DI[8] = {-1, 0, 1, 2, 0, 1, 0, 1};
__device__ constexpr int U5_DJ[8] = {0, 0, 0, 0, -1, -1, 1, 1};
__device__ constexpr int U5_U1[8] = {1, 0, 2, -1, 3, -1, 4, -1};
__device__ constexpr int U5_U2[8] = {-1, 1, 0, 2, -1, 3, -1, 4};
}  // namespace

constexpr int kSt4Group = 4;   // stage chunks per item: the B fragments are loaded once per item

template <int MODE>
__global__ void __launch_bounds__(32, 12) k_st4(Geo g, Ops op, const int4* __restrict__ seg, int nseg,
                                            const double* __restrict__ x,
                                            const double* __restrict__ rin,
                                            double* __restrict__ y, double* partials,
                                            PcgState* st, int dotmode) {
  constexpr int NS = 4, B2 = 16;
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
  const long long rs = (long long)g.TS * NS, cs = (long long)g.K * rs;
  const int kp = (g.K + 1) / 2;                       // node pairs per column
  const long long npairs = (long long)kp * g.N;
  const int ngr = (nseg + kSt4Group - 1) / kSt4Group;
  const int which = rw >> 2, orow = rw & 3;           // my B entry: node a1 / a2, output row
  double dot = 0.0;
  // items = (node pair, group of stage chunks): the groups of a pair go to consecutive warps
#pragma unroll 1
  for (long long item = blockIdx.x; item < npairs * ngr; item += gridDim.x) {
    const long long pr = item / ngr;
    const int gi = (int)(item - pr * ngr);
    const int j = (int)(pr / kp), i1 = 2 * (int)(pr % kp);
    const bool has2 = i1 + 1 < g.K;
    const long long node1 = (long long)j * g.K + i1;
    const long long mynode = node1 + which;           // the node my B entries belong to
    const bool bok = which == 0 || has2;
    // my output: node a1 (qd < 2) or a2, features 2 (qd & 1), +1
    const int onode = qd >> 1;
    const bool ook = onode == 0 || has2;
    const long long obase = (long long)j * cs + (long long)(i1 + onode) * rs + 2 * (qd & 1);
    // A-fragment sources (stage 0) and validity of the input nodes
    const double* xa = x + (long long)j * cs + (long long)i1 * rs + qd;
    bool z13[18], z5[8];
#pragma unroll
    for (int e = 0; e < 18; ++e) {
      const int ii = i1 + U13_DI[e], jj = j + U13_DJ[e];
      z13[e] = ii >= 0 && ii < g.K && jj >= 0 && jj < g.N;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ii = i1 + U5_DI[e], jj = j + U5_DJ[e];
      z5[e] = ii >= 0 && ii < g.K && jj >= 0 && jj < g.N;
    }
    // B fragments of the Xi parts (one class: nxc == 1), loaded once per item
    double bm[8], bp[8];
    {
      const double* xi = op.xi + mynode * 5 * B2 + orow * NS + qd;
      const double* xit = op.xit + mynode * 5 * B2 + orow * NS + qd;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int u = which == 0 ? U5_U1[e] : U5_U2[e];
        bm[e] = (u >= 0 && bok) ? __ldg(xi + u * B2) : 0.0;
        bp[e] = (u >= 0 && bok) ? __ldg(xit + u * B2) : 0.0;
      }
    }
    double bpsi[MODE == kDelta ? 18 : 1];
    int cur = -1;
    const int s1 = min(nseg, (gi + 1) * kSt4Group);
#pragma unroll 1
    for (int sgi = gi * kSt4Group; sgi < s1; ++sgi) {
      const int4 sg = seg[sgi];
      const int t0 = sg.x, nvalid = sg.y, pc = sg.z;
      const int t = t0 + rw;
      const bool tv = rw < nvalid;
      double2 acc[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) acc[a] = make_double2(0.0, 0.0);
      if (MODE == kDelta) {
        if (pc != cur) {      // Psi B fragments of this stage class
          const double* P = op.psi + ((long long)pc * g.nk + mynode) * 13 * B2 + orow * NS + qd;
#pragma unroll
          for (int e = 0; e < 18; ++e) {
            const int o = which == 0 ? U13_O1[e] : U13_O2[e];
            bpsi[e] = (o >= 0 && bok) ? __ldg(P + o * B2) : 0.0;
          }
          cur = pc;
        }
#pragma unroll
        for (int e = 0; e < 18; ++e) {
          const double av = (z13[e] && tv) ? __ldg(xa + U13_DJ[e] * cs + U13_DI[e] * rs +
                                                   (long long)t * NS)
                                           : 0.0;
          dmma(acc[e & 3], av, bpsi[e]);
        }
      }
      // Xi_{t-1} x_{t-1} (t >= 1) and Xi_t' x_{t+1} (t + 1 <= T)
      const bool tm = tv && t >= 1, tp = tv && t + 1 < g.T1;
      double2 em = make_double2(0.0, 0.0), ep = em;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double* xz = xa + U5_DJ[e] * cs + U5_DI[e] * rs;
        const double am = (z5[e] && tm) ? __ldg(xz + (long long)(t - 1) * NS) : 0.0;
        const double ap = (z5[e] && tp) ? __ldg(xz + (long long)(t + 1) * NS) : 0.0;
        if (MODE == kDelta) {
          dmma(acc[e & 3], am, bm[e]);
          dmma(acc[(e + 2) & 3], ap, bp[e]);
        } else {
          dmma(em, am, bm[e]);
          dmma(ep, ap, bp[e]);
        }
      }
      double2 out;
      if (MODE == kDelta) {
        out = add2(add2(acc[0], acc[1]), add2(acc[2], acc[3]));
      } else {   // y = r + (-(Xi_{t-1} x_{t-1}) - Xi_t' x_{t+1})   (gq_grid.cu convention)
        const double2 rv = (tv && ook) ? ld16(rin + obase + (long long)t * NS)
                                       : make_double2(0.0, 0.0);
        out.x = rv.x + ((0.0 - em.x) - ep.x);
        out.y = rv.y + ((0.0 - em.y) - ep.y);
      }
      if (tv && ook && (MODE != kDelta || slab_owned(g, t))) {
        *reinterpret_cast<double2*>(y + obase + (long long)t * NS) = out;
        if (MODE == kDelta && dotmode != kDotNone) {
          const double2 xs = ld16(x + obase + (long long)t * NS);
          dot = fma(out.x, xs.x, dot);
          dot = fma(out.y, xs.y, dot);
        }
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

// Delta: uncapped (102 registers; every cap tried was slower: 96 -> 3.80 ms, 80 -> 3.17 ms
// vs 2.52 ms at config 5).  Outer rhs: capped at 64 registers (from 66 at the default
// bound, 122 at a looser one), 1.078 -> 0.997 ms.
template <int MODE>
__global__ void __launch_bounds__(32) k_st8(Geo g, Ops op, const int4* __restrict__ seg,
                                            int nseg, const double* __restrict__ x,
                                            const double* __restrict__ rin,
                                            double* __restrict__ y, double* partials,
                                            PcgState* st, int dotmode) {
  st8_body<MODE>(g, op, seg, nseg, x, rin, y, partials, st, dotmode);
}

__global__ void __launch_bounds__(32, 32) k_st8_rhs(Geo g, Ops op, const int4* __restrict__ seg,
                                                   int nseg, const double* __restrict__ x,
                                                   const double* __restrict__ rin,
                                                   double* __restrict__ y, double* partials,
                                                   PcgState* st, int dotmode) {
  st8_body<kOuterRhs>(g, op, seg, nseg, x, rin, y, partials, st, dotmode);
}

static int s8env(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

bool st8_supported(const Geo& g, int nxc) {
  return (g.n == 8 || g.n == 4) && nxc == 1 && s8env("GQ_NO_ST8", 0) == 0;
}

template <int MODE>
static cudaError_t st8_launch(const Geo& g, const Ops& op, const int4* seg, int nseg,
                              const double* x, const double* rin, double* y, int sm_count,
                              double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  if (g.n == 4) {
    static int cache4[64] = {0};
    int per_sm4 = 1;
    cudaError_t e4 = kernel_occupancy(k_st4<MODE>, 32, 0, cache4, per_sm4);
    if (e4 != cudaSuccess) return e4;
    const long long items = (long long)((g.K + 1) / 2) * g.N * ((nseg + kSt4Group - 1) / kSt4Group);
    const long long blocks4 = std::min<long long>(items, (long long)per_sm4 * sm_count);
    k_st4<MODE><<<(unsigned)blocks4, 32, 0, s>>>(g, op, seg, nseg, x, rin, y, partials, st, dotmode);
    return cudaGetLastError();
  }
  static int cache[64] = {0};
  int per_sm = 1;
  cudaError_t e = MODE == kDelta ? kernel_occupancy(k_st8<kDelta>, 32, 0, cache, per_sm)
                                 : kernel_occupancy(k_st8_rhs, 32, 0, cache, per_sm);
  if (e != cudaSuccess) return e;
  const long long blocks = std::min<long long>(g.nk, (long long)per_sm * sm_count);
  if (MODE == kDelta)
    k_st8<kDelta><<<(unsigned)blocks, 32, 0, s>>>(g, op, seg, nseg, x, rin, y, partials, st, dotmode);
  else
    k_st8_rhs<<<(unsigned)blocks, 32, 0, s>>>(g, op, seg, nseg, x, rin, y, partials, st, dotmode);
  return cudaGetLastError();
}

cudaError_t launch_st8(const Geo& g, const Ops& op, const int4* seg, int nseg, int mode,
                       const double* x, const double* rin, double* y, int sm_count,
                       double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  if (mode == kDelta)
    return st8_launch<kDelta>(g, op, seg, nseg, x, rin, y, sm_count, partials, st, dotmode, s);
  return st8_launch<kOuterRhs>(g, op, seg, nseg, x, rin, y, sm_count, partials, st, kDotNone, s);
}

long long st8_max_blocks(int sm_count) { return 64LL * sm_count; }

}  // namespace gq
