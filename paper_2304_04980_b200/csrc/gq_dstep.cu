// Delta apply for n = 2 with the stage index as the loop axis ("t-loop" stencil).
//
// Factored form of the reduced operator (kkt_assembly.py:487-544 assembles the same matrix
// as Psi / Xi blocks):
//
//   z_t = Q_t^-1 (d_t - Ahat_t' d_{t+1})                       (t < T; z_T = Q_T^-1 d_T)
//   (Delta d)_t = z_t - Ahat_{t-1} z_{t-1} + B_{t-1} R_{t-1}^-1 B_{t-1}' d_t   (t >= 1)
//   (Delta d)_0 = z_0
//
// which expands to Psi_t d_t + Xi_{t-1} d_{t-1} + Xi_t' d_{t+1} with Psi_t = Q_t^-1 +
// Ahat Q_{t-1}^-1 Ahat' + B R^-1 B' and Xi_t = -Ahat_t Q_t^-1 (kkt_assembly.py:379-403).
// Ahat_t is the 5-point grid stencil of the dynamics (A on the node, the four coupling
// blocks toward in-grid neighbours), so both products are 5-point stencils in (i, j).
//
// Mapping.  A CTA owns a 32 x 8 tile of grid nodes (rows i x columns j) and a range of
// stages, and walks the stages in order.  Every thread owns one node of the tile plus its
// one-node halo (34 x 10 "z domain", 340 threads); its operator blocks (Ahat' column,
// Q^-1, Ahat row, B R^-1 B': 48 doubles) sit in registers for the whole range -- they
// depend on t only through the stage classes -- so the inner loop reads no operator data.
// Per stage a thread forms z_t of its node from d_{t+1} of its 5-point neighbourhood,
// publishes z_t in a shared plane, and (interior threads) forms y_t from z_{t-1} of its
// neighbourhood: two 5-point stencils, 52 DFMA and 10 shared accesses per node-stage.
//
// Data movement.  d arrives by TMA as a 3-D box per chunk: 4 stages (64 contiguous bytes of a
// node) x 36 rows x 12 columns (tile + 2-node halo; out-of-grid nodes and stages past T
// zero-filled), with the 64-byte swizzle so that the 16-byte loads of 32 consecutive rows
// hit distinct bank groups; three chunks in flight on mbarriers, the stream continuing into
// the CTA's next item.  y leaves the same way: a 4-stage output box per chunk, stored by TMA
// while the next chunk is computed.  (A stage-outer 4-D box -- one contiguous plane per
// stage, 16-byte rows -- was measured: TMA moves 16-byte rows about 4x slower per byte and
// the loads fell behind.)
//
// Schedule.  Per stage a thread forms z_t of its node and publishes it in z plane t & 1;
// output threads form y_t = z_t + (B R^-1 B' d_t - Ahat_{t-1} z_{t-1}), the second term
// issued first (it only needs the previous plane), as FMA chains over pre-negated blocks.
// One __syncthreads per stage orders the planes.  Chunks whose four stages share their
// stage classes run a fully unrolled stage loop: every shared-memory address is a register
// base plus an immediate.
//
// Reference: gridlq/kkt_assembly.py:346-403 (SchurOperator.apply), pcg.py:99-108 (the
// curvature y.d and alpha fused at the end).
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "gq_async.cuh"
#include "gq_internal.h"

namespace gq {

namespace {

using namespace as;

#ifndef GQ_DSTEP_TI
#define GQ_DSTEP_TI 32
#endif
constexpr int TI = GQ_DSTEP_TI, TJ = 8;      // output tile: rows x columns
// CTAs per SM: one 352-thread CTA at TI = 32 (measured: two 192-thread CTAs at TI = 16 run
// the headline Delta in the same 0.24 ms, with 15% more shared-memory traffic for the halo)
constexpr int MINB = TI == 16 ? 2 : 1;
constexpr int ZI = TI + 2, ZJ = TJ + 2;      // z domain (tile + 1-node halo)
constexpr int PI = TI + 4, PJ = TJ + 4;      // d plane (tile + 2-node halo)
constexpr int NZ = ZI * ZJ;                  // 340 z nodes, one per thread
constexpr int NTHR = (NZ + 31) / 32 * 32;    // 352
constexpr int CH = 4;                        // stages per TMA chunk
constexpr int ROWB = CH * 16;                // bytes of one node in a chunk box
constexpr int BOX = ROWB * PI * PJ;          // 27648 bytes per chunk box
constexpr int NSLOT = 3;
constexpr int YBOX = ROWB * TI * TJ;         // 16384 bytes: one chunk of the output tile
constexpr int NYB = 3;                       // output boxes in flight (TMA stores)
constexpr int MAXT1 = 4096;                  // stage-class tables kept in shared memory
constexpr int NZP = 2;                       // z planes (double buffered by stage parity)
// Halo threads run the y body too (never stored) and read z one row / column outside the
// domain: each plane carries guard bands of >= ZI + 1 entries on both sides so those reads
// stay inside the allocation.  Front band and stride are multiples of 8 entries, so both
// planes start 128-byte aligned (a quarter warp's 8 consecutive LDS.128 = one wavefront).
constexpr int ZG = (ZI + 1 + 7) / 8 * 8;                   // front guard (entries)
constexpr int PZ = (ZG + NZ + ZI + 1 + 7) / 8 * 8;         // plane stride (entries)
static_assert(PZ - ZG - NZ >= ZI + 1, "back guard band");
// shared memory without the stage-class tables (3 * T1 ints, appended at launch)
constexpr int SMEM0 = 1024 /*align*/ + NSLOT * BOX + NYB * YBOX + NZP * PZ * 16 + NSLOT * 8;
static_assert((NSLOT * BOX + NYB * YBOX) % 128 == 0, "z planes start 128-byte aligned");
static_assert(BOX % 1024 == 0 && YBOX % 1024 == 0, "boxes keep the 1024-byte swizzle alignment");

// box coordinates: (stage offset in doubles, row, column)
__device__ __forceinline__ void tma3(unsigned dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                     unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma3_store(const CUtensorMap* tm, unsigned src, int c0, int c1,
                                           int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
          reinterpret_cast<uint64_t>(tm)),
      "r"(c0), "r"(c1), "r"(c2), "r"(src)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_init_u(unsigned bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_u(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_u(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_u(unsigned bar, unsigned parity) {
  for (long long i = 0; !mbar_try_u(bar, parity); ++i)
    if (i > (1LL << 28)) __trap();   // a protocol bug traps instead of hanging the device
}
__device__ __forceinline__ double2 lds2u(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts2u(unsigned a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}

// M x (M row-major 2 x 2); products of independent blocks are summed as a tree
__device__ __forceinline__ double2 mv(const double* M, double2 x) {
  return make_double2(fma(M[0], x.x, M[1] * x.y), fma(M[2], x.x, M[3] * x.y));
}
__device__ __forceinline__ double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
// acc + M x as one FMA chain per component
__device__ __forceinline__ double2 mac(double2 acc, const double* M, double2 x) {
  return make_double2(fma(M[1], x.y, fma(M[0], x.x, acc.x)), fma(M[3], x.y, fma(M[2], x.x, acc.y)));
}
// acc + M x
__device__ __forceinline__ double2 mva(double2 acc, const double* M, double2 x) {
  return make_double2(fma(M[0], x.x, fma(M[1], x.y, acc.x)), fma(M[2], x.x, fma(M[3], x.y, acc.y)));
}

struct DsArgs {
  Geo g;
  DstepOps op;
  double* y;
  double* partials;
  PcgState* st;
  int dotmode;
  int ntI, nr, RL, n_items;
};

// operator blocks of one node, per stage class
struct NodeOps {
  double M[5][4];   // z stencil: -Ahat(v, a)' for v = a, north, south, west, east of a
  double Qi[4];     // Q_t^-1 (a)
  double W[5][4];   // y stencil: -Ahat(a, v)
  double BB[4];     // B R^-1 B' (a)
};

__device__ __forceinline__ void ld4(double* dst, const double* src) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(src));
  const double2 b = __ldg(reinterpret_cast<const double2*>(src + 2));
  dst[0] = a.x; dst[1] = a.y; dst[2] = b.x; dst[3] = b.y;
}
__device__ __forceinline__ void zero4(double* d) { d[0] = d[1] = d[2] = d[3] = 0.0; }

// z-stencil blocks of node (i, j) for dynamics set dc: M[u] = Ahat(a + off(u), a)'
__device__ __forceinline__ void load_zops(NodeOps& o, const Geo& g, const DstepOps& op, int dc, int i, int j,
                          bool in) {
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    double b[4];
    zero4(b);
    const int ii = i + odi(u), jj = j + odj(u);
    if (in && ii >= 0 && ii < g.K && jj >= 0 && jj < g.N) {
      const long long nb = (long long)jj * g.K + ii;
      if (u == 0)
        ld4(b, op.A + ((long long)dc * g.nk + nb) * 4);
      else   // the neighbour's coupling toward a
        ld4(b, op.C + (((long long)dc * 4 + slot_dir(slot_opp(u))) * g.nk + nb) * 4);
    }
    o.M[u][0] = -b[0]; o.M[u][1] = -b[2]; o.M[u][2] = -b[1]; o.M[u][3] = -b[3];   // -transpose
  }
}
__device__ __forceinline__ void load_q(NodeOps& o, const Geo& g, const DstepOps& op, int qc, int i, int j,
                       bool in) {
  zero4(o.Qi);
  if (in) ld4(o.Qi, op.qinv + ((long long)qc * g.nk + (long long)j * g.K + i) * 4);
}
// y-stencil blocks of node (i, j) for dynamics set dc: W[u] = Ahat(a, a + off(u))
__device__ __forceinline__ void load_yops(NodeOps& o, const Geo& g, const DstepOps& op, int dc, int i, int j,
                          bool in) {
  const long long node = (long long)j * g.K + i;
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    zero4(o.W[u]);
    const int ii = i + odi(u), jj = j + odj(u);
    if (in && ii >= 0 && ii < g.K && jj >= 0 && jj < g.N) {
      if (u == 0)
        ld4(o.W[u], op.A + ((long long)dc * g.nk + node) * 4);
      else
        ld4(o.W[u], op.C + (((long long)dc * 4 + slot_dir(u)) * g.nk + node) * 4);
#pragma unroll
      for (int e = 0; e < 4; ++e) o.W[u][e] = -o.W[u][e];
    }
  }
  zero4(o.BB);
  if (in) ld4(o.BB, op.brb + ((long long)dc * g.nk + node) * 4);
}

__global__ void __launch_bounds__(NTHR, MINB) k_dstep(const __grid_constant__ CUtensorMap dmap,
                                                   const __grid_constant__ CUtensorMap ymap,
                                                   const DsArgs a) {
  extern __shared__ unsigned char smem_raw[];
  const Geo& g = a.g;
  PcgState* st = a.st;
  if (st != nullptr) {
    if (a.dotmode == kDotStep) {
      // first kernel of a PCG step: the step budget (pcg.py:98) decides for the whole step
      const bool stop = st->done || st->step >= st->max_steps;
      if (blockIdx.x == 0 && threadIdx.x == 0) st->skip = stop ? 1 : 0;
      if (stop) return;
    } else if (halted(st)) {
      return;
    }
  }
  const unsigned base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const unsigned ybase = base + NSLOT * BOX;            // output boxes
  const unsigned zpl = ybase + NYB * YBOX + ZG * 16;    // z planes: NZP x PZ double2
  const unsigned bars = ybase + NYB * YBOX + NZP * PZ * 16;
  int* tcls = reinterpret_cast<int*>(smem_raw + (bars + NSLOT * 8 - smem_u32(smem_raw)));
  const int tid = threadIdx.x;
  const int T = g.T;
  // stage-class tables: tcls[t] = dynamics set of Ahat_t (t < T; T -> T-1), tcls[T1 + t] =
  // cost set of Q_t; sigc[c] = the packed classes (Ahat_t, Q_t, Ahat_{t-1}) shared by all
  // stages of chunk c, -1 if they differ, the chunk holds stage 0 or a stage-slab halo row
  int* sigc = tcls + 2 * g.T1;
  auto dz_of = [&](int t) { return a.op.dcls[min(t, T - 1)]; };
  for (int t = tid; t < g.T1; t += NTHR) {
    tcls[t] = dz_of(t);
    tcls[g.T1 + t] = a.op.ccls[t];
  }
  for (int c = tid; c * CH < g.T1; c += NTHR) {
    int sg = -1;
    const int t0 = c * CH;
    if (t0 >= 1 && t0 + CH <= g.T1) {
      const int dz = dz_of(t0), q = a.op.ccls[t0], dy = a.op.dcls[t0 - 1];
      bool same = dz < 1024 && q < 1024 && dy < 1024;
      for (int t = t0; t < t0 + CH; ++t)
        same = same && dz_of(t) == dz && a.op.ccls[t] == q && a.op.dcls[t - 1] == dy &&
               slab_owned(g, t);
      if (same) sg = dz | (q << 10) | (dy << 20);
    }
    sigc[c] = sg;
  }
  if (tid == 0)
    for (int s = 0; s < NSLOT; ++s) mbar_init_u(bars + 8 * s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  const bool zn = tid < NZ;
  const int zi = zn ? tid % ZI : 0, zj = zn ? tid / ZI : 0;
  const bool inner = zn && zi >= 1 && zi <= TI && zj >= 1 && zj <= TJ;
  // 64-byte swizzle: 16-byte chunk s of box row R sits at R * 64 + ((s ^ ((R >> 1) & 3)) << 4).
  // Box bases are 1024-aligned and R * 64 has zero low bits, so the address is
  // (box + q) ^ (s << 4) with q = R * 64 + (((R >> 1) & 3) << 4).  pq: the z stencil's five
  // d points (self, north, south, west, east); yq: the node's row of an output box.
  unsigned pq[5];
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    const unsigned R = (unsigned)((zj + 1 + odj(u)) * PI + (zi + 1 + odi(u)));
    pq[u] = R * ROWB + (((R >> 1) & 3u) << 4);
  }
  const unsigned yR = inner ? (unsigned)((zj - 1) * TI + (zi - 1)) : 0u;
  const unsigned yq = yR * ROWB + (((yR >> 1) & 3u) << 4);
  const unsigned zme = (unsigned)tid * 16;
  double dot = 0.0;
  unsigned seq = 0;    // d chunks loaded by this CTA (ring slot / phase bookkeeping)
  unsigned yseq = 0;   // output boxes stored by this CTA
  int pre = 0;         // chunks of the next item already in flight (issued by this one)
  // item geometry: tile origin, stage range [ta, tb), chunk range [c0, c1]
  struct It {
    int i0, j0, ta, tb, c0, c1;
  };
  auto item_at = [&](int item) {
    It r;
    const int tile = item / a.nr, rr = item - tile * a.nr;
    r.i0 = (tile % a.ntI) * TI;
    r.j0 = (tile / a.ntI) * TJ;
    r.ta = rr * a.RL;
    r.tb = min(g.T1, r.ta + a.RL);
    r.c0 = (r.ta > 0 ? r.ta - 1 : 0) / CH;
    r.c1 = r.tb / CH;
    return r;
  };
  // chunk c of item `it` into ring position sq
  auto issue_at = [&](const It& it, int c, unsigned sq) {
    if (tid == 0) {
      const unsigned slot = sq % NSLOT;
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_expect_u(bars + 8 * slot, BOX);
      tma3(base + slot * BOX, &dmap, c * CH * 2, it.i0 - 2, it.j0 - 2, bars + 8 * slot);
    }
  };

#pragma unroll 1
  for (int item = blockIdx.x; item < a.n_items; item += gridDim.x) {
    const It it = item_at(item);
    const int i0 = it.i0, j0 = it.j0, ta = it.ta, tb = it.tb, c0 = it.c0, c1 = it.c1;
    const int sfirst = ta > 0 ? ta - 1 : 0;
    const int clast = (tb - 1) / CH;
    const int i = i0 - 1 + zi, j = j0 - 1 + zj;
    const bool in = zn && i >= 0 && i < g.K && j >= 0 && j < g.N;
    const bool outp = inner && in;
    const unsigned sq0 = seq;
    seq = sq0 + (unsigned)(c1 - c0 + 1);
    // the stream of chunks continues into the next item of this CTA (no pipeline bubble at
    // item boundaries): ring position sq0 + (c1 - c0 + 1) + k is its chunk c0' + k
    const bool has_next = item + (int)gridDim.x < a.n_items;
    const It nx = item_at(has_next ? item + (int)gridDim.x : item);

    auto issue = [&](int c) {
      if (c <= c1) {
        issue_at(it, c, sq0 + (unsigned)(c - c0));
      } else if (has_next && nx.c0 + (c - c1 - 1) <= nx.c1) {
        issue_at(nx, nx.c0 + (c - c1 - 1), sq0 + (unsigned)(c - c0));
        ++pre;
      }
    };
    auto wait = [&](int c) {
      const unsigned sq = sq0 + (unsigned)(c - c0);
      mbar_wait_u(bars + 8 * (sq % NSLOT), (sq / NSLOT) & 1u);
    };
    for (int k = pre; k < 2 && c0 + k <= c1; ++k) issue(c0 + k);
    pre = 0;
    wait(c0);

    NodeOps o;
    int cz = -1, cq = -1, cy = -1;   // stage classes currently in registers
    double2 dt = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int c = c0; c <= clast; ++c) {
      // chunk c + 2 takes the slot of chunk c - 1, which no stage from here on reads
      issue(c + 2);          // c + 2 past c1: the next item's first chunks
      if (c + 1 <= c1) wait(c + 1);
      const unsigned sq = sq0 + (unsigned)(c - c0);
      const unsigned pb0 = base + (sq % NSLOT) * BOX;           // box of chunk c
      const unsigned pb1 = base + ((sq + 1) % NSLOT) * BOX;     // ... of chunk c + 1
      const unsigned yb = ybase + (yseq % NYB) * YBOX;          // output box of chunk c
      const bool ychunk = c * CH >= ta;      // every stage of the chunk is an output stage
      // one stage (s = stage within the chunk).  Every z-domain thread runs the whole body
      // (halo threads form a y they never store): straight-line code lets the scheduler
      // interleave the independent z and y chains; only the stores and the dot are predicated.
      auto stage = [&](int s, int t, bool yo, bool owned) {
        const unsigned pb = s + 1 < CH ? pb0 : pb1, sx = (unsigned)((s + 1) % CH) << 4;
        const double2 d0 = lds2u((pb + pq[0]) ^ sx), dN = lds2u((pb + pq[1]) ^ sx);
        const double2 dS = lds2u((pb + pq[2]) ^ sx), dW = lds2u((pb + pq[3]) ^ sx);
        const double2 dE = lds2u((pb + pq[4]) ^ sx);
        // y_t - z_t = B_{t-1} R_{t-1}^-1 B_{t-1}' d_t - Ahat_{t-1} z_{t-1}  (none at t = 0)
        double2 yb_ = make_double2(0.0, 0.0);
        if (t >= 1) {   // uniform
          const unsigned zp = zpl + (unsigned)((t - 1) & 1) * PZ * 16 + zme;
          const double2 zC = lds2u(zp), zN = lds2u(zp - 16), zS = lds2u(zp + 16);
          const double2 zW = lds2u(zp - ZI * 16), zE = lds2u(zp + ZI * 16);
          yb_ = mv(o.BB, dt);
          yb_ = mac(yb_, o.W[0], zC);
          yb_ = mac(yb_, o.W[1], zN);
          yb_ = mac(yb_, o.W[2], zS);
          yb_ = mac(yb_, o.W[3], zW);
          yb_ = mac(yb_, o.W[4], zE);
        }
        // z_t = Q_t^-1 (d_t - Ahat_t' d_{t+1}); d past stage T is zero-filled: z_T = Q_T^-1 d_T
        double2 v = mac(dt, o.M[0], d0);
        v = mac(v, o.M[1], dN);
        v = mac(v, o.M[2], dS);
        v = mac(v, o.M[3], dW);
        v = mac(v, o.M[4], dE);
        const double2 z = mv(o.Qi, v);
        sts2u(zpl + (unsigned)(t & 1) * PZ * 16 + zme, z);
        const double2 yv = add(z, yb_);
        const bool keep = yo && owned;
        const double2 ys = keep ? yv : make_double2(0.0, 0.0);   // slab halo rows stay zero
        dot = fma(ys.x, dt.x, dot);
        dot = fma(ys.y, dt.y, dot);
        if (yo) sts2u((yb + yq) ^ ((unsigned)s << 4), ys);
        dt = d0;
      };
      if (sigc[c] >= 0 && sigc[c] == (cz | (cq << 10) | (cy << 20)) && c * CH >= ta &&
          c * CH + CH <= tb) {
        // steady state: the chunk's stages share their classes, all are output stages
#pragma unroll
        for (int s = 0; s < CH; ++s) {
          if (zn) stage(s, c * CH + s, outp, true);
          __syncthreads();
        }
      } else {
#pragma unroll 1
        for (int s = 0; s < CH; ++s) {
          const int t = c * CH + s;
          if (t < sfirst || t >= tb) continue;   // uniform over the CTA
          {
            const int wz = tcls[t], wq = tcls[g.T1 + t];
            if (wz != cz) { load_zops(o, g, a.op, wz, i, j, in); cz = wz; }
            if (wq != cq) { load_q(o, g, a.op, wq, i, j, in); cq = wq; }
            if (t >= ta && t >= 1) {
              const int wy = tcls[t - 1];
              if (wy != cy) { load_yops(o, g, a.op, wy, i, j, in); cy = wy; }
            }
          }
          if (zn) {
            if (t == sfirst) dt = lds2u((pb0 + pq[0]) ^ ((unsigned)s << 4));
            stage(s, t, outp && t >= ta, slab_owned(g, t));
          }
          __syncthreads();
        }
      }
      if (ychunk) {
        if (tid == 0) {
          // the chunk's output box -> y (rows / columns / stages past the grid are clipped)
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          tma3_store(&ymap, yb, c * CH * 2, i0, j0);
          bulk_commit();
          bulk_wait_read<1>();   // the box stored NYB - 1 chunks ago may be rewritten now
        }
        ++yseq;
      }
    }
  }
  if (tid == 0) bulk_wait_all();

  if (st != nullptr && a.dotmode != kDotNone) {
    double c;
    if (grid_reduce<false>(dot, a.partials, &st->counter[0], c) && threadIdx.x == 0) {
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

// ---- outer rhs  y = r - (Xi_{t-1} x_{t-1} + Xi_t' x_{t+1})  by TMA tiles ------------------
//
// nested_jacobi.py:117-121 (rhs_s = r + Xi~ delta_{s-1}), kkt_assembly.py:414-425 (the
// time-coupling part of Delta).  No plane exchange is needed here: with one Xi class the ten
// 2 x 2 blocks of a node (Xi(a, .) and Xi(., a)') stay in registers and a thread forms y_t of
// its node from x_{t-1} and x_{t+1} of its 5-point neighbourhood directly.
//
// A CTA (128 threads, two per SM) owns a 16 x 8 tile of nodes for a run of 8-stage chunks;
// chunk c is stages 8c + 1 .. 8c + 8, whole 128-byte lines of the padded layout (stage 0 of a
// tile is read and written straight from global memory when its first chunk starts).  Per
// chunk one x box arrives by TMA -- the tile with a one-node halo, 128-byte rows with the
// 128-byte swizzle, through a tensor map whose origin is stage 2, so that the box of chunk c
// holds x_{t+1} for all of its stages -- and one r box of the tile; y is formed in the r box
// and leaves by TMA from there.  The five points of x_{t+1} read at stage t stay in registers
// and serve as x_{t-1} two stages later: 5 + 1 shared loads, 1 store and 40 DFMA per
// node-stage, one __syncthreads per chunk.  Items are whole tiles (pieces of a tile's chunks on
// small grids), dealt round-robin; both rings run through item boundaries.
//
// Measured on the way (headline, one launch): 4-stage boxes as in k_dstep (64-byte rows bound
// the TMA unit near 3.9 TB/s of loads per chip) 0.184 ms; 8-stage boxes with r / y rows that
// straddle two lines (origin at stage 0) 0.175 ms, whole lines 0.154 ms; with the r ring one
// box deeper than the x ring (r is refilled only after its y store has left) 0.129 ms; one
// CTA per SM with deeper rings 0.158-0.170 ms (four warps do not hide the arithmetic).  The
// same traffic with the arithmetic removed takes 0.126 ms: what is left is DRAM traffic (the
// halo rows of neighbouring tiles are read at different times and miss L2).
namespace rs {
constexpr int TI = 16, TJ = 8;                   // tile
constexpr int CH = 8;                            // stages per chunk
constexpr int ROWB = CH * 16;                    // 128-byte rows
constexpr int QI = TI + 2, QJ = TJ + 2;          // x box: tile + 1-node halo
constexpr int XBYTES = ROWB * QI * QJ;
constexpr int XBOX = (XBYTES + 1023) / 1024 * 1024;   // slot stride (swizzle alignment)
constexpr int YBOX = ROWB * TI * TJ;             // r / y box
constexpr int NX = 2;                            // x boxes in the ring
constexpr int NR = 3;                            // r / y boxes in the ring
constexpr int NT = TI * TJ;                      // one thread per tile node
constexpr int SMEM = 1024 + NX * XBOX + NR * YBOX + (NX + NR) * 8;
static_assert(YBOX % 1024 == 0, "boxes keep the 1024-byte swizzle alignment");
}  // namespace rs

struct RsArgs {
  Geo g;
  const double* x;
  const double* r;
  double* y;
  const double* xi;    // [N][K][5][2][2]
  const double* xit;
  PcgState* st;
  int ntI, nch, tiles, pieces;
  long long total;     // items = tiles x pieces
};

__global__ void __launch_bounds__(rs::NT, 2) k_rstep(const __grid_constant__ CUtensorMap xmap,
                                                     const __grid_constant__ CUtensorMap rmap,
                                                     const __grid_constant__ CUtensorMap ymap,
                                                     const RsArgs a) {
  constexpr int TI = rs::TI, TJ = rs::TJ, CH = rs::CH, ROWB = rs::ROWB, QI = rs::QI;
  constexpr int XBYTES = rs::XBYTES, XBOX = rs::XBOX, YBOX = rs::YBOX, NX = rs::NX, NR = rs::NR;
  extern __shared__ unsigned char smem_raw[];
  const Geo& g = a.g;
  if (halted(a.st)) return;
  const unsigned base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const unsigned rbase = base + NX * XBOX;
  const unsigned xbar = rbase + NR * YBOX, rbar = xbar + NX * 8;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NX; ++s) mbar_init_u(xbar + 8 * s, 1);
    for (int s = 0; s < NR; ++s) mbar_init_u(rbar + 8 * s, 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  const int ti = tid % TI, tj = tid / TI;
  // 128-byte swizzle: 16-byte piece s of box row R sits at R * 128 + ((s ^ (R & 7)) << 4)
  unsigned pq[5];
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    const unsigned R = (unsigned)((tj + 1 + odj(u)) * QI + (ti + 1 + odi(u)));
    pq[u] = R * ROWB + ((R & 7u) << 4);
  }
  const unsigned yq = (unsigned)tid * ROWB + (((unsigned)tid & 7u) << 4);

  // Items are (tile, piece of its chunks); item k of this CTA is blockIdx.x + k * gridDim.x,
  // tiles fastest, so that at any time the CTAs work on neighbouring tiles at about the same
  // chunk (the halo rows of a box are then still in L2 from the neighbour's own read).
  struct Cur {
    int k, c, cs, ce, i0, j0;
    bool valid;
  };
  auto start = [&](Cur& u, int k) {
    const long long item = blockIdx.x + (long long)k * gridDim.x;
    u.k = k;
    u.valid = item < a.total;
    if (!u.valid) return;
    const int piece = (int)(item / a.tiles), tile = (int)(item - (long long)piece * a.tiles);
    u.cs = u.c = piece * a.nch / a.pieces;
    u.ce = (piece + 1) * a.nch / a.pieces;
    u.i0 = (tile % a.ntI) * TI;
    u.j0 = (tile / a.ntI) * TJ;
  };
  auto step = [&](Cur& u) {
    if (++u.c == u.ce) start(u, u.k + 1);
  };
  // producers (every thread tracks the cursors, thread 0 issues).  The x map starts at stage
  // 2: its box c holds stages 8c + 2 .. 8c + 9.  An item that starts inside a tile first takes
  // the box before its first chunk (x_{t-1}, x_t of its first stage).
  Cur px, pr, cu;
  start(px, 0);
  pr = cu = px;
  bool px_pre = px.valid && px.c > 0;
  unsigned px_q = 0, pr_q = 0;
  auto produce_x = [&](unsigned limit) {
    while (px.valid && px_q < limit) {
      if (tid == 0) {
        const unsigned slot = px_q % NX;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_u(xbar + 8 * slot, XBYTES);
        tma3(base + slot * XBOX, &xmap, (px_pre ? px.c - 1 : px.c) * CH * 2, px.i0 - 1,
             px.j0 - 1, xbar + 8 * slot);
      }
      ++px_q;
      if (px_pre) {
        px_pre = false;
      } else {
        step(px);
        px_pre = px.valid && px.c == px.cs && px.c > 0;
      }
    }
  };
  auto produce_r = [&](unsigned limit) {
    while (pr.valid && pr_q < limit) {
      if (tid == 0) {
        const unsigned slot = pr_q % NR;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_u(rbar + 8 * slot, YBOX);
        tma3(rbase + slot * YBOX, &rmap, pr.c * CH * 2, pr.i0, pr.j0, rbar + 8 * slot);
      }
      ++pr_q;
      step(pr);
    }
  };
  auto wait_x = [&](unsigned q) { mbar_wait_u(xbar + 8 * (q % NX), (q / NX) & 1u); };
  auto wait_r = [&](unsigned q) { mbar_wait_u(rbar + 8 * (q % NR), (q / NR) & 1u); };
  auto xpts = [&](unsigned q, int s, double2* v) {
    const unsigned xb = base + (q % NX) * XBOX, sx = (unsigned)s << 4;
#pragma unroll
    for (int u = 0; u < 5; ++u) v[u] = lds2u((xb + pq[u]) ^ sx);
  };

  produce_x(NX);
  produce_r(NR);
  unsigned xq = 0, rq = 0;   // next x box / r box to consume
  double Xm[5][4], Xp[5][4];
  double2 xa[5], xb_[5];     // x_{t-1}, x_t of the 5-point neighbourhood
#pragma unroll 1
  for (; cu.valid; step(cu)) {
    const int i0 = cu.i0, j0 = cu.j0, c = cu.c;
    if (c == cu.cs) {   // a new item: the node's Xi blocks and the stage window
      const int i = i0 + ti, j = j0 + tj;
      const bool in = i < g.K && j < g.N;
      const long long node = (long long)j * g.K + i;
#pragma unroll
      for (int u = 0; u < 5; ++u) {
        zero4(Xm[u]);
        zero4(Xp[u]);
        if (in) {
          ld4(Xm[u], a.xi + (node * 5 + u) * 4);
          ld4(Xp[u], a.xit + (node * 5 + u) * 4);
        }
      }
      if (c > 0) {
        wait_x(xq);
        xpts(xq, CH - 2, xa);
        xpts(xq, CH - 1, xb_);
        ++xq;
        __syncthreads();   // the box may be refilled
      } else {
        // stage 0 straight from global memory: x_0 and x_1 open the window, and
        // y_0 = r_0 - Xi_0' x_1 (no Xi_{-1})
        double2 ep = make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < 5; ++u) {
          const int ii = i + odi(u), jj = j + odj(u);
          xa[u] = xb_[u] = make_double2(0.0, 0.0);
          if (in && ii >= 0 && ii < g.K && jj >= 0 && jj < g.N) {
            const double2* px =
                reinterpret_cast<const double2*>(a.x + ((long long)jj * g.K + ii) * g.TS * 2);
            xa[u] = __ldg(px);
            xb_[u] = __ldg(px + 1);
          }
          ep = mac(ep, Xp[u], xb_[u]);
        }
        if (in) {
          const double2 rv = __ldg(reinterpret_cast<const double2*>(a.r + node * g.TS * 2));
          *reinterpret_cast<double2*>(a.y + node * g.TS * 2) =
              make_double2(rv.x + ((0.0 - 0.0) - ep.x), rv.y + ((0.0 - 0.0) - ep.y));
        }
      }
    }
    // every box before xq is free: the barrier that ended the previous chunk ordered the reads
    produce_x(xq + NX);
    wait_x(xq);
    wait_r(rq);
    const unsigned rb = rbase + (rq % NR) * YBOX;
#pragma unroll
    for (int s = 0; s < CH; ++s) {
      double2 xc[5];
      xpts(xq, s, xc);
      const unsigned ra = (rb + yq) ^ ((unsigned)s << 4);
      const double2 rv = lds2u(ra);
      // four short FMA chains per component instead of two long ones
      double2 em = mv(Xm[0], xa[0]), em2 = mv(Xm[2], xa[2]);
      double2 ep = mv(Xp[0], xc[0]), ep2 = mv(Xp[2], xc[2]);
      em = mac(em, Xm[1], xa[1]);
      ep = mac(ep, Xp[1], xc[1]);
      em2 = mac(em2, Xm[3], xa[3]);
      ep2 = mac(ep2, Xp[3], xc[3]);
      em2 = mac(em2, Xm[4], xa[4]);
      ep2 = mac(ep2, Xp[4], xc[4]);
      em = add(em, em2);
      ep = add(ep, ep2);
      // y = r + (-(Xi_{t-1} x_{t-1}) - Xi_t' x_{t+1})   (the convention of gq_grid.cu)
      sts2u(ra, make_double2(rv.x + ((0.0 - em.x) - ep.x), rv.y + ((0.0 - em.y) - ep.y)));
#pragma unroll
      for (int u = 0; u < 5; ++u) {
        xa[u] = xb_[u];
        xb_[u] = xc[u];
      }
    }
    __syncthreads();
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      tma3_store(&ymap, rb, c * CH * 2, i0, j0);
      bulk_commit();
      bulk_wait_read<1>();   // the box stored one chunk ago (refilled next) has been read out
    }
    produce_r(rq + NR);
    ++rq;
    ++xq;
  }
  if (tid == 0) bulk_wait_all();
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
    else
      cudaGetLastError();
  });
  return fn;
}

}  // namespace

// "shared-memory attribute set" flags per kernel and device (one process may drive several
// GPUs in the in-process stage-slab mode)
static bool& device_flag(int kernel) {
  static bool flags[2][64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  return flags[kernel][(dev < 0 || dev >= 64) ? 63 : dev];
}

bool dstep_supported(const Geo& g) {
  return g.n == 2 && g.T >= 1 && g.T1 <= MAXT1 && encoder() != nullptr;
}

// Worth it when the grid fills the machine: a CTA walks its stages one barrier at a time, so
// a grid of a few tiles is latency-bound (config 2, 16 x 16: 24 us against 8 us for the
// lane-per-stage stencil).  GQ_DSTEP=1 forces it (tests: every golden case on this path).
bool dstep_preferred(const Geo& g, int sm_count) {
  const char* e = getenv("GQ_DSTEP");
  if (e && *e == '1') return true;
  const long long tiles = (long long)((g.K + TI - 1) / TI) * ((g.N + TJ - 1) / TJ);
  return tiles >= sm_count / 2;
}

long long dstep_max_blocks(int sm_count) { return sm_count; }

// vector v[j][i][t][k] as a 3-D tensor (2*T1 doubles, K rows, N columns); box = one chunk of
// the tile with a halo of 2 nodes (Delta input) or none (its output)
bool dstep_make_map(const Geo& g, const double* base, int halo, CUtensorMap* m) {
  EncodeTiled enc = encoder();
  if (!enc || base == nullptr) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)g.T1 * 2, (cuuint64_t)g.K, (cuuint64_t)g.N};
  const cuuint64_t strides[2] = {(cuuint64_t)g.TS * 16, (cuuint64_t)g.TS * 16 * g.K};
  const cuuint32_t box[3] = {(cuuint32_t)(CH * 2), (cuuint32_t)(TI + 2 * halo),
                             (cuuint32_t)(TJ + 2 * halo)};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
             box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// views for k_rstep: 8-stage boxes with the 128-byte swizzle, origin at stage 1 (whole lines
// of the padded layout); the x view (input = true) starts at stage 2 and carries a one-node halo
bool rstep_make_map(const Geo& g, const double* base, bool input, CUtensorMap* m) {
  EncodeTiled enc = encoder();
  if (!enc || base == nullptr) return false;
  const int stages = input ? g.T - 1 : g.T;   // from stage 2 (x) / stage 1 (r, y) on
  if (stages < 1) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)stages * 2, (cuuint64_t)g.K, (cuuint64_t)g.N};
  const cuuint64_t strides[2] = {(cuuint64_t)g.TS * 16, (cuuint64_t)g.TS * 16 * g.K};
  const cuuint32_t box[3] = {(cuuint32_t)(rs::CH * 2), (cuuint32_t)(input ? rs::QI : rs::TI),
                             (cuuint32_t)(input ? rs::QJ : rs::TJ)};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base + (input ? 4 : 2)),
             dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

cudaError_t launch_dstep(const Geo& g, const CUtensorMap& dmap, const CUtensorMap& ymap,
                         const DstepOps& op, double* y, double* partials, PcgState* st,
                         int dotmode, int sm_count, cudaStream_t s) {
  const size_t smem = (size_t)SMEM0 + 3 * (size_t)g.T1 * 4;
  bool& attr = device_flag(0);   // the attribute is per device
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_dstep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         SMEM0 + 3 * MAXT1 * 4);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int per_sm = 1;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dstep, NTHR, smem);
  if (e != cudaSuccess) return e;
  per_sm = std::max(per_sm, 1);
  DsArgs a;
  a.g = g;
  a.op = op;
  a.y = y;
  a.partials = partials;
  a.st = st;
  a.dotmode = dotmode;
  a.ntI = (g.K + TI - 1) / TI;
  const int ntJ = (g.N + TJ - 1) / TJ;
  const long long tiles = (long long)a.ntI * ntJ;
  const long long slots = (long long)per_sm * sm_count;
  // stage ranges: chunk-aligned lengths; pick the one minimising waves x (range + prologue)
  int best = ((g.T1 + CH - 1) / CH) * CH;
  long long best_cost = -1;
  for (int rl = CH; rl <= ((g.T1 + CH - 1) / CH) * CH; rl += CH) {
    const long long items = tiles * ((g.T1 + rl - 1) / rl);
    const long long cost = ((items + slots - 1) / slots) * (rl + 2 * CH);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = rl;
    }
  }
  a.RL = best;
  a.nr = (g.T1 + best - 1) / best;
  a.n_items = (int)(tiles * a.nr);
  const int blocks = (int)std::min<long long>(a.n_items, slots);
  k_dstep<<<blocks, NTHR, smem, s>>>(dmap, ymap, a);
  return cudaGetLastError();
}

cudaError_t launch_rstep(const Geo& g, const CUtensorMap& xmap, const CUtensorMap& rmap,
                         const CUtensorMap& ymap, const double* x, const double* r,
                         double* y, const double* xi, const double* xit, PcgState* st,
                         int sm_count, cudaStream_t s) {
  bool& attr = device_flag(1);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_rstep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         rs::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  RsArgs a;
  a.g = g;
  a.x = x;
  a.r = r;
  a.y = y;
  a.xi = xi;
  a.xit = xit;
  a.st = st;
  a.ntI = (g.K + rs::TI - 1) / rs::TI;
  a.nch = (g.T + rs::CH - 1) / rs::CH;   // chunk c = stages 8c + 1 .. 8c + 8
  a.tiles = a.ntI * ((g.N + rs::TJ - 1) / rs::TJ);
  const long long slots = 2LL * sm_count;
  // One piece per tile once the tiles fill the machine: the kernel is bound by DRAM traffic,
  // and CTAs that walk neighbouring tiles in step find each other's halo rows in L2 (headline:
  // 462 MB read and 0.118 ms with one piece, 580 MB and 0.141 ms with four, 584 MB and
  // 0.134 ms with equal contiguous runs of the (tile, chunk) sequence).  Small grids are cut
  // into pieces to give every CTA slot an item.
  a.pieces = a.tiles >= slots ? 1 : (int)std::max<long long>(1, std::min<long long>(a.nch, slots / a.tiles));
  if (const char* e = getenv("GQ_RS_PIECES")) a.pieces = std::max(1, std::min(a.nch, atoi(e)));
  a.total = (long long)a.tiles * a.pieces;
  const int blocks = (int)std::min<long long>(a.total, slots);
  k_rstep<<<blocks, rs::NT, rs::SMEM, s>>>(xmap, rmap, ymap, a);
  return cudaGetLastError();
}

}  // namespace gq
