// Pair-chain sweeps, CTA-cooperative and TMA-fed ("cta" kernels), n = 2.
//
// Same recurrences as the per-warp chain kernels of gq_chain.cu (block_linalg.py:336-358,
// nested_jacobi.py:85-103):
//
//   forward   w_k = L_k^-1 tau_k  - (L_k^-1 Omega~_k) theta  - G_k w_{k-1}
//   backward  x_k = L_k^-T w_k    - H_k x_{k+1}
//
// with every product an m8n8k4 fp64 DMMA, 8 chains (stages) on M.  What changes is the data
// movement.  A CTA holds CW = 5 consumer warps on ONE column pair v and 40 consecutive
// stages (warp w: stages t0 + 8w .. +7), so all five warps walk the same blocks k with the
// same factor tiles:
//
//   * one elected thread (warp 0, lane 0) feeds a ring of R shared-memory slots per block
//     step with TMA: the block's right-hand-side records for all 40 stages as ONE 3-D tensor
//     box (stages x 2 rows x 2 columns), the theta neighbour records as four column boxes,
//     and the block's factor tiles as one bulk copy.  No per-lane LDGSTS, no address math in
//     the consumers, out-of-grid rows / columns / stages arrive zero-filled by the TMA unit;
//   * a slot completes on its `full` mbarrier (transaction bytes) and is released by the five
//     consumer warps on its `empty` mbarrier; the producer refills it P = R - 1 steps ahead;
//   * a record is staged with a 2-stage pad (42 stages = 672 B), so consecutive records
//     start two 16-byte bank groups apart and the A-fragment reads of a quarter warp
//     (4 records x 2 chains) are conflict-free when the four records of a k-pair have
//     distinct indices mod 4.  The inner sweep's 16 input records (tau + 12 theta) are
//     grouped into four such k-pairs; the forward tiles are rebuilt at setup in that order
//     (k_build_cta), so the kernel reads one 8x8 B tile per k-pair.
//
// Stage 0 is handled apart: Psi_0 = Q_0^-1 is block-diagonal (kkt_assembly.py:522), so its
// pair "chain" has no coupling (G = H = 0, Omega~ = 0) and x = L^-T L^-1 tau per block.  The
// CTAs holding the first stage range of a pair solve it with one thread per block.
//
// The forward iterate w is parked in `out` (L2 evict-last) and read back by the backward
// pass through the TMA; each consumer fences its generic-proxy stores against the async
// proxy before releasing the turnaround barrier the producer waits on.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gq_async.cuh"
#include "gq_internal.h"

namespace gq {

namespace {

using namespace as;

// CW consumer warps per CTA (5 by default; 1 gives a per-warp TMA pipeline)
template <int CW>
struct Cg {
  static constexpr int CT = 32 * CW;            // threads per CTA
  static constexpr int CST = 8 * CW;            // stages per CTA item
  static constexpr int PITCH = 2 * (CST + 2);   // doubles per staged record (2-stage pad)
  static constexpr int RECB = 8 * PITCH;        // bytes per record (672 at CW = 5)
};

template <bool INNER, int CW>
struct Cc {
  static constexpr int PITCH = Cg<CW>::PITCH, RECB = Cg<CW>::RECB;
  // forward: tau box (4 records) | a-1 box (4) | a+2 box (4) | a-2 box (2) | pad (2) |
  //          a+3 box (2) | factor tiles
  static constexpr int NRF = INNER ? 18 : 4;
  static constexpr int FF = INNER ? 320 : 128;   // forward factor doubles staged per block
  static constexpr int FB = 128;                 // L^-T | -H
  static constexpr int FWD = NRF * PITCH + FF;
  static constexpr int BWD = 8 * PITCH + FB;     // w box | r box | factor tiles
  static constexpr int RAW = FWD > BWD ? FWD : BWD;
  static constexpr int SLOT = (RAW + 15) / 16 * 16;   // doubles, 128-byte multiple
  static constexpr uint32_t FWD_TX = INNER ? (3 * 4 + 2 * 2) * RECB + FF * 8 : 4 * RECB + FF * 8;
};

// record of local pair node nd (= 2 dr + dc) inside a (stages x 2 rows x 2 columns) box
__host__ __device__ constexpr int box_rec(int nd) { return (nd >> 1) + 2 * (nd & 1); }

// theta records of the inner sweep: record index -> (column offset, row offset) relative to
// (column 2v, row 2k); -99 for tau records and padding
__host__ __device__ constexpr int cta_dcol(int r) {
  return r < 4 ? -99 : r < 8 ? -1 : r < 12 ? 2 : r < 14 ? -2 : (r >= 16 && r < 18) ? 3 : -99;
}
__host__ __device__ constexpr int cta_drow(int r) {
  return r < 4 ? 0 : r < 8 ? r - 5 : r < 12 ? r - 9 : r < 14 ? r - 12 : r - 16;
}
// record read by lane quad qd for k-pair group gi (gi 0 = tau; 1..3 theta)
__host__ __device__ constexpr int cta_grec(int gi, int qd) {
  return gi == 0 ? box_rec(qd) : gi == 1 ? 4 + qd : gi == 2 ? 8 + qd : (qd < 2 ? 12 + qd : 14 + qd);
}
// theta record order of the per-warp chain tiles (gq_chain.cu th_dc / th_dr)
__host__ __device__ constexpr int th_dc2(int r) { return r < 2 ? -2 : r < 6 ? -1 : r < 10 ? 2 : 3; }
__host__ __device__ constexpr int th_dr2(int r) {
  return (r == 0 || r == 3 || r == 7 || r == 10) ? 0
       : (r == 1 || r == 4 || r == 8 || r == 11) ? 1
       : (r == 2 || r == 6) ? -1 : 2;
}

__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                     uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void stg2_last(double* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x),
               "d"(v.y), "l"(pol)
               : "memory");
}

struct CtaMaps {
  CUtensorMap rhs;    // box 84 x 2 rows x 2 cols over the sweep right-hand side
  CUtensorMap th4;    // box 84 x 4 rows x 1 col over theta
  CUtensorMap th2;    // box 84 x 2 rows x 1 col over theta
  CUtensorMap w;      // box 84 x 2 x 2 over the output (parked forward iterate)
  CUtensorMap r;      // box 84 x 2 x 2 over the dot partner (PCG residual)
};

struct CtaArgs {
  Geo g;
  const double* ff;    // forward tiles per (class, pair, block), stride 320: inner -> k-pair
                       // groups (k_build_cta), outer -> chain tiles L^-1 | -G | ...
  const double* fb;    // chain backward tiles L^-T | -H, stride 128
  const double* ff0;   // chain forward tiles (stride 320) for the stage-0 solve
  int c0, c1;          // Psi classes of stage 0 and of stages >= 1
  const double* rhs;
  const double* th;
  double* out;
  const double* rdot;
  int nch, n_items;
  double* partials;
  PcgState* st;
  int dotmode;
};

}  // namespace

template <bool INNER, int R, int CW>
__global__ void __launch_bounds__(32 * CW) k_chain_cta(const __grid_constant__ CtaMaps tm,
                                                       const CtaArgs a) {
  using C = Cc<INNER, CW>;
  constexpr int CT = Cg<CW>::CT, CST = Cg<CW>::CST, PITCH = Cg<CW>::PITCH, RECB = Cg<CW>::RECB;
  extern __shared__ unsigned char smraw[];
  if (halted(a.st)) return;
  // 128-byte aligned ring; offsetting smraw keeps the pointer in the shared window, so the
  // fragment reads compile to LDS (generic LDs are not ordered before the slot release)
  double* ring = reinterpret_cast<double*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + R * C::SLOT);
  uint64_t* empty = full + R;
  uint64_t* fwdb = empty + R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rw = lane >> 2, qd = lane & 3;
  const Geo& g = a.g;
  const bool dotting = a.dotmode != kDotNone;
  const bool producer = threadIdx.x == 0;
  if (producer) {
    for (int i = 0; i < R; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, CW);
    }
    mbar_init(fwdb, CW);
    fence_mbar_init();
    fence_proxy_async();
  }
  __syncthreads();
  const uint64_t pol_k = pol_last();
  const long long rs = (long long)g.T1 * 2, cs = (long long)g.K * rs, rs2 = 2 * rs;
  const int nb = g.nb, K = g.K;
  const uint32_t bwd_tx = (dotting ? 8 : 4) * RECB + C::FB * 8;
  double dot = 0.0;

  // A-fragment offsets (doubles into a slot): record of k-pair group gi, my chain's stage
  const int so2 = 2 * (8 * warp + rw);
  int gofs[4];
#pragma unroll
  for (int gi = 0; gi < 4; ++gi) gofs[gi] = cta_grec(gi, qd) * PITCH + so2;
  const int nofs = box_rec(qd) * PITCH + so2;       // node qd (tau / w / r boxes)
  const int bofs = rw * 8 + 2 * qd;                 // B fragment inside an 8x8 tile
  const int dr = qd >> 1, dc = qd & 1;              // my output node inside the block

  uint32_t s_issue = 0, s_use = 0, it = 0;
  // producer: issue step s_issue (forward block k or backward block k of item (v, t0))
  auto issue_fwd = [&](int v, int t0, int k) {
    const uint32_t s = s_issue++;
    const int slot = s % R;
    if (s >= (uint32_t)R) mbar_wait(empty + slot, ((s / R) - 1) & 1);
    double* sl = ring + slot * C::SLOT;
    const int col = 2 * v, e0 = 2 * t0;
    mbar_expect_tx(full + slot, C::FWD_TX);
    tma3(sl, &tm.rhs, e0, 2 * k, col, full + slot);
    if (INNER) {
      tma3(sl + 4 * PITCH, &tm.th4, e0, 2 * k - 1, col - 1, full + slot);
      tma3(sl + 8 * PITCH, &tm.th4, e0, 2 * k - 1, col + 2, full + slot);
      tma3(sl + 12 * PITCH, &tm.th2, e0, 2 * k, col - 2, full + slot);
      tma3(sl + 16 * PITCH, &tm.th2, e0, 2 * k, col + 3, full + slot);
    }
    bulk_g2s(sl + C::NRF * PITCH, a.ff + (((long long)a.c1 * g.V + v) * nb + k) * 320, C::FF * 8,
             full + slot);
  };
  auto issue_bwd = [&](int v, int t0, int k) {
    const uint32_t s = s_issue++;
    const int slot = s % R;
    if (s >= (uint32_t)R) mbar_wait(empty + slot, ((s / R) - 1) & 1);
    double* sl = ring + slot * C::SLOT;
    const int col = 2 * v, e0 = 2 * t0;
    mbar_expect_tx(full + slot, bwd_tx);
    tma3(sl, &tm.w, e0, 2 * k, col, full + slot);
    if (dotting) tma3(sl + 4 * PITCH, &tm.r, e0, 2 * k, col, full + slot);
    bulk_g2s(sl + 8 * PITCH, a.fb + (((long long)a.c1 * g.V + v) * nb + k) * 128, C::FB * 8,
             full + slot);
  };
  // Release a consumed slot.  `dep` is a value computed from every fragment read from the
  // slot: passing it into the arrive's asm makes the arrive depend on the reads' results, so
  // no read can still be in flight when the producer's next TMA overwrites the slot.
  // (arithmetic never yields this signalling-NaN pattern, so the test is always true, but the
  // compiler cannot drop the dependency and must finish the DMMAs before the arrive).
  auto release = [&](int slot, double2 dep) {
    __syncwarp();
    if (lane == 0 && __double_as_longlong(dep.x + dep.y) != 0x7FF4DEADBEEF0001LL)
      mbar_arrive1(empty + slot);
  };

#pragma unroll 1
  for (int item = blockIdx.x; item < a.n_items; item += gridDim.x, ++it) {
    const int v = item / a.nch, c = item - v * a.nch;
    const int t0 = 1 + CST * c, col = 2 * v;
    const int tw = t0 + 8 * warp;
    const int nvalid = min(8, g.T1 - tw);
    const bool ook = rw < nvalid && col + dc < g.N;
    const long long obase = (long long)(col + dc) * cs + (long long)dr * rs + (long long)(tw + rw) * 2;
    constexpr int P = R - 1;
    const int pro = P < nb ? P : nb;
    if (producer)
      for (int k = 0; k < pro; ++k) issue_fwd(v, t0, k);

    if (c == 0) {
      // stage 0: x = L^-T L^-1 tau per block (block-diagonal Phi~_{v,0}), one thread per block
      const double* F0 = a.ff0 + ((long long)a.c0 * g.V + v) * nb * 320;
      const double* B0 = a.fb + ((long long)a.c0 * g.V + v) * nb * 128;
#pragma unroll 1
      for (int k = threadIdx.x; k < nb; k += CT) {
        double tau[8], w[8];
#pragma unroll
        for (int nd = 0; nd < 4; ++nd) {
          const int r_ = 2 * k + (nd >> 1), c_ = col + (nd & 1);
          double2 tv = make_double2(0.0, 0.0);
          if (r_ < K && c_ < g.N)
            tv = __ldg(reinterpret_cast<const double2*>(a.rhs + (long long)c_ * cs + (long long)r_ * rs));
          tau[2 * nd] = tv.x;
          tau[2 * nd + 1] = tv.y;
        }
        const double* L = F0 + (long long)k * 320;
        const double* U = B0 + (long long)k * 128;
#pragma unroll
        for (int o = 0; o < 8; ++o) {
          double sacc = 0.0;
#pragma unroll
          for (int f = 0; f < 8; ++f) sacc = fma(__ldg(L + o * 8 + f), tau[f], sacc);
          w[o] = sacc;
        }
#pragma unroll
        for (int nd = 0; nd < 4; ++nd) {
          double x2[2];
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int o = 2 * nd + cc;
            double sacc = 0.0;
#pragma unroll
            for (int f = 0; f < 8; ++f) sacc = fma(__ldg(U + o * 8 + f), w[f], sacc);
            x2[cc] = sacc;
          }
          const int r_ = 2 * k + (nd >> 1), c_ = col + (nd & 1);
          if (r_ < K && c_ < g.N) {
            const long long off = (long long)c_ * cs + (long long)r_ * rs;
            *reinterpret_cast<double2*>(a.out + off) = make_double2(x2[0], x2[1]);
            if (dotting) {
              const double2 rv = __ldg(reinterpret_cast<const double2*>(a.rdot + off));
              dot = fma(x2[0], rv.x, dot);
              dot = fma(x2[1], rv.y, dot);
            }
          }
        }
      }
    }

    // ---------------- forward ----------------
    double2 wd = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int k = 0; k < nb; ++k) {
      if (producer && k + P < nb) issue_fwd(v, t0, k + P);
      __syncwarp();
      const uint32_t s = s_use++;
      const int slot = s % R;
      mbar_wait(full + slot, (s / R) & 1);
      __syncwarp();   // lanes leave the spin at different polls: reconverge before the DMMAs
      const double* sl = ring + slot * C::SLOT;
      const double* sf = sl + C::NRF * PITCH;
      double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0, g0 = a0, g1 = a0;
      if (INNER) {
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) {
          const double2 av = lds2(sl + gofs[gi]);
          const double2 b = lds2(sf + gi * 64 + bofs);
          if (gi & 1) {
            dmma(a2, av.x, b.x);
            dmma(a3, av.y, b.y);
          } else {
            dmma(a0, av.x, b.x);
            dmma(a1, av.y, b.y);
          }
        }
        const double2 bg = lds2(sf + 256 + bofs);
        dmma(g0, wd.x, bg.x);
        dmma(g1, wd.y, bg.y);
      } else {
        const double2 av = lds2(sl + nofs);
        const double2 b = lds2(sf + bofs);
        dmma(a0, av.x, b.x);
        dmma(a1, av.y, b.y);
        const double2 bg = lds2(sf + 64 + bofs);
        dmma(g0, wd.x, bg.x);
        dmma(g1, wd.y, bg.y);
      }
      double2 wn = add2(a0, a1);
      if (INNER) wn = add2(wn, add2(a2, a3));
      wn = add2(wn, add2(g0, g1));
      wd = wn;
      release(slot, wn);
      if (ook && 2 * k + dr < K) stg2_last(a.out + obase + (long long)k * rs2, wn, pol_k);
    }
    // the backward pass reads the parked w through the async proxy
    fence_async_global();
    __syncwarp();
    if (lane == 0) mbar_arrive1(fwdb);
    if (producer) {
      mbar_wait(fwdb, it & 1);
      for (int k = nb - 1; k >= 0 && k >= nb - pro; --k) issue_bwd(v, t0, k);
    }
    __syncwarp();

    // ---------------- backward ----------------
    double2 xd = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int k = nb - 1; k >= 0; --k) {
      if (producer && k - P >= 0) issue_bwd(v, t0, k - P);
      __syncwarp();
      const uint32_t s = s_use++;
      const int slot = s % R;
      mbar_wait(full + slot, (s / R) & 1);
      __syncwarp();   // lanes leave the spin at different polls: reconverge before the DMMAs
      const double* sl = ring + slot * C::SLOT;
      const double* sf = sl + 8 * PITCH;
      double2 a0 = make_double2(0.0, 0.0), a1 = a0, g0 = a0, g1 = a0;
      const double2 wv = lds2(sl + nofs);
      const double2 bl = lds2(sf + bofs), bh = lds2(sf + 64 + bofs);
      double2 rv = make_double2(0.0, 0.0);
      if (dotting) rv = lds2(sl + 4 * PITCH + nofs);
      dmma(a0, wv.x, bl.x);
      dmma(a1, wv.y, bl.y);
      dmma(g0, xd.x, bh.x);
      dmma(g1, xd.y, bh.y);
      const double2 xn = add2(add2(a0, a1), add2(g0, g1));
      xd = xn;
      release(slot, add2(xn, rv));
      if (ook && 2 * k + dr < K) {
        *reinterpret_cast<double2*>(a.out + obase + (long long)k * rs2) = xn;
        if (dotting) {
          dot = fma(xn.x, rv.x, dot);
          dot = fma(xn.y, rv.y, dot);
        }
      }
    }
  }
  if (dotting) {
    double mu;
    if (grid_reduce<false>(dot, a.partials, &a.st->counter[2], mu) && threadIdx.x == 0) {
      if (a.dotmode == kDotInit) {
        a.st->mu = mu;                       // pcg.py:92
      } else {
        a.st->beta = mu / a.st->mu;          // pcg.py:127-131
        a.st->mu = mu;
      }
    }
  }
}

// ---- setup: forward tiles in k-pair group order -----------------------------------------
// gt[(pc, v, k)][gi][o][2 qd + c] = coefficient of output o on record cta_grec(gi, qd), state
// component c;  gt[..][4] = -G.  Built from the per-warp chain tiles (gq_chain.cu, stride
// 320: L^-1 | -G | -M as 8x8 tiles, M = L^-1 Omega~ over 12 theta records).
__global__ void k_build_cta(long long nblk, const double* __restrict__ ff, double* __restrict__ gt) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= nblk * 8) return;
  const long long b = gid / 8;
  const int o = (int)(gid % 8);
  const double* F = ff + b * 320;
  double* G = gt + b * 320;
  for (int gi = 0; gi < 4; ++gi)
    for (int q = 0; q < 4; ++q)
      for (int cc = 0; cc < 2; ++cc) {
        const int rec = cta_grec(gi, q);
        double val = 0.0;
        if (rec < 4) {
          const int nd = 2 * (rec & 1) + (rec >> 1);   // box record -> local node (2 dr + dc)
          val = F[o * 8 + 2 * nd + cc];
        } else {
          const int dcol = cta_dcol(rec), drow = cta_drow(rec);
          for (int rt = 0; rt < 12; ++rt)
            if (th_dc2(rt) == dcol && th_dr2(rt) == drow) {
              const int f = 2 * rt + cc;                 // theta feature of M (8 x 24 tiles)
              val = F[128 + (f >> 3) * 64 + o * 8 + (f & 7)];
            }
        }
        G[gi * 64 + o * 8 + 2 * q + cc] = val;
      }
  for (int f = 0; f < 8; ++f) G[256 + o * 8 + f] = F[64 + o * 8 + f];
}

// max |.| of the coupling tiles (G, M, H) of one class: stage 0 must be uncoupled
__global__ void k_cta_check(long long nblk, const double* __restrict__ ff,
                            const double* __restrict__ fb, unsigned long long* bad) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= nblk) return;
  const double* F = ff + gid * 320;
  const double* B = fb + gid * 128;
  bool nz = false;
  for (int i = 64; i < 320; ++i) nz |= F[i] != 0.0;
  for (int i = 64; i < 128; ++i) nz |= B[i] != 0.0;
  if (nz) atomicAdd(bad, 1ull);
}

// ---- host side -----------------------------------------------------------------------------

namespace {

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

int env_i(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

// vector v[j][i][t][k] as a 3-D tensor (2*T1 doubles, K rows, N columns)
bool make_map(CUtensorMap* m, const Geo& g, const double* base, int rows, int cols, int pitch) {
  EncodeTiled enc = encoder();
  if (!enc || base == nullptr) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)g.T1 * 2, (cuuint64_t)g.K, (cuuint64_t)g.N};
  const cuuint64_t strides[2] = {(cuuint64_t)g.T1 * 16, (cuuint64_t)g.T1 * 16 * g.K};
  const cuuint32_t box[3] = {(cuuint32_t)pitch, (cuuint32_t)rows, (cuuint32_t)cols};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
             box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <bool INNER, int R, int CW>
cudaError_t cta_launch(const CtaMaps& tm, const CtaArgs& a, int sm_count, cudaStream_t s) {
  constexpr int CT = Cg<CW>::CT;
  // GQ_CTA_CPS caps the resident CTAs per SM (extra dynamic shared memory per CTA)
  const int cps = env_i("GQ_CTA_CPS", 0);
  size_t smem = (size_t)R * Cc<INNER, CW>::SLOT * 8 + (2 * R + 1) * 8 + 128;
  if (cps > 0) smem = std::max(smem, (size_t)(225 * 1024 / cps));
  static int cache[8][64] = {{0}};
  int per_sm = 1;
  cudaError_t e = kernel_occupancy(k_chain_cta<INNER, R, CW>, CT, smem, cache[std::min(cps, 7)], per_sm);
  if (e != cudaSuccess) return e;
  // persistent only when asked (GQ_CTA_PERSIST=1); by default one CTA per item
  int blocks = a.n_items;
  if (env_i("GQ_CTA_PERSIST", 0)) blocks = std::max(1, std::min(a.n_items, per_sm * sm_count));
  k_chain_cta<INNER, R, CW><<<blocks, CT, smem, s>>>(tm, a);
  return cudaGetLastError();
}

}  // namespace

bool cta_supported(const Geo& g, const int* pcls) {
  // opt-in (GQ_CTA=1): parity-green but slower than the per-warp chain kernel at the
  // headline size ("CTA-cooperative TMA sweep")
  if (env_i("GQ_NO_CTA", 0) || !env_i("GQ_CTA", 0)) return false;
  if (g.n != 2 || (g.N & 1) || g.T1 < 2 || encoder() == nullptr) return false;
  if (pcls[0] == pcls[1]) return false;
  for (int t = 2; t < g.T1; ++t)
    if (pcls[t] != pcls[1]) return false;
  return true;
}

cudaError_t launch_build_cta(const Geo& g, int npc, const double* ff, double* gt,
                             cudaStream_t s) {
  const long long nblk = (long long)npc * g.V * g.nb;
  k_build_cta<<<(unsigned)((nblk * 8 + 127) / 128), 128, 0, s>>>(nblk, ff, gt);
  return cudaGetLastError();
}

cudaError_t cta_check_stage0(const Geo& g, int c0, const double* ff, const double* fb,
                             bool& ok, cudaStream_t s) {
  unsigned long long* bad = nullptr;
  cudaError_t e = cudaMalloc(&bad, sizeof(unsigned long long));
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(bad, 0, sizeof(unsigned long long), s);
  const long long nblk = (long long)g.V * g.nb;
  const long long off = (long long)c0 * nblk;
  k_cta_check<<<(unsigned)((nblk + 127) / 128), 128, 0, s>>>(nblk, ff + off * 320, fb + off * 128, bad);
  unsigned long long h = 1;
  e = cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(bad);
  ok = (h == 0);
  return e;
}

template <int CW>
static cudaError_t chain_cta_w(const Geo& g, const CtaOps& co, bool inner, const double* rhs,
                               const double* th, double* out, const double* rdot, int sm_count,
                               double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  constexpr int CST = Cg<CW>::CST, PITCH = Cg<CW>::PITCH;
  CtaMaps tm;
  memset(&tm, 0, sizeof(tm));
  const bool dotting = dotmode != kDotNone;
  if (!make_map(&tm.rhs, g, rhs, 2, 2, PITCH) || !make_map(&tm.w, g, out, 2, 2, PITCH))
    return cudaErrorInvalidValue;
  if (inner && (!make_map(&tm.th4, g, th, 4, 1, PITCH) || !make_map(&tm.th2, g, th, 2, 1, PITCH)))
    return cudaErrorInvalidValue;
  if (!inner) tm.th4 = tm.th2 = tm.rhs;
  if (dotting) {
    if (!make_map(&tm.r, g, rdot, 2, 2, PITCH)) return cudaErrorInvalidValue;
  } else {
    tm.r = tm.rhs;
  }
  CtaArgs a;
  a.g = g;
  a.ff = inner ? co.gt : co.ff;
  a.fb = co.fb;
  a.ff0 = co.ff;
  a.c0 = co.c0;
  a.c1 = co.c1;
  a.rhs = rhs;
  a.th = th;
  a.out = out;
  a.rdot = rdot;
  a.nch = (g.T1 - 1 + CST - 1) / CST;
  a.n_items = g.V * a.nch;
  a.partials = partials;
  a.st = st;
  a.dotmode = dotmode;
  const int r = env_i(inner ? "GQ_CTA_R_INNER" : "GQ_CTA_R_OUTER", inner ? 3 : 5);
  if (inner) {
    if (r == 6) return cta_launch<true, 6, CW>(tm, a, sm_count, s);
    if (r == 4) return cta_launch<true, 4, CW>(tm, a, sm_count, s);
    if (r == 2) return cta_launch<true, 2, CW>(tm, a, sm_count, s);
    return cta_launch<true, 3, CW>(tm, a, sm_count, s);
  }
  if (r == 3) return cta_launch<false, 3, CW>(tm, a, sm_count, s);
  if (r == 7) return cta_launch<false, 7, CW>(tm, a, sm_count, s);
  return cta_launch<false, 5, CW>(tm, a, sm_count, s);
}

static int cta_w() { return env_i("GQ_CTA_W", 5); }

cudaError_t launch_chain_cta(const Geo& g, const CtaOps& co, bool inner, const double* rhs,
                             const double* th, double* out, const double* rdot, int sm_count,
                             double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  switch (cta_w()) {
    case 1: return chain_cta_w<1>(g, co, inner, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
    case 2: return chain_cta_w<2>(g, co, inner, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
    default: return chain_cta_w<5>(g, co, inner, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
  }
}

long long cta_max_blocks(const Geo& g) {
  return (long long)g.V * ((g.T1 - 1 + 8 - 1) / 8);   // the finest item split (CW = 1)
}

}  // namespace gq
