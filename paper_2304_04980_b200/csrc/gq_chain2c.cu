// Pair-chain sweeps for n = 2 with CTA-shared factor tiles ("chain2c"), opt-in GQ_CHAIN2C=1.
//
// The per-warp chain kernel of gq_chain.cu stages each block's factor tiles (2.5 KB inner,
// 1 KB outer/backward) into every warp's ring.  Here a CTA of W warps works on one column
// pair and W consecutive class-1 stage chunks; the tiles are copied once per CTA into a ring
// of P+1 slots (one 16-byte cp.async per thread and block) and read by all warps, while the
// records keep the per-warp LDGSTS rings.  Per-warp shared memory drops from 5 KB to 2.5 KB
// per slot (inner), so twice the warps fit.  Two CTA barriers per block step.  Stage 0
// (block-diagonal Phi~_{v,0}: G = H = Omega~ = 0, checked at setup) is solved by the threads
// of the first CTA of each pair, x = L^-T L^-1 tau per block.
#include <algorithm>
#include <cstdlib>

#include "gq_async.cuh"
#include "gq_internal.h"

namespace gq {

namespace {

using namespace as;

constexpr int Q2 = 8, QQ2 = 64, REC2 = 20;   // record: 8 stages x 2 states, padded to 20

__host__ __device__ constexpr int c2_thdc(int r) { return r < 2 ? -2 : r < 6 ? -1 : r < 10 ? 2 : 3; }
__host__ __device__ constexpr int c2_thdr(int r) {
  return (r == 0 || r == 3 || r == 7 || r == 10) ? 0
       : (r == 1 || r == 4 || r == 8 || r == 11) ? 1
       : (r == 2 || r == 6) ? -1 : 2;
}
__device__ __forceinline__ void stg2_last2(double* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x),
               "d"(v.y), "l"(pol)
               : "memory");
}

template <bool INNER>
struct C2 {
  static constexpr int NRF = INNER ? 16 : 4;                 // forward records
  static constexpr int SLOT = (NRF > 8 ? NRF : 8) * REC2;    // record ring slot (doubles)
  static constexpr int FF = INNER ? 320 : 128;               // forward factor doubles
  static constexpr int FS = FF;                              // factor ring slot (>= 128)
};

}  // namespace

template <bool INNER, int W, int P>
__global__ void __launch_bounds__(32 * W) k_chain2c(Geo g, ChainOps co, const double* __restrict__ rhs,
                                                    const double* __restrict__ th, double* out,
                                                    const double* __restrict__ rdot, int n_items,
                                                    double* partials, PcgState* st, int dotmode) {
  using C = C2<INNER>;
  constexpr int R = P + 1;
  extern __shared__ __align__(16) double sm2[];
  if (halted(st)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, rw = lane >> 2, qd = lane & 3;
  const int tid = threadIdx.x;
  double* fring = sm2;                                       // [R][FS]
  double* ring = sm2 + R * C::FS + warp * R * C::SLOT;       // [R][SLOT] of this warp
  const unsigned fring_u = smem_u32(fring), ring_u = smem_u32(ring);
  const uint64_t pol_k = pol_last();
  const bool dotting = dotmode != kDotNone;
  const long long rs = (long long)g.T1 * 2, cs = (long long)g.K * rs, rs2 = 2 * rs;
  const int nb = g.nb, K = g.K;
  double dot = 0.0;
  // lane -> record chunk: 8 chunks (16 B) per record, 4 records per warp instruction
  const int wch = lane & 7, wrec = lane >> 3;
  const int bofs = rw * 8 + 2 * qd;

#pragma unroll 1
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int v = item / co.ngrp, gi = item - v * co.ngrp;
    const int4 gr = co.grp[gi];
    const int cls = gr.z;
    const bool wv = warp < gr.y;
    const int4 sg = co.seg[gr.x + (wv ? warp : 0)];
    const int t0 = sg.x, nvalid = wv ? sg.y : 0;
    const int a = 2 * v;
    const bool okb = a + 1 < g.N;
    const long long col_a = (long long)a * cs + (long long)t0 * 2;
    const bool stage_ok = (wch >> 0) < 8 && wch < nvalid;     // chunk wch = stage wch
    const int wofs = stage_ok ? 2 * wch : 0;
    const long long fblk = (long long)cls * g.V + v;
    const int dr = qd >> 1, dc = qd & 1;                     // my output node (chain rw)
    const long long oofs = col_a + (long long)dc * cs + (long long)dr * rs + rw * 2;
    const bool ook = rw < nvalid && (dc ? okb : true);

    __syncthreads();   // previous item done with the rings
    // ---- stage 0 (first CTA of the pair): x = L^-T L^-1 tau per block ----
    if (gi == 0 && co.c0 >= 0) {
      const double* F0 = co.ff + ((long long)co.c0 * g.V + v) * nb * 320;
      const double* B0 = co.fb + ((long long)co.c0 * g.V + v) * nb * 128;
      for (int k = tid; k < nb; k += 32 * W) {
        double tau[8], w[8];
#pragma unroll
        for (int nd = 0; nd < 4; ++nd) {
          const int r_ = 2 * k + (nd >> 1), c_ = a + (nd & 1);
          double2 tv = make_double2(0.0, 0.0);
          if (r_ < K && c_ < g.N)
            tv = __ldg(reinterpret_cast<const double2*>(rhs + (long long)c_ * cs + (long long)r_ * rs));
          tau[2 * nd] = tv.x;
          tau[2 * nd + 1] = tv.y;
        }
        const double* L = F0 + (long long)k * 320;
        const double* U = B0 + (long long)k * 128;
#pragma unroll
        for (int o = 0; o < 8; ++o) {
          double s = 0.0;
#pragma unroll
          for (int f = 0; f < 8; ++f) s = fma(__ldg(L + o * 8 + f), tau[f], s);
          w[o] = s;
        }
#pragma unroll
        for (int nd = 0; nd < 4; ++nd) {
          double x2[2];
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            double s = 0.0;
#pragma unroll
            for (int f = 0; f < 8; ++f) s = fma(__ldg(U + (2 * nd + cc) * 8 + f), w[f], s);
            x2[cc] = s;
          }
          const int r_ = 2 * k + (nd >> 1), c_ = a + (nd & 1);
          if (r_ < K && c_ < g.N) {
            const long long off = (long long)c_ * cs + (long long)r_ * rs;
            *reinterpret_cast<double2*>(out + off) = make_double2(x2[0], x2[1]);
            if (dotting) {
              const double2 rv = __ldg(reinterpret_cast<const double2*>(rdot + off));
              dot = fma(x2[0], rv.x, dot);
              dot = fma(x2[1], rv.y, dot);
            }
          }
        }
      }
    }

    // ---------------- forward ----------------
    const double* fsrc[C::NRF / 4];
    bool fok[C::NRF / 4];
    int frow[C::NRF / 4];
#pragma unroll
    for (int j = 0; j < C::NRF / 4; ++j) {
      const int r = 4 * j + wrec;
      const bool own = r < 4;
      const int cdc = own ? (r & 1) : c2_thdc(r - 4);
      const int cdr = own ? (r >> 1) : c2_thdr(r - 4);
      fok[j] = stage_ok && a + cdc >= 0 && a + cdc < g.N;
      frow[j] = cdr;
      fsrc[j] = (own ? rhs : th) + col_a + (long long)(fok[j] ? cdc : 0) * cs + (long long)cdr * rs + wofs;
    }
    const unsigned rdst = lane_opaque(ring_u + (unsigned)((wrec * REC2 + 2 * wch) * 8));
    const double* ffv = co.ff + fblk * nb * 320;
    auto issue_f = [&](int k) {
      const int slot = k % R;
#pragma unroll
      for (int j = 0; j < C::NRF / 4; ++j) {
        const int row = 2 * k + frow[j];
        const bool ok = fok[j] && row >= 0 && row < K;
        ldgsts(rdst + (unsigned)((slot * C::SLOT + 4 * j * REC2) * 8),
               ok ? fsrc[j] + (long long)k * rs2 : rhs, ok ? 16 : 0, 0);
      }
      for (int c = tid; c < C::FF / 2; c += 32 * W)
        ldgsts(fring_u + (unsigned)((slot * C::FS + 2 * c) * 8), ffv + (long long)k * 320 + 2 * c, 16, 0);
    };
    const int pro = P < nb ? P : nb;
    for (int k = 0; k < pro; ++k) {
      issue_f(k);
      commit();
    }
    for (int k = pro; k < P; ++k) commit();
    double2 wd = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int k = 0; k < nb; ++k) {
      __syncthreads();              // slot (k + P) % R (block k - 1) is free in every warp
      if (k + P < nb) issue_f(k + P);
      commit();
      wait_groups<P>();
      __syncthreads();              // block k's tiles (copied by all threads) are visible
      const int slot = k % R;
      const double* sl = ring + slot * C::SLOT;
      const double* sf = fring + slot * C::FS;
      // A fragments: tau (record = node qd), theta k-pairs (records 4 + 4p + qd)
      const double2 tv = lds2(sl + qd * REC2 + rw * 2);
      double2 a0 = make_double2(0.0, 0.0), a1 = a0, g0 = a0, g1 = a0, m0 = a0, m1 = a0, m2 = a0, m3 = a0;
      {
        const double2 b = lds2(sf + bofs);
        dmma(a0, tv.x, b.x);
        dmma(a1, tv.y, b.y);
      }
      if (INNER) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const double2 b = lds2(sf + 2 * QQ2 + p * 64 + bofs);
          const double2 tq = lds2(sl + (4 + 4 * p + qd) * REC2 + rw * 2);
          if (p & 1) {
            dmma(m2, tq.x, b.x);
            dmma(m3, tq.y, b.y);
          } else {
            dmma(m0, tq.x, b.x);
            dmma(m1, tq.y, b.y);
          }
        }
      }
      {
        const double2 b = lds2(sf + QQ2 + bofs);
        dmma(g0, wd.x, b.x);
        dmma(g1, wd.y, b.y);
      }
      double2 sm = add2(a0, a1);
      if (INNER) sm = add2(sm, add2(add2(m0, m1), add2(m2, m3)));
      const double2 wn = add2(sm, add2(g0, g1));
      wd = wn;
      if (ook && 2 * k + dr < K) stg2_last2(out + oofs + (long long)k * rs2, wn, pol_k);
    }
    wait_groups<0>();
    __threadfence();
    __syncthreads();

    // ---------------- backward ----------------
    const double* bsrc[2];
    bool bok[2];
    int brow[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int r = 4 * j + wrec;
      const int bdc = r & 1, bdr = (r >> 1) & 1;
      bok[j] = stage_ok && (bdc ? okb : true) && (r < 4 || dotting);
      brow[j] = bdr;
      bsrc[j] = (r < 4 ? (const double*)out : (dotting ? rdot : rhs)) + col_a +
                (long long)(bdc && okb ? 1 : 0) * cs + (long long)bdr * rs + wofs;
    }
    const double* fbv = co.fb + fblk * nb * 128;
    auto issue_b = [&](int i) {   // i-th backward step = block nb - 1 - i
      const int k = nb - 1 - i, slot = i % R;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const bool ok = bok[j] && 2 * k + brow[j] < K;
        ldgsts(rdst + (unsigned)((slot * C::SLOT + 4 * j * REC2) * 8),
               ok ? bsrc[j] + (long long)k * rs2 : rhs, ok ? 16 : 0, 0);
      }
      for (int c = tid; c < 64; c += 32 * W)
        ldgsts(fring_u + (unsigned)((slot * C::FS + 2 * c) * 8), fbv + (long long)k * 128 + 2 * c, 16, 0);
    };
    for (int i = 0; i < pro; ++i) {
      issue_b(i);
      commit();
    }
    for (int i = pro; i < P; ++i) commit();
    double2 xd = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int i = 0; i < nb; ++i) {
      const int k = nb - 1 - i;
      __syncthreads();
      if (i + P < nb) issue_b(i + P);
      commit();
      wait_groups<P>();
      __syncthreads();
      const int slot = i % R;
      const double* sl = ring + slot * C::SLOT;
      const double* sf = fring + slot * C::FS;
      const double2 wv = lds2(sl + qd * REC2 + rw * 2);
      double2 a0 = make_double2(0.0, 0.0), a1 = a0, g0 = a0, g1 = a0;
      const double2 bl = lds2(sf + bofs), bh = lds2(sf + QQ2 + bofs);
      dmma(a0, wv.x, bl.x);
      dmma(a1, wv.y, bl.y);
      dmma(g0, xd.x, bh.x);
      dmma(g1, xd.y, bh.y);
      const double2 xn = add2(add2(a0, a1), add2(g0, g1));
      xd = xn;
      if (ook && 2 * k + dr < K) {
        *reinterpret_cast<double2*>(out + oofs + (long long)k * rs2) = xn;
        if (dotting) {
          const double2 rv = lds2(sl + (4 + qd) * REC2 + rw * 2);
          dot = fma(xn.x, rv.x, dot);
          dot = fma(xn.y, rv.y, dot);
        }
      }
    }
    wait_groups<0>();
  }
  if (dotting) {
    double mu;
    if (grid_reduce<false>(dot, partials, &st->counter[2], mu) && threadIdx.x == 0) {
      if (dotmode == kDotInit) {
        st->mu = mu;                       // pcg.py:92
      } else {
        st->beta = mu / st->mu;            // pcg.py:127-131
        st->mu = mu;
      }
    }
  }
}

static int c2env(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

bool chain2c_enabled() { return c2env("GQ_CHAIN2C", 0) == 1; }

template <bool INNER, int W, int P>
static cudaError_t chain2c_launch(const Geo& g, const ChainOps& co, const double* rhs,
                                  const double* th, double* out, const double* rdot,
                                  int sm_count, double* partials, PcgState* st, int dotmode,
                                  cudaStream_t s) {
  constexpr size_t smem = (size_t)((P + 1) * C2<INNER>::FS + W * (P + 1) * C2<INNER>::SLOT) * sizeof(double);
  static int cache[64] = {0};
  int per_sm = 1;
  cudaError_t e = kernel_occupancy(k_chain2c<INNER, W, P>, 32 * W, smem, cache, per_sm);
  if (e != cudaSuccess) return e;
  const int n_items = g.V * co.ngrp;
  const int blocks = std::max(1, std::min(n_items, per_sm * sm_count));
  k_chain2c<INNER, W, P><<<blocks, 32 * W, smem, s>>>(g, co, rhs, th, out, rdot, n_items,
                                                     partials, st, dotmode);
  return cudaGetLastError();
}

cudaError_t launch_chain2c(const Geo& g, const ChainOps& co, bool inner, const double* rhs,
                           const double* th, double* out, const double* rdot, int sm_count,
                           double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  const int p = c2env(inner ? "GQ_CHAIN2C_P_INNER" : "GQ_CHAIN2C_P_OUTER", inner ? 4 : 7);
  if (inner)
    return p == 2 ? chain2c_launch<true, 5, 2>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s)
                  : chain2c_launch<true, 5, 4>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
  return p == 4 ? chain2c_launch<false, 5, 4>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s)
                : chain2c_launch<false, 5, 7>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
}

}  // namespace gq
