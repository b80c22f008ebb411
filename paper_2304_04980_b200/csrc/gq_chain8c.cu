// Pair-chain sweeps for n = 8 with CTA-shared factor tiles ("chain8c").
//
// Same recurrences as gq_chain.cu (block_linalg.py:336-358, nested_jacobi.py:85-103) at
// n = 8 (q = 32, every 8x8 tile one DMMA k-pair), but a CTA of W warps works on ONE column
// pair and W consecutive class-pure stage chunks, so the warps walk the same blocks with the
// same factor tiles.  The tiles of a block (L^-1 | -G and, for inner sweeps, the 20 raw
// cross-pair Psi blocks of its four nodes: 26 KB; L^-T | -H: 16 KB) are copied ONCE per CTA
// with cp.async into a double buffer and read by all warps as LDS -- the per-warp kernel
// reads them from L2 once per warp.  Records stay on per-warp LDGSTS rings; one block of
// prefetch, two CTA barriers per block step (the step itself is ~100-200 DMMAs per warp).
#include <algorithm>
#include <cstdlib>

#include "gq_async.cuh"
#include "gq_internal.h"

namespace gq {

namespace {

using namespace as;

constexpr int NS8 = 8, Q8 = 32, QQ8 = 1024, NT8 = 4;
constexpr int REC8 = 80;   // 8 stages x 8 states, padded by 16 doubles (bank groups)
constexpr int OMB = 320;   // cross-pair blocks per node: 5 x 64

__host__ __device__ constexpr int c8_thdc(int r) { return r < 2 ? -2 : r < 6 ? -1 : r < 10 ? 2 : 3; }
__host__ __device__ constexpr int c8_thdr(int r) {
  return (r == 0 || r == 3 || r == 7 || r == 10) ? 0
       : (r == 1 || r == 4 || r == 8 || r == 11) ? 1
       : (r == 2 || r == 6) ? -1 : 2;
}
__host__ __device__ constexpr int c8_threc(int dc, int u) {
  return dc == 0 ? (u == 0 ? 0 : u == 1 ? 2 : u == 2 ? 3 : u == 3 ? 4 : 7)
                 : (u == 0 ? 3 : u == 1 ? 6 : u == 2 ? 7 : u == 3 ? 8 : 10);
}

__device__ __forceinline__ void stg2_last8(double* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x),
               "d"(v.y), "l"(pol)
               : "memory");
}

template <bool INNER>
struct C8 {
  static constexpr int NRF = INNER ? 16 : 4;
  static constexpr int SLOT = (NRF > 8 ? NRF : 8) * REC8;             // doubles per ring slot
  static constexpr int FBUF = INNER ? 2 * QQ8 + 4 * OMB : 2 * QQ8;    // doubles per factor buffer
};

}  // namespace

template <bool INNER, int W>
__global__ void __launch_bounds__(32 * W, INNER ? 1 : 2) k_chain8c(Geo g, ChainOps co,
                                                       const double* __restrict__ rhs,
                                                       const double* __restrict__ th, double* out,
                                                       const double* __restrict__ rdot,
                                                       int n_items, double* partials,
                                                       PcgState* st, int dotmode) {
  using C = C8<INNER>;
  extern __shared__ __align__(128) double sm8[];
  if (halted(st)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, rw = lane >> 2, qd = lane & 3;
  const int tid = threadIdx.x;
  double* fbuf = sm8;                                   // [2][FBUF]
  double* ring = sm8 + 2 * C::FBUF + warp * 2 * C::SLOT;   // [2][SLOT] for this warp
  const unsigned fbuf_u = smem_u32(fbuf), ring_u = smem_u32(ring);
  const uint64_t pol_k = pol_last();
  const bool dotting = dotmode != kDotNone;
  const long long rs = (long long)g.TS * NS8, cs = (long long)g.K * rs, rs2 = 2 * rs;
  const int nb = g.nb, K = g.K;
  double dot = 0.0;

#pragma unroll 1
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int v = item / co.ngrp;
    const int4 gr = co.grp[item - v * co.ngrp];
    const int cls = gr.z;
    const bool wv = warp < gr.y;
    const int4 sg = co.seg[gr.x + (wv ? warp : 0)];
    const int t0 = sg.x, nvalid = wv ? sg.y : 0;
    const int a = 2 * v;
    const long long col_a = (long long)a * cs + (long long)t0 * NS8;
    const int wst = lane >> 2;                    // stage of my 16-byte record chunk
    const bool stage_ok = wst < nvalid;
    const int wofs = stage_ok ? 2 * lane : 0;
    const long long fblk = (long long)cls * g.V + v;   // (class, pair) block base

    // output fragment addressing: tile h = node h (dr = h >> 1, dc = h & 1)
    long long oofs[NT8];
    bool ook[NT8];
#pragma unroll
    for (int h = 0; h < NT8; ++h) {
      oofs[h] = col_a + (long long)(h & 1) * cs + (long long)(h >> 1) * rs + rw * NS8 + 2 * qd;
      ook[h] = rw < nvalid && a + (h & 1) < g.N;
    }
    // cooperative factor copies into buffer `b`
    auto copy_ff = [&](int k, int b) {
      const double* src = co.ff + (fblk * nb + k) * (2 * QQ8 + Q8 * 12 * NS8);
      constexpr int NCH = C::FBUF / 2;
      const unsigned dst0 = fbuf_u + (unsigned)(b * C::FBUF * 8);
      for (int c = tid; c < NCH; c += 32 * W) {
        const double* sp = nullptr;
        bool ok = true;
        if (c < QQ8) {
          sp = src + 2 * c;
        } else {
          const int e = c - QQ8, nd = e / (OMB / 2), off = e % (OMB / 2);
          const int row = 2 * k + (nd >> 1), col = a + (nd & 1);
          ok = row < K && col < g.N;
          sp = ok ? co.omega + (((long long)cls * g.nk + (long long)col * K + row) * 5) * 64 + 2 * off
                  : src;
        }
        ldgsts(dst0 + 16u * c, sp, ok ? 16 : 0, 0);
      }
    };
    auto copy_fb = [&](int k, int b) {
      const double* src = co.fb + (fblk * nb + k) * (2 * QQ8);
      const unsigned dst0 = fbuf_u + (unsigned)(b * C::FBUF * 8);
      for (int c = tid; c < QQ8; c += 32 * W) ldgsts(dst0 + 16u * c, src + 2 * c, 16, 0);
    };

    // ---------------- forward ----------------
    const double* fsrc[C::NRF];
    bool fcol[C::NRF];
    int frow[C::NRF];
#pragma unroll
    for (int j = 0; j < C::NRF; ++j) {
      const bool own = j < 4;
      const int dc = own ? (j & 1) : c8_thdc(j - 4);
      const int dr = own ? (j >> 1) : c8_thdr(j - 4);
      fcol[j] = stage_ok && a + dc >= 0 && a + dc < g.N;
      frow[j] = dr;
      fsrc[j] = (own ? rhs : th) + col_a + (long long)(fcol[j] ? dc : 0) * cs + (long long)dr * rs + wofs;
    }
    const unsigned rdst = lane_opaque(ring_u + 16u * lane);
    auto issue_f = [&](int k, int slot) {
#pragma unroll
      for (int j = 0; j < C::NRF; ++j) {
        const int row = 2 * k + frow[j];
        const bool ok = fcol[j] && row >= 0 && row < K;
        ldgsts(rdst + (unsigned)((slot * C::SLOT + j * REC8) * 8), ok ? fsrc[j] + (long long)k * rs2 : rhs,
               ok ? 16 : 0, 0);
      }
    };
    __syncthreads();   // the previous item's readers are done with the buffers
    issue_f(0, 0);
    copy_ff(0, 0);
    commit();
    double2 wd[NT8];
#pragma unroll
    for (int h = 0; h < NT8; ++h) wd[h] = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int k = 0; k < nb; ++k) {
      const int b = k & 1;
      if (k + 1 < nb) {
        __syncthreads();   // buffer / slot b^1 (block k-1) is free
        issue_f(k + 1, b ^ 1);
        copy_ff(k + 1, b ^ 1);
      }
      commit();
      wait_groups<1>();
      __syncthreads();     // block k's records and tiles are visible
      const double* sl = ring + b * C::SLOT;
      const double* sf = fbuf + b * C::FBUF;
      double2 z[NT8];
#pragma unroll
      for (int p = 0; p < NT8; ++p) z[p] = lds2(sl + p * REC8 + rw * NS8 + 2 * qd);
      if (INNER) {
        // z = tau - Psi_cross theta (nested_jacobi.py:85-103 with Omega~ = -Psi_cross)
#pragma unroll
        for (int p = 0; p < NT8; ++p) {
          const int dr = p >> 1, dc = p & 1;
          double2 s0 = make_double2(0.0, 0.0), s1 = s0;
#pragma unroll
          for (int u = 0; u < 5; ++u) {
            const double2 tq = lds2(sl + (4 + c8_threc(dc, u) + dr) * REC8 + rw * NS8 + 2 * qd);
            const double2 bb = lds2(sf + 2 * QQ8 + p * OMB + u * 64 + rw * 8 + 2 * qd);
            if (u & 1) {
              dmma(s1, tq.x, bb.x);
              dmma(s1, tq.y, bb.y);
            } else {
              dmma(s0, tq.x, bb.x);
              dmma(s0, tq.y, bb.y);
            }
          }
          z[p].x = z[p].x - (s0.x + s1.x);
          z[p].y = z[p].y - (s0.y + s1.y);
        }
      }
      double2 wn[NT8];
#pragma unroll
      for (int h = 0; h < NT8; ++h) {
        double2 a0 = make_double2(0.0, 0.0), a1 = a0, g0 = a0, g1 = a0;
#pragma unroll
        for (int p = 0; p < NT8; ++p) {
          const double2 bl = lds2(sf + (h * NT8 + p) * 64 + rw * 8 + 2 * qd);
          dmma(a0, z[p].x, bl.x);
          dmma(a1, z[p].y, bl.y);
          const double2 bg = lds2(sf + QQ8 + (h * NT8 + p) * 64 + rw * 8 + 2 * qd);
          dmma(g0, wd[p].x, bg.x);
          dmma(g1, wd[p].y, bg.y);
        }
        wn[h] = add2(add2(a0, a1), add2(g0, g1));
      }
#pragma unroll
      for (int h = 0; h < NT8; ++h) {
        wd[h] = wn[h];
        if (ook[h] && 2 * k + (h >> 1) < K) stg2_last8(out + oofs[h] + (long long)k * rs2, wn[h], pol_k);
      }
    }
    wait_groups<0>();
    __threadfence();   // the parked w is read back by this warp's own LDGSTS below
    __syncthreads();

    // ---------------- backward ----------------
    const double* bsrc[8];
    bool bok[8];
    int brow[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int dc = j & 1, dr = (j >> 1) & 1;
      bok[j] = stage_ok && a + dc < g.N && (j < 4 || dotting);
      brow[j] = dr;
      bsrc[j] = (j < 4 ? (const double*)out : (dotting ? rdot : rhs)) + col_a +
                (long long)(a + dc < g.N ? dc : 0) * cs + (long long)dr * rs + wofs;
    }
    auto issue_b = [&](int k, int slot) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool ok = bok[j] && 2 * k + brow[j] < K;
        ldgsts(rdst + (unsigned)((slot * C::SLOT + j * REC8) * 8), ok ? bsrc[j] + (long long)k * rs2 : rhs,
               ok ? 16 : 0, 0);
      }
    };
    issue_b(nb - 1, 0);
    copy_fb(nb - 1, 0);
    commit();
    double2 xd[NT8];
#pragma unroll
    for (int h = 0; h < NT8; ++h) xd[h] = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int i = 0; i < nb; ++i) {
      const int k = nb - 1 - i, b = i & 1;
      if (k > 0) {
        __syncthreads();
        issue_b(k - 1, b ^ 1);
        copy_fb(k - 1, b ^ 1);
      }
      commit();
      wait_groups<1>();
      __syncthreads();
      const double* sl = ring + b * C::SLOT;
      const double* sf = fbuf + b * C::FBUF;
      double2 wv[NT8];
#pragma unroll
      for (int p = 0; p < NT8; ++p) wv[p] = lds2(sl + p * REC8 + rw * NS8 + 2 * qd);
      double2 xn[NT8];
#pragma unroll
      for (int h = 0; h < NT8; ++h) {
        double2 a0 = make_double2(0.0, 0.0), a1 = a0, g0 = a0, g1 = a0;
#pragma unroll
        for (int p = 0; p < NT8; ++p) {
          const double2 bl = lds2(sf + (h * NT8 + p) * 64 + rw * 8 + 2 * qd);
          dmma(a0, wv[p].x, bl.x);
          dmma(a1, wv[p].y, bl.y);
          const double2 bh = lds2(sf + QQ8 + (h * NT8 + p) * 64 + rw * 8 + 2 * qd);
          dmma(g0, xd[p].x, bh.x);
          dmma(g1, xd[p].y, bh.y);
        }
        xn[h] = add2(add2(a0, a1), add2(g0, g1));
      }
#pragma unroll
      for (int h = 0; h < NT8; ++h) {
        xd[h] = xn[h];
        if (ook[h] && 2 * k + (h >> 1) < K) {
          *reinterpret_cast<double2*>(out + oofs[h] + (long long)k * rs2) = xn[h];
          if (dotting) {
            const double2 rv = lds2(sl + (4 + h) * REC8 + rw * NS8 + 2 * qd);
            dot = fma(xn[h].x, rv.x, dot);
            dot = fma(xn[h].y, rv.y, dot);
          }
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

static int c8env(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

bool chain8c_enabled() { return c8env("GQ_NO_CHAIN8C", 0) == 0; }

template <bool INNER>
static cudaError_t chain8c_launch(const Geo& g, const ChainOps& co, const double* rhs,
                                  const double* th, double* out, const double* rdot,
                                  int sm_count, double* partials, PcgState* st, int dotmode,
                                  cudaStream_t s) {
  constexpr int W = 8;
  constexpr size_t smem = (size_t)(2 * C8<INNER>::FBUF + W * 2 * C8<INNER>::SLOT) * sizeof(double);
  static int cache[64] = {0};
  int per_sm = 1;
  cudaError_t e = kernel_occupancy(k_chain8c<INNER, W>, 32 * W, smem, cache, per_sm);
  if (e != cudaSuccess) return e;
  const int n_items = g.V * co.ngrp;
  const int blocks = std::max(1, std::min(n_items, per_sm * sm_count));
  k_chain8c<INNER, W><<<blocks, 32 * W, smem, s>>>(g, co, rhs, th, out, rdot, n_items, partials,
                                                  st, dotmode);
  return cudaGetLastError();
}

cudaError_t launch_chain8c(const Geo& g, const ChainOps& co, bool inner, const double* rhs,
                           const double* th, double* out, const double* rdot, int sm_count,
                           double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  return inner ? chain8c_launch<true>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s)
               : chain8c_launch<false>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
}

}  // namespace gq
