// Pair-chain sweeps for n = 2 with CTA-shared factor tiles on an mbarrier ring ("chainx").
//
// Same arithmetic as the per-warp chain kernel (gq_chain.cu): one warp owns 8 chains (8
// stages of one class of one column pair v) and walks the nb two-row blocks forward then
// backward (block_linalg.py:336-358, nested_jacobi.py:85-103) on m8n8k4 fp64 DMMAs:
//
//   forward   w_k = L_k^-1 tau_k  - (L_k^-1 Omega~_k) theta  - G_k w_{k-1}
//   backward  x_k = L_k^-T w_k    - H_k x_{k+1}
//
// What changes is where the factor tiles come from.  The tiles of block k depend only on
// (stage class, pair v, k), so the W warps of a CTA take W stage chunks of the SAME pair and
// class and share one copy: a producer warp streams the tiles of the 2 nb factor steps
// (forward k = 0..nb-1, then backward k = nb-1..0) with bulk copies into an R-slot ring
// (full barrier: the copy's transaction count; empty barrier: one arrival per consumer
// warp), R steps ahead of the slowest consumer.  Per warp and block that removes the
// 2.5 KB (inner forward) / 1 KB staging copy of the per-warp kernel and its share of the
// shared-memory ring, so about twice as many warps fit per SM.  Records (right-hand side,
// theta neighbours, parked forward iterate, the dot partner) stay on per-warp cp.async rings
// P blocks ahead, exactly as in the per-warp kernel.
//
// A consumer warp releases a factor slot only after the DMMAs that read it have produced
// their results (the arrive takes a DMMA output as an operand), so no shared-memory read of
// the slot can still be in flight when the producer's next bulk copy lands in it.
#include <algorithm>
#include <cstdlib>

#include "gq_async.cuh"
#include "gq_internal.h"

namespace gq {

namespace {

using namespace as;

constexpr int NS = 2, Q = 8, QQ = 64, TC = 24, KT = 3;
constexpr int FFS = 2 * QQ + Q * TC;   // forward factor doubles per block (L^-1 | -G | -M)
constexpr int FBS = 2 * QQ;            // backward factor doubles per block (L^-T | -H)
constexpr int REC = 8 * NS;            // record: 8 stages x 2 doubles
constexpr int RSTR = REC + 2 * NS;     // padded record stride (conflict-free A fragments)
constexpr int CPR = REC / 2;           // 16-byte chunks per record
constexpr int RPI = 32 / CPR;          // records per warp instruction

__host__ __device__ constexpr int th_dc(int r) {
  return r < 2 ? -2 : r < 6 ? -1 : r < 10 ? 2 : 3;
}
__host__ __device__ constexpr int th_dr(int r) {
  return (r == 0 || r == 3 || r == 7 || r == 10) ? 0
       : (r == 1 || r == 4 || r == 8 || r == 11) ? 1
       : (r == 2 || r == 6) ? -1 : 2;
}

template <bool INNER, bool FR>
struct Cx {
  static constexpr int NRF = INNER ? 16 : (FR ? 8 : 4);   // forward records per block
  static constexpr int JF = NRF / RPI, JB = 8 / RPI;
  static constexpr int FF = INNER ? FFS : 2 * QQ;        // forward factor doubles staged
  static constexpr int FSL = FF > FBS ? FF : FBS;         // factor slot (doubles)
  static constexpr int RSL = (NRF > 8 ? NRF : 8) * RSTR;  // record slot (doubles)
};

__device__ __forceinline__ void mbar_init_s(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
// Release a factor slot.  `dep` is a DMMA output computed from the slot's fragments: the
// comparison against a NaN payload no DMMA produces makes the arrive depend on it, so the
// compiler cannot hoist the arrive above the DMMAs (whose operands were the slot's LDS).
__device__ __forceinline__ void mbar_release(uint64_t* bar, double dep) {
  if (__double_as_longlong(dep) != 0x7FF4DEADBEEF0001LL)
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void stg2_keep(double* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x),
               "d"(v.y), "l"(pol)
               : "memory");
}

}  // namespace

struct ChainxArgs {
  Geo g;
  const double* ff;    // [npc][V][nb] forward tiles (ChainOps::ff)
  const double* fb;    // [npc][V][nb] backward tiles
  const int4* seg;     // class-pure chunks of <= 8 stages
  const int4* grp;     // CTA items: (first chunk, chunk count <= W, class, 0)
  int ngrp;            // items per pair
  const double* rhs;
  const double* th;
  double* out;
  const double* rdot;
  const double* yv;    // FR: r -= alpha y fused in (rhs = r, written back)
  double* rupd;
  double* partials;
  PcgState* st;
  int dotmode;
};

template <bool INNER, bool FR, int P, int R, int W>
__global__ void __launch_bounds__(32 * (W + 1)) k_chainx(const ChainxArgs a) {
  using C = Cx<INNER, FR>;
  extern __shared__ __align__(128) double smem[];
  PcgState* st = a.st;
  if (halted(st)) return;
  const Geo& g = a.g;
  const int item = blockIdx.x;
  const int v = item / a.ngrp;
  const int4 gr = a.grp[item - v * a.ngrp];
  const int nact = gr.y, cls = gr.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* fring = smem;                                   // R factor slots
  uint64_t* full = reinterpret_cast<uint64_t*>(fring + R * C::FSL);
  uint64_t* empty = full + R;
  double* ring = reinterpret_cast<double*>(empty + R) + warp * (P + 1) * C::RSL;
  const int nb = g.nb, K = g.K;
  const int nsteps = 2 * nb;
  if (threadIdx.x == 0) {
    for (int i = 0; i < R; ++i) {
      mbar_init_s(full + i, 1);
      mbar_init_s(empty + i, nact);
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  const double alpha = FR ? st->alpha : 0.0;
  double dot = 0.0, rmax = 0.0;
  const bool dotting = a.dotmode != kDotNone;

  if (warp == W) {
    // ---- producer: factor tiles of every step into the ring, R steps ahead ----
    if (lane == 0) {
      const double* ffb = a.ff + ((long long)cls * g.V + v) * nb * FFS;
      const double* fbb = a.fb + ((long long)cls * g.V + v) * nb * FBS;
      for (int s = 0; s < nsteps; ++s) {
        const int slot = s % R;
        if (s >= R) mbar_wait(empty + slot, ((s / R) - 1) & 1);
        const bool fwd = s < nb;
        const int k = fwd ? s : nsteps - 1 - s;
        const unsigned bytes = (fwd ? C::FF : FBS) * 8;
        mbar_expect_tx(full + slot, bytes);
        bulk_g2s(fring + slot * C::FSL, fwd ? ffb + (long long)k * FFS : fbb + (long long)k * FBS,
                 bytes, full + slot);
      }
    }
  } else if (warp < nact) {
    // ---- consumer warp: chunk gr.x + warp ----
    const int4 sg = a.seg[gr.x + warp];
    const int t0 = sg.x, nvalid = sg.y;
    const uint64_t pol_s = pol_first(), pol_k = pol_last();
    const int rw = lane >> 2, qd = lane & 3;
    const long long rs = (long long)g.T1 * NS;
    const long long cs = (long long)K * rs;
    const long long rs2 = 2 * rs;
    const int acol = 2 * v;
    const bool okb = acol + 1 < g.N;
    const long long col_a = (long long)acol * cs + (long long)t0 * NS;
    const int wch = lane % CPR;
    const int wst = wch / (NS / 2);
    const bool stage_ok = wst < nvalid;
    const int wofs = stage_ok ? 2 * wch : 0;
    const unsigned ring_u = smem_u32(ring);
    auto aofs = [&](int rec, int f0) { return (rec + f0 / NS) * RSTR + rw * NS + (f0 % NS); };
    const int R1 = P + 1;

    // forward record sources (tau / y: the pair's own four nodes; theta: twelve neighbours)
    const double* fsrc[C::JF];
    int fsz[C::JF], frow[C::JF];
#pragma unroll
    for (int j = 0; j < C::JF; ++j) {
      const int r = j * RPI + lane / CPR;
      const bool own = r < 4 || FR;
      const int dc = own ? (r & 1) : th_dc(r - 4);
      const int dr = own ? ((r & 3) >> 1) : th_dr(r - 4);
      const bool colok = acol + dc >= 0 && acol + dc < g.N;
      fsz[j] = (colok && stage_ok) ? 16 : 0;
      frow[j] = dr;
      fsrc[j] = (r < 4 ? a.rhs : (FR ? a.yv : a.th)) + col_a + (long long)(colok ? dc : 0) * cs +
                (long long)dr * rs + wofs;
    }
    const unsigned rec_dst = lane_opaque(ring_u + (unsigned)(((lane / CPR) * RSTR + 2 * wch) * 8));
    auto issue_f = [&](int k, int slot, bool chk) {
      const unsigned sb = lane_opaque((unsigned)(slot * C::RSL * 8));
#pragma unroll
      for (int j = 0; j < C::JF; ++j) {
        const int row = 2 * k + frow[j];
        const bool ok = fsz[j] && (!chk || (row >= 0 && row < K));
        ldgsts(rec_dst + sb + j * RPI * RSTR * 8, ok ? fsrc[j] + k * rs2 : a.rhs, ok ? 16 : 0,
               pol_s);
      }
    };
    // output fragment: features 2qd, 2qd+1 of chain (stage) rw
    const int f0 = 2 * qd, nd = f0 / NS, cc = f0 % NS;
    const int orow = nd >> 1;
    const long long oofs = col_a + (long long)(nd & 1) * cs + (long long)(nd >> 1) * rs + rw * NS + cc;
    const bool ook = rw < nvalid && ((nd & 1) ? okb : true);

    {
      const int pro = P < nb ? P : nb;
      for (int p = 0; p < pro; ++p) {
        issue_f(p, p, true);
        commit();
      }
      for (int p = pro; p < P; ++p) commit();
    }
    double2 wd = make_double2(0.0, 0.0);
    int slot = 0, islot = P % R1;
#pragma unroll 1
    for (int k = 0; k < nb; ++k) {
      const int kk = k + P;
      if (kk < nb) issue_f(kk, islot, kk == nb - 1 || kk == 0);
      commit();
      wait_groups<P>();
      const int fs = k % R;
      mbar_wait(full + fs, (k / R) & 1);
      __syncwarp();
      const double* sl = ring + slot * C::RSL;
      const double* sf = fring + fs * C::FSL;
      double2 tv = lds2(sl + aofs(0, 2 * qd));
      if constexpr (FR) {
        // r -= alpha y (pcg.py:111) on the staged records; written back, feeds max|r|
        const double2 yy = lds2(sl + aofs(4, 2 * qd));
        tv.x = __dsub_rn(tv.x, __dmul_rn(alpha, yy.x));
        tv.y = __dsub_rn(tv.y, __dmul_rn(alpha, yy.y));
        if (ook && !(k == nb - 1 && 2 * k + orow >= K)) {
          *reinterpret_cast<double2*>(a.rupd + oofs + (long long)k * rs2) = tv;
          rmax = nmax(rmax, nmax(fabs(tv.x), fabs(tv.y)));
        }
      }
      double2 a0 = make_double2(0.0, 0.0), a1 = a0, g0 = a0, g1 = a0, m0 = a0, m1 = a0, m2 = a0,
              m3 = a0;
      {
        const double2 b = lds2(sf + rw * 8 + 2 * qd);
        dmma(a0, tv.x, b.x);
        dmma(a1, tv.y, b.y);
      }
      if constexpr (INNER) {
#pragma unroll
        for (int p = 0; p < KT; ++p) {
          const double2 b = lds2(sf + 2 * QQ + p * 64 + rw * 8 + 2 * qd);
          const double2 tq = lds2(sl + aofs(4, 8 * p + 2 * qd));
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
        const double2 b = lds2(sf + QQ + rw * 8 + 2 * qd);
        dmma(g0, wd.x, b.x);
        dmma(g1, wd.y, b.y);
      }
      double2 sm = add2(a0, a1);
      if (INNER) sm = add2(sm, add2(add2(m0, m1), add2(m2, m3)));
      const double2 wn = add2(sm, add2(g0, g1));
      __syncwarp();
      if (lane == 0) mbar_release(empty + fs, wn.x + wn.y);
      wd = wn;
      if (ook && !(k == nb - 1 && 2 * k + orow >= K))
        stg2_keep(a.out + oofs + (long long)k * rs2, wn, pol_k);
      slot = slot + 1 == R1 ? 0 : slot + 1;
      islot = islot + 1 == R1 ? 0 : islot + 1;
      __syncwarp();
    }
    wait_groups<0>();
    __threadfence();
    __syncwarp();

    // ---------------- backward ----------------
    const double* bsrc[C::JB];
    int bsz[C::JB], brow[C::JB];
#pragma unroll
    for (int j = 0; j < C::JB; ++j) {
      const int r = j * RPI + lane / CPR;
      const int dc = r & 1, dr = (r >> 1) & 1;
      const bool ok = stage_ok && (dc ? okb : true) && (r < 4 || dotting);
      bsz[j] = ok ? 16 : 0;
      brow[j] = dr;
      bsrc[j] = (r < 4 ? (const double*)a.out : (dotting ? a.rdot : a.rhs)) + col_a +
                (long long)(dc && okb ? 1 : 0) * cs + (long long)dr * rs + wofs;
    }
    auto issue_b = [&](int k, int slot_) {
      const unsigned sb = lane_opaque((unsigned)(slot_ * C::RSL * 8));
#pragma unroll
      for (int j = 0; j < C::JB; ++j) {
        const bool ok = bsz[j] && 2 * k + brow[j] < K;
        ldgsts(rec_dst + sb + j * RPI * RSTR * 8, ok ? bsrc[j] + k * rs2 : a.rhs, ok ? 16 : 0,
               pol_s);
      }
    };
    {
      const int pro = P < nb ? P : nb;
      for (int p = 0; p < pro; ++p) {
        issue_b(nb - 1 - p, p);
        commit();
      }
      for (int p = pro; p < P; ++p) commit();
    }
    double2 xd = make_double2(0.0, 0.0);
    slot = 0;
    islot = P % R1;
#pragma unroll 1
    for (int k = nb - 1; k >= 0; --k) {
      const int kk = k - P;
      if (kk >= 0) issue_b(kk, islot);
      commit();
      wait_groups<P>();
      const int s = nsteps - 1 - k, fs = s % R;
      mbar_wait(full + fs, (s / R) & 1);
      __syncwarp();
      const double* sl = ring + slot * C::RSL;
      const double* sf = fring + fs * C::FSL;
      const double2 wv = lds2(sl + aofs(0, 2 * qd));
      double2 a0 = make_double2(0.0, 0.0), a1 = a0, g0 = a0, g1 = a0;
      {
        const double2 b = lds2(sf + rw * 8 + 2 * qd);
        dmma(a0, wv.x, b.x);
        dmma(a1, wv.y, b.y);
      }
      {
        const double2 b = lds2(sf + QQ + rw * 8 + 2 * qd);
        dmma(g0, xd.x, b.x);
        dmma(g1, xd.y, b.y);
      }
      const double2 xn = add2(add2(a0, a1), add2(g0, g1));
      __syncwarp();
      if (lane == 0) mbar_release(empty + fs, xn.x + xn.y);
      xd = xn;
      if (ook && !(k == nb - 1 && 2 * k + orow >= K)) {
        *reinterpret_cast<double2*>(a.out + oofs + (long long)k * rs2) = xn;
        if (dotting) {
          const double2 rv = lds2(sl + aofs(4, 2 * qd));
          dot = fma(xn.x, rv.x, dot);
          dot = fma(xn.y, rv.y, dot);
        }
      }
      slot = slot + 1 == R1 ? 0 : slot + 1;
      islot = islot + 1 == R1 ? 0 : islot + 1;
      __syncwarp();
    }
    wait_groups<0>();
    __syncwarp();
  }

  if constexpr (FR) {
    // max |r| over the grid, then the reference's history / convergence step (pcg.py:113-121)
    double res;
    if (grid_reduce<true>(rmax, a.partials, &st->counter[1], res) && threadIdx.x == 0) {
      st->res = res;
      st->hist[st->step] = res;
      st->step += 1;
      if (res < st->tol && !st->defer) {
        st->converged = 1;
        st->done = 1;
      }
    }
  }
  if (dotting) {
    double mu;
    if (grid_reduce<false>(dot, a.partials, &st->counter[2], mu) && threadIdx.x == 0) {
      if (a.dotmode == kDotInit) {
        st->mu = mu;                       // pcg.py:92
      } else {
        st->beta = mu / st->mu;            // pcg.py:127-131
        st->mu = mu;
      }
    }
  }
}

// ---- host side ---------------------------------------------------------------------------

namespace {
int cx_env(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}
constexpr int kW = 5;   // consumer warps per CTA (T = 200: 25 class-1 chunks = 5 groups)
}  // namespace

bool chainx_supported(const Geo& g) { return g.n == 2 && cx_env("GQ_CHAINX", 0) == 1; }
int chainx_warps() { return kW; }

template <bool INNER, bool FR, int P, int R>
static cudaError_t chainx_launch(const ChainxArgs& a, int n_items, cudaStream_t s) {
  using C = Cx<INNER, FR>;
  constexpr size_t smem = (size_t)R * C::FSL * 8 + 2 * R * 8 + (size_t)kW * (P + 1) * C::RSL * 8;
  static int cache[64] = {0};
  int per_sm = 1;
  cudaError_t e = kernel_occupancy(k_chainx<INNER, FR, P, R, kW>, 32 * (kW + 1), smem, cache, per_sm);
  if (e != cudaSuccess) return e;
  k_chainx<INNER, FR, P, R, kW><<<n_items, 32 * (kW + 1), smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_chainx(const Geo& g, const ChainOps& co, const int4* grp, int ngrp, bool inner,
                          const double* rhs, const double* th, double* out, const double* rdot,
                          double* partials, PcgState* st, int dotmode, const double* yv,
                          double* rupd, cudaStream_t s) {
  ChainxArgs a;
  a.g = g;
  a.ff = co.ff;
  a.fb = co.fb;
  a.seg = co.seg;
  a.grp = grp;
  a.ngrp = ngrp;
  a.rhs = rhs;
  a.th = th;
  a.out = out;
  a.rdot = rdot;
  a.yv = yv;
  a.rupd = rupd;
  a.partials = partials;
  a.st = st;
  a.dotmode = dotmode;
  const int n_items = g.V * ngrp;
  if (yv != nullptr) return chainx_launch<false, true, 6, 8>(a, n_items, s);
  if (inner) return chainx_launch<true, false, 3, 6>(a, n_items, s);
  return chainx_launch<false, false, 6, 8>(a, n_items, s);
}

}  // namespace gq
