// Pair-chain sweeps on the fp64 tensor cores, CTA-shared factor tiles (n = 2).
//
// Same recurrences and the same arithmetic as gq_chain.cu (block_linalg.py:336-358,
// nested_jacobi.py:85-103):
//
//   forward   w_k = L_k^-1 tau_k  - (L_k^-1 Omega~_k) theta  - G_k w_{k-1}
//   backward  x_k = L_k^-T w_k    - H_k x_{k+1}
//
// with 8 consecutive stages of one column pair on the M dimension of m8n8k4 DMMAs.  The
// per-warp kernel of gq_chain.cu copies each block's factor tiles (3.5 KB) and twelve theta
// neighbour records per warp: 8-9 KB through L2 and ~125 L1 wavefronts per block for 2.5-3 KB
// of vector data, and it runs at the L2 -> SM and L1 data-pipe limits.  Here:
//
//   * A CTA (the only one of its SM) takes up to W stage chunks of ONE column pair and one
//     stage class.  A producer warp streams the pair's factor tiles block by block into a
//     D-slot shared-memory ring with bulk (TMA) copies, one copy per CTA and block instead of
//     one per warp; the W consumer warps read their B fragments from the ring.  full/empty
//     mbarriers per slot couple the warps only loosely: a warp may run D - 2 blocks ahead of
//     the slowest one.
//   * The theta records of the two middle columns at rows 2k+1, 2k+2 are the rows -1, 0 of the
//     next block: their A fragments are carried in registers, so a block fetches eight theta
//     records instead of twelve (record order in gq_chain.cuh).
//   * Only the records go through the per-warp cp.async ring (1.9 KB per slot).
//   * The loop-carried G w / H x products are issued first in each block.
//   * Stage 0 (Psi_0 = Q_0^-1: block-diagonal, no coupling along the chain or across pairs,
//     verified on the device at setup) is solved apart, one thread per block.
#include <algorithm>
#include <cstdlib>

#include "gq_chain.cuh"

namespace gq {

namespace {

using namespace as;

__device__ __forceinline__ void stg2_park(double* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p),
               "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void stg2_out(double* p, double2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(v.x), "d"(v.y)
               : "memory");
}
// vector data read once (prologue fragments): bypass L1
__device__ __forceinline__ double2 ldcg2(const double* p) {
  return __ldcg(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <bool INNER, bool FR, bool DOT>
struct Cm {
  static constexpr int NS = 2;
  static constexpr int Q = 4 * NS, QQ = Q * Q;
  static constexpr int TC = 12 * NS;                  // theta feature count of the M tile
  static constexpr int KT = TC / 8;                   // its k-pairs ...
  static constexpr int KC = KT / 3;                   // ... of which the first KC are carried
  static constexpr int FFS = 2 * QQ + Q * TC;         // forward factor doubles per block
  static constexpr int FF = INNER ? FFS : 2 * QQ;     // ... used by this sweep
  static constexpr int FB = 2 * QQ;                   // backward factor doubles per block
  static constexpr int TS = FF > FB ? FF : FB;        // doubles per tile-ring slot
  static constexpr int REC = 8 * NS;                  // record: 8 stages x NS
  static constexpr int RSTR = REC + 2 * NS;           // padded stride (conflict-free A reads)
  static constexpr int CPR = REC / 2;                 // 16-byte chunks per record
  static constexpr int RPI = 32 / CPR;                // records per warp copy instruction
  // forward records: tau (4), then theta records 4..11 (inner) or y (4, fused r update)
  static constexpr int NRF = INNER ? 12 : (FR ? 8 : 4);
  static constexpr int NRB = DOT ? 8 : 4;             // backward: w (4) [+ r (4) for q.r]
  static constexpr int JF = NRF / RPI, JB = NRB / RPI;
  static constexpr int SLOT = (NRF > NRB ? NRF : NRB) * RSTR;   // doubles per record slot
};

// what a sweep reads and writes besides the chain itself
struct SweepIo {
  const double* rhs;
  const double* th;
  double* out;
  const double* rdot;
  const double* yv;
  double* rupd;
  double alpha;
};

// One chain (8 stages of pair v from stage t0) forward and backward.  `tiles` is the CTA's
// factor ring; step q of the CTA's tile stream (q0 + k forward, q0 + nb + (nb-1-k) backward)
// lives in slot q % D.
template <bool INNER, bool FR, bool DOT, int P, int D>
__device__ __forceinline__ void chains_item(const Geo& g, const SweepIo& io, double* ring,
                                            const double* tiles, uint64_t* full,
                                            uint64_t* empty, unsigned q0, int v, int t0,
                                            int nvalid, uint64_t pol_k, double& dot,
                                            double& rmax) {
  using C = Cm<INNER, FR, DOT>;
  constexpr int NS = 2, QQ = C::QQ, KT = C::KT, KC = C::KC, REC = C::RSTR, R = P + 1;
  const int lane = threadIdx.x & 31, rw = lane >> 2, qd = lane & 3;
  const long long rs = (long long)g.T1 * NS;
  const long long cs = (long long)g.K * rs;
  const long long rs2 = 2 * rs;
  const int nb = g.nb, K = g.K;
  const int a = 2 * v;
  const bool okb = a + 1 < g.N;
  const long long col_a = (long long)a * cs + (long long)t0 * NS;
  const int wch = lane % C::CPR;                         // my 16-byte chunk of a record
  const int wst = wch / (NS / 2);                        // ... and the stage it belongs to
  const bool stage_ok = wst < nvalid;
  const int wofs = stage_ok ? 2 * wch : 0;               // stage-invalid lanes read stage 0
  const unsigned ring_u = smem_u32(ring);
  const double* rhs = io.rhs;
  // A-fragment offset of feature pair f0 = 8p + 2qd of chain rw inside a record slot
  auto aofs = [&](int f0) { return (f0 / NS) * REC + rw * NS + (f0 % NS); };
  const int bofs = rw * 8 + 2 * qd;                      // my B-fragment pair inside a tile

  // ---------------- forward ----------------
  const double* fsrc[C::JF];
  int fsz[C::JF], frow[C::JF];
#pragma unroll
  for (int j = 0; j < C::JF; ++j) {
    const int r = j * C::RPI + lane / C::CPR;
    const bool own = r < 4 || FR;                    // tau or y: the pair's own four nodes
    const int dc = own ? (r & 1) : th_dc(r);
    const int dr = own ? ((r & 3) >> 1) : th_dr(r);
    const bool colok = a + dc >= 0 && a + dc < g.N;
    fsz[j] = (colok && stage_ok) ? 16 : 0;
    frow[j] = dr;
    // off-grid columns are redirected to the pair's own column (never read: size 0)
    fsrc[j] = (r < 4 ? rhs : (FR ? io.yv : io.th)) + col_a + (long long)(colok ? dc : 0) * cs +
              (long long)dr * rs + wofs;
  }
  // per-lane shared destination, kept in a vector register (no [R + UR] LDGSTS forms)
  const unsigned rec_dst = lane_opaque(ring_u + (unsigned)(((lane / C::CPR) * REC + 2 * wch) * 8));

  // last block (and the prologue): rows outside [0, K) zero-fill
  auto issue_f_chk = [&](int k, int slot) {
    const unsigned sb = lane_opaque((unsigned)(slot * C::SLOT * 8));
#pragma unroll
    for (int j = 0; j < C::JF; ++j) {
      const bool ok = fsz[j] && 2 * k + frow[j] < K;
      ldgsts(rec_dst + sb + j * C::RPI * REC * 8, ok ? fsrc[j] + k * rs2 : rhs, ok ? 16 : 0, 0);
    }
  };

  double2 wd = make_double2(0.0, 0.0);

  // output fragment addressing: lane holds features 2qd, 2qd+1 (node qd) of chain (stage) rw
  const int orow = qd >> 1;
  const long long oofs = col_a + (long long)(qd & 1) * cs + (long long)orow * rs + rw * NS;
  const bool ook = rw < nvalid && ((qd & 1) ? okb : true);

  // carried theta fragments of block 0: rows -1 (zero) and 0 of the two middle columns
  double2 carry[KC];
  if constexpr (INNER) {
#pragma unroll
    for (int p = 0; p < KC; ++p) {
      const int f0 = 8 * p + 2 * qd, rec = f0 / NS, cc = f0 % NS;
      const int dc = th_dc(rec), dr = th_dr(rec);
      const bool ok = dr == 0 && a + dc >= 0 && a + dc < g.N && rw < nvalid;
      carry[p] = ok ? ldcg2(io.th + col_a + (long long)dc * cs + rw * NS + cc)
                    : make_double2(0.0, 0.0);
    }
  }

  {
    const int pro = P < nb ? P : nb;
#pragma unroll 1
    for (int p = 0; p < pro; ++p) {
      issue_f_chk(p, p);
      commit();
    }
#pragma unroll 1
    for (int p = pro; p < P; ++p) commit();
  }
  // running sources of block k + P
  const double* fcur[C::JF];
#pragma unroll
  for (int j = 0; j < C::JF; ++j) fcur[j] = fsz[j] ? fsrc[j] + (long long)P * rs2 : rhs;

  int slot = 0, islot = P % R;
  unsigned q = q0;
#pragma unroll 1
  for (int k = 0; k < nb; ++k, ++q) {
    const int kk = k + P;
    if (kk < nb) {
      if (kk == nb - 1) {
        issue_f_chk(kk, islot);
      } else {
        const unsigned sb = lane_opaque((unsigned)(islot * C::SLOT * 8));
#pragma unroll
        for (int j = 0; j < C::JF; ++j)
          ldgsts(rec_dst + sb + j * C::RPI * REC * 8, fcur[j], fsz[j], 0);
      }
    }
    commit();
#pragma unroll
    for (int j = 0; j < C::JF; ++j)
      if (fsz[j]) fcur[j] += rs2;
    // this block's factor tiles: L^-1 | -G | -M
    const unsigned ts = q % D;
    mbar_wait(full + ts, (q / D) & 1u);
    __syncwarp();
    const double* sf = tiles + ts * C::TS + bofs;
    const double2 bl = lds2(sf), bg = lds2(sf + QQ);
    double2 bm[INNER ? KT : 1];
    if constexpr (INNER) {
#pragma unroll
      for (int p = 0; p < KT; ++p) bm[p] = lds2(sf + 2 * QQ + p * 64);
    }
    // loop-carried product first: -G w_{k-1}
    double2 g0 = make_double2(0.0, 0.0), g1 = g0;
    dmma(g0, wd.x, bg.x);
    dmma(g1, wd.y, bg.y);
    wait_groups<P>();
    __syncwarp();

    const double* sl = ring + slot * C::SLOT;
    double2 tv = lds2(sl + aofs(2 * qd));
    if constexpr (FR) {
      // r -= alpha y (pcg.py:111) on the staged records; the updated residual is this sweep's
      // right-hand side, is written back, and feeds max|r| (pcg.py:113)
      const double2 yy = lds2(sl + 4 * REC + aofs(2 * qd));
      tv.x = __dsub_rn(tv.x, __dmul_rn(io.alpha, yy.x));
      tv.y = __dsub_rn(tv.y, __dmul_rn(io.alpha, yy.y));
      if (ook && !(k == nb - 1 && 2 * k + orow >= K)) {
        stg2_out(io.rupd + oofs + (long long)k * rs2, tv);
        rmax = nmax(rmax, nmax(fabs(tv.x), fabs(tv.y)));
      }
    }
    double2 a0 = make_double2(0.0, 0.0), a1 = a0, m0 = a0, m1 = a0, m2 = a0, m3 = a0;
    dmma(a0, tv.x, bl.x);
    dmma(a1, tv.y, bl.y);
    if constexpr (INNER) {
      double2 tq[KT];
#pragma unroll
      for (int p = 0; p < KC; ++p) tq[p] = carry[p];
#pragma unroll
      for (int p = KC; p < KT; ++p) tq[p] = lds2(sl + aofs(8 * p + 2 * qd));
#pragma unroll
      for (int p = 0; p < KC; ++p) carry[p] = tq[KC + p];
#pragma unroll
      for (int p = 0; p < KT; ++p) {
        if (p & 1) {
          dmma(m2, tq[p].x, bm[p].x);
          dmma(m3, tq[p].y, bm[p].y);
        } else {
          dmma(m0, tq[p].x, bm[p].x);
          dmma(m1, tq[p].y, bm[p].y);
        }
      }
    }
    // every B fragment of the slot has been consumed by an issued DMMA: release it
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + ts);
    double2 sm = add2(a0, a1);
    if constexpr (INNER) sm = add2(sm, add2(add2(m0, m1), add2(m2, m3)));
    wd = add2(sm, add2(g0, g1));
    if (ook && !(k == nb - 1 && 2 * k + orow >= K))
      stg2_park(io.out + oofs + (long long)k * rs2, wd, pol_k);
    slot = slot + 1 == R ? 0 : slot + 1;
    islot = islot + 1 == R ? 0 : islot + 1;
    __syncwarp();
  }
  wait_groups<0>();
  // w was stored by other lanes of this warp: order the stores before the copies that read
  // them back.  CTA scope is enough (same SM, L1 bypassed both ways).
  __threadfence_block();
  __syncwarp();

  // ---------------- backward ----------------
  const double* bsrc[C::JB];
  int bsz[C::JB], brow[C::JB];
#pragma unroll
  for (int j = 0; j < C::JB; ++j) {
    const int r = j * C::RPI + lane / C::CPR;
    const int dc = r & 1, dr = (r >> 1) & 1;
    const bool ok = stage_ok && (dc ? okb : true);
    bsz[j] = ok ? 16 : 0;
    brow[j] = dr;
    bsrc[j] = (r < 4 ? (const double*)io.out : io.rdot) + col_a +
              (long long)(dc && okb ? 1 : 0) * cs + (long long)dr * rs + wofs;
  }
  auto issue_b_chk = [&](int k, int slot_) {
    const unsigned sb = lane_opaque((unsigned)(slot_ * C::SLOT * 8));
#pragma unroll
    for (int j = 0; j < C::JB; ++j) {
      const bool ok = bsz[j] && 2 * k + brow[j] < K;
      ldgsts(rec_dst + sb + j * C::RPI * REC * 8, ok ? bsrc[j] + k * rs2 : rhs, ok ? 16 : 0, 0);
    }
  };
  {
    const int pro = P < nb ? P : nb;
#pragma unroll 1
    for (int p = 0; p < pro; ++p) {
      issue_b_chk(nb - 1 - p, p);
      commit();
    }
#pragma unroll 1
    for (int p = pro; p < P; ++p) commit();
  }
  const double* bcur[C::JB];
#pragma unroll
  for (int j = 0; j < C::JB; ++j)
    bcur[j] = bsz[j] ? bsrc[j] + (long long)(nb - 1 - P) * rs2 : rhs;

  double2 xd = make_double2(0.0, 0.0);
  slot = 0;
  islot = P % R;
#pragma unroll 1
  for (int k = nb - 1; k >= 0; --k, ++q) {
    const int kk = k - P;
    if (kk >= 0) {
      const unsigned sb = lane_opaque((unsigned)(islot * C::SLOT * 8));
#pragma unroll
      for (int j = 0; j < C::JB; ++j)
        ldgsts(rec_dst + sb + j * C::RPI * REC * 8, bcur[j], bsz[j], 0);
    }
    commit();
#pragma unroll
    for (int j = 0; j < C::JB; ++j)
      if (bsz[j]) bcur[j] -= rs2;
    // this block's factor tiles: L^-T | -H
    const unsigned ts = q % D;
    mbar_wait(full + ts, (q / D) & 1u);
    __syncwarp();
    const double* sf = tiles + ts * C::TS + bofs;
    const double2 bl = lds2(sf), bh = lds2(sf + QQ);
    // loop-carried product first: -H x_{k+1}
    double2 g0 = make_double2(0.0, 0.0), g1 = g0;
    dmma(g0, xd.x, bh.x);
    dmma(g1, xd.y, bh.y);
    wait_groups<P>();
    __syncwarp();

    const double* sl = ring + slot * C::SLOT;
    const double2 wv = lds2(sl + aofs(2 * qd));
    double2 a0 = make_double2(0.0, 0.0), a1 = a0;
    dmma(a0, wv.x, bl.x);
    dmma(a1, wv.y, bl.y);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + ts);
    xd = add2(add2(a0, a1), add2(g0, g1));
    if (ook && !(k == nb - 1 && 2 * k + orow >= K)) {
      stg2_out(io.out + oofs + (long long)k * rs2, xd);
      if constexpr (DOT) {
        const double2 rv = lds2(sl + 4 * REC + aofs(2 * qd));
        dot = fma(xd.x, rv.x, dot);
        dot = fma(xd.y, rv.y, dot);
      }
    }
    slot = slot + 1 == R ? 0 : slot + 1;
    islot = islot + 1 == R ? 0 : islot + 1;
    __syncwarp();
  }
  wait_groups<0>();
  __syncwarp();
}

// Stage 0 of pair v, block k, by one thread: Psi_0 = Q_0^-1 couples nothing outside the
// block (G = H = M = 0 for its class, checked by k_cls0_check at setup), so
// x = L^-T L^-1 tau.  Tiles of an 8 x 8 matrix are the matrix itself, row-major.
template <bool FR, bool DOT>
__device__ void stage0_block(const Geo& g, const ChainOps& co, const SweepIo& io, int v, int k,
                             int t0, int cls, double& dot, double& rmax) {
  constexpr int NS = 2, Q = 8;
  using C = Cm<true, false, false>;
  const int a = 2 * v;
  double tau[Q], rr[Q];
  long long idx[4];
  bool ok[4];
#pragma unroll
  for (int nd = 0; nd < 4; ++nd) {
    const int col = a + (nd & 1), row = 2 * k + (nd >> 1);
    ok[nd] = col < g.N && row < g.K;
    idx[nd] = ok[nd] ? vidx(g, col, row, t0) : 0;
    double2 t = make_double2(0.0, 0.0);
    if (ok[nd]) {
      t = ldcg2(io.rhs + idx[nd]);
      if constexpr (FR) {
        const double2 yy = ldcg2(io.yv + idx[nd]);
        t.x = __dsub_rn(t.x, __dmul_rn(io.alpha, yy.x));
        t.y = __dsub_rn(t.y, __dmul_rn(io.alpha, yy.y));
        stg2_out(io.rupd + idx[nd], t);
        rmax = nmax(rmax, nmax(fabs(t.x), fabs(t.y)));
      }
    }
    tau[NS * nd] = t.x;
    tau[NS * nd + 1] = t.y;
    rr[NS * nd] = rr[NS * nd + 1] = 0.0;
    if constexpr (DOT) {
      if (ok[nd]) {
        const double2 r2 = ldcg2(io.rdot + idx[nd]);
        rr[NS * nd] = r2.x;
        rr[NS * nd + 1] = r2.y;
      }
    }
  }
  const double* F = co.ff + (((long long)cls * g.V + v) * g.nb + k) * C::FFS;
  const double* B = co.fb + (((long long)cls * g.V + v) * g.nb + k) * C::FB;
  double w[Q], x[Q];
#pragma unroll
  for (int p = 0; p < Q; ++p) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c <= p; ++c) s = fma(__ldg(F + p * Q + c), tau[c], s);
    w[p] = s;
  }
#pragma unroll
  for (int p = 0; p < Q; ++p) {
    double s = 0.0;
#pragma unroll
    for (int c = p; c < Q; ++c) s = fma(__ldg(B + p * Q + c), w[c], s);
    x[p] = s;
  }
#pragma unroll
  for (int nd = 0; nd < 4; ++nd)
    if (ok[nd]) {
      stg2_out(io.out + idx[nd], make_double2(x[NS * nd], x[NS * nd + 1]));
      if constexpr (DOT) {
        dot = fma(x[NS * nd], rr[NS * nd], dot);
        dot = fma(x[NS * nd + 1], rr[NS * nd + 1], dot);
      }
    }
}

// Deterministic CTA + grid reduction: lane sums/maxes by butterfly, warp partials folded in
// warp order by thread 0, CTA partials folded by the last CTA.
template <bool MAX>
__device__ bool cta_grid_reduce(double v, double* red, double* partials, unsigned int* counter,
                                double& outv) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = MAX ? warp_max(v) : warp_sum(v);
  __shared__ int is_last;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = red[0];
    for (int i = 1; i < nw; ++i) acc = MAX ? nmax(acc, red[i]) : acc + red[i];
    partials[blockIdx.x] = acc;
    __threadfence();
    is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last || w != 0) return false;
  __threadfence();
  double acc = 0.0;
  for (int b = lane; b < (int)gridDim.x; b += 32) {
    const double p = __ldcg(partials + b);
    acc = MAX ? nmax(acc, p) : acc + p;
  }
  acc = MAX ? warp_max(acc) : warp_sum(acc);
  outv = acc;
  if (lane == 0) *counter = 0u;
  return lane == 0;
}

// Group = up to W consecutive chunks (co.seg[co.s0 ..], all of one class) of one pair; groups
// of a pair are consecutive, CTA b takes groups b, b + gridDim.x, ...
template <bool INNER, bool FR, bool DOT, int P, int W, int D>
__global__ void __launch_bounds__(32 * (W + 1), 1)
    k_chains(Geo g, ChainOps co, SweepIo io, double* partials, PcgState* st, int dotmode) {
  extern __shared__ __align__(128) double smem_all[];
  using C = Cm<INNER, FR, DOT>;
  if (halted(st)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* tiles = smem_all;
  uint64_t* full = reinterpret_cast<uint64_t*>(tiles + D * C::TS);
  uint64_t* empty = full + D;
  double* red = reinterpret_cast<double*>(empty + D);
  double* ring = red + 32 + (size_t)warp * (P + 1) * C::SLOT;
  if (threadIdx.x == 0) {
    for (int i = 0; i < D; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, W);
    }
    fence_proxy_async();
  }
  __syncthreads();
  if constexpr (FR) io.alpha = st->alpha;
  double rmax = 0.0, dot = 0.0;
  const uint64_t pol_k = pol_last();
  const int nb = g.nb;
  const int nchunk = co.nseg - co.s0;
  const int gpp = (nchunk + W - 1) / W;            // groups per pair
  const int per = (nchunk + gpp - 1) / gpp;        // chunks per group (the last may be short)
  const int ngroups = g.V * gpp;
  const int cls = co.seg[co.s0].z;
  unsigned q0 = 0;
#pragma unroll 1
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x, q0 += 2u * nb) {
    const int v = grp / gpp, h = grp - v * gpp;
    const int c0 = co.s0 + h * per;
    const int nact = min(per, co.nseg - c0);
    if (warp == W) {
      // producer: forward tiles of blocks 0..nb-1, then backward tiles of blocks nb-1..0
      if (lane == 0) {
        const double* ffp = co.ff + ((long long)cls * g.V + v) * nb * C::FFS;
        const double* fbp = co.fb + ((long long)cls * g.V + v) * nb * C::FB;
#pragma unroll 1
        for (int i = 0; i < 2 * nb; ++i) {
          const unsigned q = q0 + i, ts = q % D;
          mbar_wait(empty + ts, ((q / D) & 1u) ^ 1u);
          const bool fwd = i < nb;
          const unsigned bytes = (fwd ? C::FF : C::FB) * 8;
          mbar_expect_tx(full + ts, bytes);
          bulk_g2s(tiles + ts * C::TS,
                   fwd ? ffp + (long long)i * C::FFS : fbp + (long long)(2 * nb - 1 - i) * C::FB,
                   bytes, full + ts);
        }
      }
      __syncwarp();
    } else {
      if (co.s0 && warp < nact) {
        // stage 0 of this pair: blocks [h nb / gpp, (h+1) nb / gpp) spread over the group's
        // warps, one block per thread
        const int b0 = (int)((long long)h * nb / gpp), b1 = (int)((long long)(h + 1) * nb / gpp);
        const int4 s0 = co.seg[0];
        for (int k = b0 + warp * 32 + lane; k < b1; k += nact * 32)
          stage0_block<FR, DOT>(g, co, io, v, k, s0.x, s0.z, dot, rmax);
        __syncwarp();
      }
      if (warp < nact) {
        const int4 sg = co.seg[c0 + warp];
        chains_item<INNER, FR, DOT, P, D>(g, io, ring, tiles, full, empty, q0, v, sg.x, sg.y,
                                          pol_k, dot, rmax);
      } else {
        // no chunk for this warp in this group: keep the slot accounting going
#pragma unroll 1
        for (int i = 0; i < 2 * nb; ++i) {
          const unsigned q = q0 + i, ts = q % D;
          mbar_wait(full + ts, (q / D) & 1u);
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + ts);
        }
      }
    }
  }
  if constexpr (FR) {
    // max |r| over the grid, then the reference's history / convergence step (pcg.py:113-121)
    double res;
    if (cta_grid_reduce<true>(rmax, red, partials, &st->counter[1], res)) {
      st->res = res;
      st->hist[st->step] = res;
      st->step += 1;
      if (res < st->tol && !st->defer) {
        st->converged = 1;
        st->done = 1;
      }
    }
  }
  if constexpr (DOT) {
    double mu;
    if (cta_grid_reduce<false>(dot, red, partials, &st->counter[2], mu)) {
      if (dotmode == kDotInit) {
        st->mu = mu;                       // pcg.py:92
      } else {
        st->beta = mu / st->mu;            // pcg.py:127-131
        st->mu = mu;
      }
    }
  }
}

// flag = 1 if any G, H or M entry of class `cls` is non-zero
__global__ void k_cls0_check(Geo g, ChainOps co, int cls, int* flag) {
  using C = Cm<true, false, false>;
  const long long nblk = (long long)g.V * g.nb;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= nblk) return;
  const double* F = co.ff + ((long long)cls * nblk + gid) * C::FFS;
  const double* B = co.fb + ((long long)cls * nblk + gid) * C::FB;
  bool nz = false;
  for (int i = C::QQ; i < C::FFS; ++i) nz |= F[i] != 0.0;
  for (int i = C::QQ; i < C::FB; ++i) nz |= B[i] != 0.0;
  if (nz) *flag = 1;
}

int env_or(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

template <bool INNER, bool FR, bool DOT, int P, int W, int D>
cudaError_t chains_launch(const Geo& g, const ChainOps& co, const SweepIo& io, int sm_count,
                          double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  using C = Cm<INNER, FR, DOT>;
  constexpr size_t smem = ((size_t)D * C::TS + 2 * D + 32 + (size_t)W * (P + 1) * C::SLOT) * 8;
  static_assert(smem <= 227 * 1024, "shared memory budget");
  static bool configured[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 63;
  auto kern = k_chains<INNER, FR, DOT, P, W, D>;
  if (!configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured[dev] = true;
  }
  const int nchunk = co.nseg - co.s0;
  const int ngroups = g.V * ((nchunk + W - 1) / W);
  const int blocks = std::max(1, std::min(ngroups, sm_count));
  kern<<<blocks, 32 * (W + 1), smem, s>>>(g, co, io, partials, st, dotmode);
  return cudaGetLastError();
}

}  // namespace

// Which sweeps the CTA-shared kernel can run: n = 2, every stage chunk of one class except an
// optional leading stage-0 chunk whose class has no coupling (checked on the device).
cudaError_t chainm_plan(const Geo& g, ChainOps& co, const int4* host_segs, cudaStream_t s) {
  co.cm = 0;
  co.s0 = 0;
  if (g.n != 2 || co.nseg < 1 || env_or("GQ_NO_CHAINM", 0)) return cudaSuccess;
  int s0 = 0;
  if (co.nseg > 1 && host_segs[0].x == 0 && host_segs[0].y == 1 && host_segs[0].z != host_segs[1].z)
    s0 = 1;
  for (int i = s0 + 1; i < co.nseg; ++i)
    if (host_segs[i].z != host_segs[s0].z) return cudaSuccess;
  if (s0) {
    int* flag = nullptr;
    cudaError_t e = cudaMalloc(&flag, sizeof(int));
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(flag, 0, sizeof(int), s);
    const long long nblk = (long long)g.V * g.nb;
    k_cls0_check<<<(unsigned)((nblk + 127) / 128), 128, 0, s>>>(g, co, host_segs[0].z, flag);
    int hflag = 1;
    e = cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(flag);
    if (e != cudaSuccess) return e;
    if (hflag) return cudaSuccess;
  }
  co.s0 = s0;
  co.cm = 1;
  return cudaSuccess;
}

bool chainm_supported(const Geo& g, const ChainOps& co, int sm_count) {
  // one CTA per SM and pair group: worth it when the groups fill most of the machine
  if (!co.cm) return false;
  (void)g;
  (void)sm_count;
  return env_or("GQ_CHAINM", 0) == 1;   // opt-in while it is slower than the per-warp kernel
}

// development dispatch over (record ring depth, consumer warps, tile ring depth)
#define CM_CASE(INNER_, P_, W_, D_, FR_, DOT_)                                                 \
  if (P == P_ && W == W_ && D == D_)                                                           \
    return chains_launch<INNER_, FR_, DOT_, P_, W_, D_>(g, co, io, sm_count, partials, st,     \
                                                        dotmode, s);

template <bool FR, bool DOT>
static cudaError_t chains_outer(const Geo& g, const ChainOps& co, const SweepIo& io, int sm_count,
                                double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  const int P = env_or("GQ_CM_PO", 4), W = env_or("GQ_CM_WO", 13), D = env_or("GQ_CM_DO", 16);
  CM_CASE(false, 4, 13, 16, FR, DOT)
  CM_CASE(false, 6, 13, 16, FR, DOT)
  CM_CASE(false, 4, 13, 32, FR, DOT)
  CM_CASE(false, 3, 13, 8, FR, DOT)
  CM_CASE(false, 4, 9, 16, FR, DOT)
  return cudaErrorInvalidValue;
}

template <bool DOT>
static cudaError_t chains_inner(const Geo& g, const ChainOps& co, const SweepIo& io, int sm_count,
                                double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  const int P = env_or("GQ_CM_PI", 3), W = env_or("GQ_CM_WI", 13), D = env_or("GQ_CM_DI", 16);
  CM_CASE(true, 3, 13, 16, false, DOT)
  CM_CASE(true, 4, 13, 16, false, DOT)
  CM_CASE(true, 2, 13, 16, false, DOT)
  CM_CASE(true, 3, 13, 32, false, DOT)
  CM_CASE(true, 3, 13, 8, false, DOT)
  CM_CASE(true, 3, 9, 16, false, DOT)
  return cudaErrorInvalidValue;
}

cudaError_t launch_chainm(const Geo& g, const ChainOps& co, bool inner, const double* rhs,
                          const double* th, double* out, const double* rdot, int sm_count,
                          double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  const bool dot = dotmode != kDotNone;
  const SweepIo io{rhs, th, out, rdot, nullptr, nullptr, 0.0};
  if (inner)
    return dot ? chains_inner<true>(g, co, io, sm_count, partials, st, dotmode, s)
               : chains_inner<false>(g, co, io, sm_count, partials, st, dotmode, s);
  return dot ? chains_outer<false, true>(g, co, io, sm_count, partials, st, dotmode, s)
             : chains_outer<false, false>(g, co, io, sm_count, partials, st, dotmode, s);
}

cudaError_t launch_chainm_fr(const Geo& g, const ChainOps& co, double* r, const double* y,
                             double* out, int sm_count, double* partials, PcgState* st,
                             cudaStream_t s) {
  const SweepIo io{r, nullptr, out, nullptr, y, r, 0.0};
  return chains_outer<true, false>(g, co, io, sm_count, partials, st, kDotNone, s);
}

}  // namespace gq
