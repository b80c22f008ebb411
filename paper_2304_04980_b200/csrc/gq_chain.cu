// Pair-chain sweeps on the fp64 tensor cores, lean edition ("chain" kernels).
//
// One warp owns 8 chains: 8 consecutive stages (one stage class) of one column pair v, and
// walks the nb = ceil(K/2) two-row blocks of the pair forward then backward
// (block_linalg.py:336-358, nested_jacobi.py:85-103):
//
//   forward   w_k = L_k^-1 tau_k  - (L_k^-1 Omega~_k) theta  - G_k w_{k-1}
//   backward  x_k = L_k^-T w_k    - H_k x_{k+1}
//
// with tau_k the block's right-hand side, theta the previous inner iterate (inner sweeps
// only), G_k = L_k^-1 C_k and H_k = L_k^-T C_{k+1}^T.  Every product is an m8n8k4 DMMA with
// the 8 chains on M: the right-hand side, the 12 theta neighbour records and the carried
// iterate are three A operands of ONE accumulation, so the cross-pair coupling that v6 ran
// on the FMA pipe (5 blocks x 4 nodes of Omega~ per lane) becomes 2*12n/8 DMMAs against the
// precomputed M_k = L_k^-1 Omega~_k.  Only the G_k w_{k-1} term is loop-carried.
//
// Data movement: per block a warp stages its records (8 stages x n doubles, contiguous in the
// stage-inner layout) and the block's factor tiles into a ring of P+1 shared-memory slots
// with cp.async P blocks ahead.  Each lane owns fixed 16-byte chunks; its global source is a
// running pointer advanced by one block stride, validity (off-grid column, stage past T) is
// folded into a loop-invariant src-size, and only the first/last block test rows -- the
// steady-state loop carries no bounds logic.  Items never straddle a stage-class boundary
// (the host splits chunks at class changes), so a slot holds one class's factors.
//
// Factor tiles: every Q x Kc matrix is stored as 8x8 tiles (tile (h,p) = rows 8h.., cols
// 8p.., row-major inside), so a B fragment is one conflict-free LDS.128 per lane
// (row rw, columns 2qd, 2qd+1 -> the two k-steps of a k-pair).
#include <algorithm>
#include <cstdlib>

#include "gq_chain.cuh"

namespace gq {

namespace {

using namespace as;

__device__ __forceinline__ void stg2_keep(double* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x),
               "d"(v.y), "l"(pol)
               : "memory");
}

// ---- Warp reduction for one-warp CTAs (deterministic last-block pattern) -------------------
__device__ bool warp_grid_sum(double v, double* partials, unsigned int* counter, double& out) {
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

__device__ bool warp_grid_max(double v, double* partials, unsigned int* counter, double& out) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = nmax(v, __shfl_xor_sync(0xffffffffu, v, o));
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
  for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) acc = nmax(acc, __ldcg(partials + b));
#pragma unroll
  for (int o = 16; o; o >>= 1) acc = nmax(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  out = acc;
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

}  // namespace

template <int NS, bool INNER, int MT = 1, bool FR = false, bool BGX = false>
struct Ch {
  static constexpr int Q = 4 * NS, QQ = Q * Q, NT = Q / 8;
  static constexpr int TC = 12 * NS;                  // theta feature count
  static constexpr int KT = TC / 8;                   // theta k-pairs
  static constexpr int FFS = 2 * QQ + Q * TC;         // forward factor doubles per block
  static constexpr int FF = INNER ? FFS : 2 * QQ;     // ... staged by this variant
  static constexpr int FB = 2 * QQ;                   // backward factor doubles per block
  static constexpr int ST = 8 * MT;                   // chains (stages) per warp
  static constexpr int REC = ST * NS;                 // record: ST stages x NS
  static constexpr int CPR = REC / 2;                 // 16-byte chunks per record
  static constexpr int RPI = 32 / CPR;                // records per warp instruction
  // forward records: tau(4) + theta(12) (inner) or tau(4) + y(4) (outer sweep fused with the
  // PCG residual update r -= alpha y)
  static constexpr int NRF = INNER ? 16 : (FR ? 8 : 4);
  static constexpr int JF = NRF / RPI, JB = 8 / RPI;  // record instructions fwd / bwd (w + r)
  static constexpr int CFF = FF / 64, CFB = FB / 64;  // factor instructions (32 x 16 B each)
  // n = 8: the factor tiles of a block (40 KB inner) are not staged; B fragments are read
  // straight from global memory (L1-cached, shared by the warps of an SM that work on the
  // same pair, see k_chain's item mapping)
  static constexpr bool BG = NS == 8 || BGX;
  static constexpr int FFST = BG ? 0 : FF, FBST = BG ? 0 : FB;   // staged factor doubles
  // record stride in shared memory: padded by 16*NS bytes so the A-fragment reads of a
  // quarter warp (4 records x 2 chains) hit 8 distinct 16-byte bank groups
  static constexpr int RSTR = REC + 2 * NS;
  static constexpr int SLOT = (NRF * RSTR + FFST) > (8 * RSTR + FBST) ? (NRF * RSTR + FFST)
                                                                     : (8 * RSTR + FBST);
  static_assert(NS == 2 || NS == 4 || NS == 8, "chain sweep needs n in {2, 4, 8}");
  static_assert(CPR <= 32 && 32 % CPR == 0, "a record must split evenly over the warp");
  static_assert(FF % 64 == 0 && FB % 64 == 0, "factor blocks must be whole warp copies");
};

using namespace as;

template <int NS, bool INNER, int P, int MT, bool TF = false, bool FR = false, bool BGX = false>
__device__ __forceinline__ void chain_item(const Geo& g, const ChainOps& co,
                                           const double* __restrict__ rhs,
                                           const double* __restrict__ th, double* out,
                                           const double* __restrict__ rdot, bool dotting,
                                           double* ring, int v, int t0, int nvalid, int cls,
                                           uint64_t pol_s, uint64_t pol_k, double& dot,
                                           int kb, int ke, const double* __restrict__ ffbase,
                                           const double* __restrict__ fbbase,
                                           double2* ucap = nullptr, uint64_t* bars = nullptr,
                                           uint32_t* phase = nullptr,
                                           const double* __restrict__ yv = nullptr,
                                           double* rupd = nullptr, double alpha = 0.0,
                                           double* rmax = nullptr) {
  // TF: the factor block of each chain block arrives by one bulk (TMA) copy issued by lane 0
  // and completes on the slot's mbarrier; records stay on per-lane LDGSTS
  using C = Ch<NS, INNER, MT, FR, BGX>;
  constexpr int QQ = C::QQ, NT = C::NT, KT = C::KT, REC = C::RSTR, R = P + 1;
  // B fragment: staged tile in shared memory, or (n = 8) the tile in global memory
  auto ldb = [](const double* p) -> double2 {
    if constexpr (C::BG)
      return __ldg(reinterpret_cast<const double2*>(p));
    else
      return lds2(p);
  };
  const int lane = threadIdx.x & 31, rw = lane >> 2, qd = lane & 3;
  const long long rs = (long long)g.TS * NS;
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
  // A-fragment offset of feature pair f0 = 8p + 2qd for chain (8m + rw) inside a record slot
  auto aofs = [&](int rec, int m, int f0) { return (rec + f0 / NS) * REC + (8 * m + rw) * NS + (f0 % NS); };

  // ---------------- forward ----------------
  const double* fsrc[C::JF];
  int fsz[C::JF], frow[C::JF];
#pragma unroll
  for (int j = 0; j < C::JF; ++j) {
    const int r = j * C::RPI + lane / C::CPR;
    const bool own = r < 4 || FR;                    // tau or y: the pair's own four nodes
    const int dc = own ? (r & 1) : th_dc(r - 4);
    const int dr = own ? ((r & 3) >> 1) : th_dr(r - 4);
    const bool colok = a + dc >= 0 && a + dc < g.N;
    fsz[j] = (colok && stage_ok) ? 16 : 0;
    frow[j] = dr;
    // off-grid columns are redirected to the pair's own column (never read: size 0)
    fsrc[j] = (r < 4 ? rhs : (FR ? yv : th)) + col_a + (long long)(colok ? dc : 0) * cs +
              (long long)dr * rs + wofs;
  }
  // per-lane shared destinations, kept in vector registers (no [R + UR] LDGSTS forms)
  const unsigned rec_dst = lane_opaque(ring_u + (unsigned)(((lane / C::CPR) * REC + 2 * wch) * 8));
  const unsigned facf_dst = lane_opaque(ring_u + (unsigned)(C::NRF * REC * 8 + 16 * lane));
  const unsigned facb_dst = lane_opaque(ring_u + (unsigned)(8 * REC * 8 + 16 * lane));
  const double* ffb = ffbase + ((long long)cls * g.V + v) * nb * C::FFS + 2 * lane;
  const double* ffb0 = ffbase + ((long long)cls * g.V + v) * nb * C::FFS;
  auto bulk_f = [&](int k, int slot_) {
    if (lane == 0) {
      mbar_expect_tx(bars + slot_, C::FF * 8);
      bulk_g2s(ring + slot_ * C::SLOT + C::NRF * REC, ffb0 + (long long)k * C::FFS, C::FF * 8,
               bars + slot_);
    }
  };
  auto fwait = [&](int slot_) {
    if constexpr (TF) {
      mbar_wait(bars + slot_, (*phase >> slot_) & 1u);
      *phase ^= 1u << slot_;
    }
  };

  // checked issue (first/last blocks and the prologue): rows outside [0, K) zero-fill
  auto issue_f_chk = [&](int k, int slot) {
    const unsigned sb = lane_opaque((unsigned)(slot * C::SLOT * 8));
#pragma unroll
    for (int j = 0; j < C::JF; ++j) {
      const int row = 2 * k + frow[j];
      const bool ok = fsz[j] && row >= 0 && row < K;
      ldgsts(rec_dst + sb + j * C::RPI * REC * 8, ok ? fsrc[j] + k * rs2 : rhs, ok ? 16 : 0,
             pol_s);
    }
    if constexpr (TF) {
      bulk_f(k, slot);
    } else {
      if constexpr (!C::BG) {
        const double* fp = ffb + (long long)k * C::FFS;
#pragma unroll
        for (int i = 0; i < C::CFF; ++i)
          ldgsts(facf_dst + sb + 512 * i, fp + 64 * i, 16, pol_k);
      }
    }
  };

  double2 wd[MT][NT];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int h = 0; h < NT; ++h) wd[m][h] = make_double2(0.0, 0.0);

  // output fragment addressing: lane holds features 8h + 2qd, +1 of chain (stage) 8m + rw
  long long oofs[MT][NT];
  bool ook[MT][NT];
  int orow[NT];
#pragma unroll
  for (int h = 0; h < NT; ++h) {
    const int f0 = 8 * h + 2 * qd, nd = f0 / NS, cc = f0 % NS;
    orow[h] = nd >> 1;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      oofs[m][h] = col_a + (long long)(nd & 1) * cs + (long long)(nd >> 1) * rs +
                   (8 * m + rw) * NS + cc;
      ook[m][h] = 8 * m + rw < nvalid && ((nd & 1) ? okb : true);
    }
  }

  {
    const int pro = P < ke - kb ? P : ke - kb;
#pragma unroll 1
    for (int p = 0; p < pro; ++p) {
      issue_f_chk(kb + p, p);
      commit();
    }
#pragma unroll 1
    for (int p = pro; p < P; ++p) commit();
  }
  // running sources of block k + P
  const double* fcur[C::JF];
#pragma unroll
  for (int j = 0; j < C::JF; ++j) fcur[j] = fsz[j] ? fsrc[j] + (long long)(kb + P) * rs2 : rhs;
  const double* fpc = ffb + (long long)(kb + P) * C::FFS;

  int slot = 0, islot = P % R;
#pragma unroll 1
  for (int k = kb; k < ke; ++k) {
    const int kk = k + P;
    if (kk < ke) {
      if (kk == nb - 1) {
        issue_f_chk(kk, islot);
      } else {
        const unsigned sb = lane_opaque((unsigned)(islot * C::SLOT * 8));
#pragma unroll
        for (int j = 0; j < C::JF; ++j)
          ldgsts(rec_dst + sb + j * C::RPI * REC * 8, fcur[j], fsz[j], pol_s);
        if constexpr (TF) {
          bulk_f(kk, islot);
        } else if constexpr (!C::BG) {
#pragma unroll
          for (int i = 0; i < C::CFF; ++i)
            ldgsts(facf_dst + sb + 512 * i, fpc + 64 * i, 16, pol_k);
        }
      }
    }
    commit();
#pragma unroll
    for (int j = 0; j < C::JF; ++j)
      if (fsz[j]) fcur[j] += rs2;
    fpc += C::FFS;
    wait_groups<P>();
    fwait(slot);
    __syncwarp();

    const double* sl = ring + slot * C::SLOT;
    const double* sf = C::BG ? ffb0 + (long long)k * C::FFS : sl + C::NRF * REC;
    // A operands: tau k-pairs and theta k-pairs of every M-tile
    double2 tv[MT][NT];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int p = 0; p < NT; ++p) tv[m][p] = lds2(sl + aofs(0, m, 8 * p + 2 * qd));
    if constexpr (FR) {
      // r -= alpha y (pcg.py:111) on the staged records; the updated residual is this sweep's
      // right-hand side, is written back, and feeds max|r| (pcg.py:113)
      const bool lastk_ = k == nb - 1;
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int p = 0; p < NT; ++p) {
          const double2 yy = lds2(sl + aofs(4, m, 8 * p + 2 * qd));
          tv[m][p].x = __dsub_rn(tv[m][p].x, __dmul_rn(alpha, yy.x));
          tv[m][p].y = __dsub_rn(tv[m][p].y, __dmul_rn(alpha, yy.y));
          if (ook[m][p] && !(lastk_ && 2 * k + orow[p] >= K)) {
            *reinterpret_cast<double2*>(rupd + oofs[m][p] + (long long)k * rs2) = tv[m][p];
            *rmax = nmax(*rmax, nmax(fabs(tv[m][p].x), fabs(tv[m][p].y)));
          }
        }
    }
    // n = 8 inner sweeps: z = tau - Psi_cross theta first (20 raw 8x8 cross-pair blocks,
    // 40 DMMAs), then w = L^-1 z - G w_prev -- instead of the precomputed L^-1 Omega~ tiles
    // (96 DMMAs); B traffic per block 26 KB instead of 40 KB
    constexpr bool ZF = NS == 8 && INNER;
    if constexpr (ZF) {
#pragma unroll
      for (int p = 0; p < NT; ++p) {
        const int dr = p >> 1, dc = p & 1, row = 2 * k + dr, col = a + dc;
        if (col < g.N && row < K) {
          const double* om =
              co.omega + (((long long)cls * g.nk + (long long)col * K + row) * 5) * 64 + rw * 8 + 2 * qd;
          double2 s0 = make_double2(0.0, 0.0), s1 = s0;
#pragma unroll
          for (int u = 0; u < 5; ++u) {
            const double2 tq = lds2(sl + aofs(4 + th_rec(dc, u, dr), 0, 2 * qd));
            const double2 b = __ldg(reinterpret_cast<const double2*>(om + u * 64));
            if (u & 1) {
              dmma(s1, tq.x, b.x);
              dmma(s1, tq.y, b.y);
            } else {
              dmma(s0, tq.x, b.x);
              dmma(s0, tq.y, b.y);
            }
          }
          tv[0][p].x = tv[0][p].x - (s0.x + s1.x);
          tv[0][p].y = tv[0][p].y - (s0.y + s1.y);
        }
      }
    }
    double2 wn[MT][NT];
#pragma unroll
    for (int h = 0; h < NT; ++h) {
      double2 a0[MT], a1[MT], g0[MT], g1[MT], m0[MT], m1[MT], m2[MT], m3[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m)
        a0[m] = a1[m] = g0[m] = g1[m] = m0[m] = m1[m] = m2[m] = m3[m] = make_double2(0.0, 0.0);
#pragma unroll
      for (int p = 0; p < NT; ++p) {
        const double2 b = ldb(sf + (h * NT + p) * 64 + rw * 8 + 2 * qd);
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          dmma(a0[m], tv[m][p].x, b.x);
          dmma(a1[m], tv[m][p].y, b.y);
        }
      }
      if (INNER && !ZF) {
#pragma unroll
        for (int p = 0; p < KT; ++p) {
          const double2 b = ldb(sf + 2 * QQ + (h * KT + p) * 64 + rw * 8 + 2 * qd);
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            const double2 tq = lds2(sl + aofs(4, m, 8 * p + 2 * qd));
            if (p & 1) {
              dmma(m2[m], tq.x, b.x);
              dmma(m3[m], tq.y, b.y);
            } else {
              dmma(m0[m], tq.x, b.x);
              dmma(m1[m], tq.y, b.y);
            }
          }
        }
      }
#pragma unroll
      for (int p = 0; p < NT; ++p) {
        const double2 b = ldb(sf + QQ + (h * NT + p) * 64 + rw * 8 + 2 * qd);
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          dmma(g0[m], wd[m][p].x, b.x);
          dmma(g1[m], wd[m][p].y, b.y);
        }
      }
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        double2 sm = add2(a0[m], a1[m]);
        if (INNER && !ZF) sm = add2(sm, add2(add2(m0[m], m1[m]), add2(m2[m], m3[m])));
        wn[m][h] = add2(sm, add2(g0[m], g1[m]));
      }
    }
    const bool lastk = k == nb - 1;
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        wd[m][h] = wn[m][h];
        if (ook[m][h] && !(lastk && 2 * k + orow[h] >= K))
          stg2_keep(out + oofs[m][h] + (long long)k * rs2, wn[m][h], pol_k);
      }
    slot = slot + 1 == R ? 0 : slot + 1;
    islot = islot + 1 == R ? 0 : islot + 1;
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
    const int r = j * C::RPI + lane / C::CPR;
    const int dc = r & 1, dr = (r >> 1) & 1;
    const bool ok = stage_ok && (dc ? okb : true) && (r < 4 || dotting);
    bsz[j] = ok ? 16 : 0;
    brow[j] = dr;
    bsrc[j] = (r < 4 ? (const double*)out : (dotting ? rdot : rhs)) + col_a +
              (long long)(dc && okb ? 1 : 0) * cs + (long long)dr * rs + wofs;
  }
  const double* fbb = fbbase + ((long long)cls * g.V + v) * nb * C::FB + 2 * lane;
  const double* fbb0 = fbbase + ((long long)cls * g.V + v) * nb * C::FB;
  auto bulk_b = [&](int k, int slot_) {
    if (lane == 0) {
      mbar_expect_tx(bars + slot_, C::FB * 8);
      bulk_g2s(ring + slot_ * C::SLOT + 8 * REC, fbb0 + (long long)k * C::FB, C::FB * 8,
               bars + slot_);
    }
  };
  auto issue_b_chk = [&](int k, int slot_) {
    const unsigned sb = lane_opaque((unsigned)(slot_ * C::SLOT * 8));
#pragma unroll
    for (int j = 0; j < C::JB; ++j) {
      const bool ok = bsz[j] && 2 * k + brow[j] < K;
      ldgsts(rec_dst + sb + j * C::RPI * REC * 8, ok ? bsrc[j] + k * rs2 : rhs, ok ? 16 : 0,
             pol_s);
    }
    if constexpr (TF) {
      bulk_b(k, slot_);
    } else {
      if constexpr (!C::BG) {
        const double* fp = fbb + (long long)k * C::FB;
#pragma unroll
        for (int i = 0; i < C::CFB; ++i)
          ldgsts(facb_dst + sb + 512 * i, fp + 64 * i, 16, pol_k);
      }
    }
  };
  {
    const int pro = P < ke - kb ? P : ke - kb;
#pragma unroll 1
    for (int p = 0; p < pro; ++p) {
      issue_b_chk(ke - 1 - p, p);
      commit();
    }
#pragma unroll 1
    for (int p = pro; p < P; ++p) commit();
  }
  const double* bcur[C::JB];
#pragma unroll
  for (int j = 0; j < C::JB; ++j)
    bcur[j] = bsz[j] ? bsrc[j] + (long long)(ke - 1 - P) * rs2 : rhs;
  const double* fbc = fbb + (long long)(ke - 1 - P) * C::FB;

  double2 xd[MT][NT];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int h = 0; h < NT; ++h) xd[m][h] = make_double2(0.0, 0.0);
  slot = 0;
  islot = P % R;
#pragma unroll 1
  for (int k = ke - 1; k >= kb; --k) {
    const int kk = k - P;
    if (kk >= kb) {
      const unsigned sb = lane_opaque((unsigned)(islot * C::SLOT * 8));
#pragma unroll
      for (int j = 0; j < C::JB; ++j)
        ldgsts(rec_dst + sb + j * C::RPI * REC * 8, bcur[j], bsz[j], pol_s);
      if constexpr (TF) {
        bulk_b(kk, islot);
      } else if constexpr (!C::BG) {
#pragma unroll
        for (int i = 0; i < C::CFB; ++i)
          ldgsts(facb_dst + sb + 512 * i, fbc + 64 * i, 16, pol_k);
      }
    }
    commit();
#pragma unroll
    for (int j = 0; j < C::JB; ++j)
      if (bsz[j]) bcur[j] -= rs2;
    fbc -= C::FB;
    wait_groups<P>();
    fwait(slot);
    __syncwarp();

    const double* sl = ring + slot * C::SLOT;
    const double* sf = C::BG ? fbb0 + (long long)k * C::FB : sl + 8 * REC;
    double2 wv[MT][NT];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int p = 0; p < NT; ++p) wv[m][p] = lds2(sl + aofs(0, m, 8 * p + 2 * qd));
    double2 xn[MT][NT];
#pragma unroll
    for (int h = 0; h < NT; ++h) {
      double2 a0[MT], a1[MT], g0[MT], g1[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) a0[m] = a1[m] = g0[m] = g1[m] = make_double2(0.0, 0.0);
#pragma unroll
      for (int p = 0; p < NT; ++p) {
        const double2 b = ldb(sf + (h * NT + p) * 64 + rw * 8 + 2 * qd);
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          dmma(a0[m], wv[m][p].x, b.x);
          dmma(a1[m], wv[m][p].y, b.y);
        }
      }
#pragma unroll
      for (int p = 0; p < NT; ++p) {
        const double2 b = ldb(sf + QQ + (h * NT + p) * 64 + rw * 8 + 2 * qd);
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          dmma(g0[m], xd[m][p].x, b.x);
          dmma(g1[m], xd[m][p].y, b.y);
        }
      }
#pragma unroll
      for (int m = 0; m < MT; ++m) xn[m][h] = add2(add2(a0[m], a1[m]), add2(g0[m], g1[m]));
    }
    const bool lastk = k == nb - 1;
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        xd[m][h] = xn[m][h];
        if (ucap != nullptr && m == 0 && h == 0) {
          if (k == kb) ucap[0] = xn[0][0];
          if (k == ke - 1) ucap[1] = xn[0][0];
        }
        if (ook[m][h] && !(lastk && 2 * k + orow[h] >= K)) {
          *reinterpret_cast<double2*>(out + oofs[m][h] + (long long)k * rs2) = xn[m][h];
          if (dotting) {
            const double2 rv = lds2(sl + aofs(4, m, 8 * h + 2 * qd));
            dot = fma(xn[m][h].x, rv.x, dot);
            dot = fma(xn[m][h].y, rv.y, dot);
          }
        }
      }
    slot = slot + 1 == R ? 0 : slot + 1;
    islot = islot + 1 == R ? 0 : islot + 1;
    __syncwarp();
  }
  wait_groups<0>();
  __syncwarp();
}

template <int NS, bool INNER, int P, int MT, bool TF, bool FR = false, bool BGX = false>
__global__ void __launch_bounds__(32) k_chain(Geo g, ChainOps co, const double* __restrict__ rhs,
                                              const double* __restrict__ th, double* out,
                                              const double* __restrict__ rdot, int n_items,
                                              double* partials, PcgState* st, int dotmode,
                                              const double* __restrict__ yv = nullptr,
                                              double* rupd = nullptr, int smc = 0) {
  extern __shared__ __align__(128) double ring[];
  if (halted(st)) return;
  const double alpha = FR ? st->alpha : 0.0;
  double rmax = 0.0;
  const uint64_t pol_s = pol_first(), pol_k = pol_last();
  const bool dotting = dotmode != kDotNone;
  const int nseg = MT == 1 ? co.nseg : co.nseg16;
  const int4* seg = MT == 1 ? co.seg : co.seg16;
  double dot = 0.0;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + (P + 1) * Ch<NS, INNER, MT, FR, BGX>::SLOT);
  uint32_t phase = 0;
  if constexpr (TF) {
    if (threadIdx.x == 0)
      for (int i = 0; i <= P; ++i) mbar_init(bars + i, 1);
    fence_proxy_async();
    __syncwarp();
  }
  // n = 8 reads its factor tiles through L1: map the work so that the warps resident on one
  // SM (blocks b = s, s + smc, s + 2 smc, ... when the grid is per_sm x smc) take consecutive
  // stage chunks of the same pair.  A different block-to-SM placement only costs L1 hits.
  const int G = gridDim.x;
  const bool grouped = Ch<NS, INNER, MT, FR, BGX>::BG && smc > 0 && G % smc == 0;
  const int per = grouped ? G / smc : 1;
  // round r covers units [r G, r G + G): a permutation of the blocks in every round, so a
  // partial last round skips exactly the units past n_items
  const int off = grouped ? (blockIdx.x % smc) * per + blockIdx.x / smc : blockIdx.x;
#pragma unroll 1
  for (int base = 0; base < n_items; base += G) {
    const int u = base + off;
    if (u >= n_items) continue;
    const int v = u / nseg;
    const int4 sg = seg[u - v * nseg];
    chain_item<NS, INNER, P, MT, TF, FR, BGX>(g, co, rhs, th, out, rdot, dotting, ring, v, sg.x,
                                         sg.y, sg.z, pol_s, pol_k, dot, 0, g.nb, co.ff, co.fb,
                                         nullptr, bars, &phase, yv, rupd, alpha, &rmax);
  }
  if constexpr (FR) {
    // max |r| over the grid, then the reference's history / convergence step (pcg.py:113-121)
    double res;
    if (warp_grid_max(rmax, partials, &st->counter[1], res) && threadIdx.x == 0) {
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
    if (warp_grid_sum(dot, partials, &st->counter[2], mu) && threadIdx.x == 0) {
      if (dotmode == kDotInit) {
        st->mu = mu;                       // pcg.py:92
      } else {
        st->beta = mu / st->mu;            // pcg.py:127-131
        st->mu = mu;
      }
    }
  }
}

// ---- factor tiles ---------------------------------------------------------------------
// ff[pc][v][k] = L^-1 | -G | -M (M = L^-1 Omega~, Q x 12n), fb[pc][v][k] = L^-T | -H, all as
// 8x8 tiles; one thread per (block, row).
template <int NS>
__global__ void k_build_chain(Geo g, int npc, const double* __restrict__ fac,
                              const double* __restrict__ omega, double* __restrict__ ff,
                              double* __restrict__ fb) {
  using C = Ch<NS, true>;
  constexpr int Q = C::Q, QQ = C::QQ, TC = C::TC, B2 = NS * NS;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)npc * g.V * g.nb * Q) return;
  const int p = (int)(gid % Q);
  const long long idx = gid / Q;                    // (pc, v, k)
  const int k = (int)(idx % g.nb);
  const int v = (int)((idx / g.nb) % g.V);
  const int pc = (int)(idx / ((long long)g.nb * g.V));
  const double* L = fac + idx * 2 * QQ;
  const double* Cm = L + QQ;
  const double* Cn = (k + 1 < g.nb) ? fac + (idx + 1) * 2 * QQ + QQ : nullptr;
  double* F = ff + idx * C::FFS;
  double* B = fb + idx * C::FB;
  for (int c = 0; c < Q; ++c) {
    double s = 0.0;
    for (int m = 0; m <= p; ++m) s = fma(L[p * Q + m], Cm[m * Q + c], s);
    F[tile_at(p, c, Q)] = L[p * Q + c];
    F[QQ + tile_at(p, c, Q)] = -s;
    B[tile_at(p, c, Q)] = L[c * Q + p];
    double h = 0.0;
    if (Cn)
      for (int m = p; m < Q; ++m) h = fma(L[m * Q + p], Cn[c * Q + m], h);
    B[QQ + tile_at(p, c, Q)] = -h;
  }
  // row p of M = L^-1 Omega~: Omega~[f][rec*NS + c] = Psi_u(node f/NS)[f%NS][c]
  const int a = 2 * v;
  double mrow[TC];
  for (int c = 0; c < TC; ++c) mrow[c] = 0.0;
  for (int f = 0; f <= p; ++f) {
    const double l = L[p * Q + f];
    if (l == 0.0) continue;
    const int nd = f / NS, fc = f % NS, dc = nd & 1, dr = nd >> 1;
    const int col = a + dc, row = 2 * k + dr;
    if (col >= g.N || row >= g.K) continue;
    const double* W = omega + ((long long)pc * g.nk + (long long)col * g.K + row) * 5 * B2;
    for (int u = 0; u < 5; ++u) {
      const int rec = th_rec(dc, u, dr);
      for (int c = 0; c < NS; ++c) mrow[rec * NS + c] = fma(l, W[u * B2 + fc * NS + c], mrow[rec * NS + c]);
    }
  }
  for (int c = 0; c < TC; ++c) F[2 * QQ + tile_at(p, c, TC)] = -mrow[c];
}

// omega[pc][node] = the five cross-pair Psi blocks in the order the chain tiles use them
// (same as gq_fast.cu k_build_rows, for sizes without the fast-path operator rows)
template <int NS>
__global__ void k_build_omega(Geo g, int npc, const double* __restrict__ psi,
                              double* __restrict__ omega) {
  constexpr int B2 = NS * NS;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)npc * g.nk) return;
  const int j = (int)((idx % g.nk) / g.K);
  const double* P = psi + idx * 13 * B2;
  const int ev[5] = {7, 9, 3, 11, 8};
  const int od[5] = {7, 10, 4, 12, 8};
  double* W = omega + idx * 5 * B2;
  for (int u = 0; u < 5; ++u) {
    const int o = (j & 1) ? od[u] : ev[u];
    for (int e = 0; e < B2; ++e) W[u * B2 + e] = P[o * B2 + e];
  }
}

cudaError_t launch_build_omega(const Geo& g, int npc, const double* psi, double* omega,
                               cudaStream_t s) {
  const long long n = (long long)npc * g.nk;
  if (g.n != 8) return cudaErrorInvalidValue;
  k_build_omega<8><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(g, npc, psi, omega);
  return cudaGetLastError();
}

// ---- host side -----------------------------------------------------------------------------

static int env_or(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

bool chain_supported(int n) {
  return (n == 2 || n == 4 || n == 8) && env_or("GQ_NO_CHAIN", 0) == 0;
}

size_t chain_ff_doubles(const Geo& g, int npc) {
  const size_t blocks = (size_t)npc * g.V * g.nb;
  return blocks * (g.n == 2 ? Ch<2, true>::FFS : g.n == 4 ? Ch<4, true>::FFS : Ch<8, true>::FFS);
}
size_t chain_fb_doubles(const Geo& g, int npc) {
  const size_t blocks = (size_t)npc * g.V * g.nb;
  return blocks * (g.n == 2 ? Ch<2, true>::FB : g.n == 4 ? Ch<4, true>::FB : Ch<8, true>::FB);
}

cudaError_t launch_build_chain(const Geo& g, int npc, const double* fac, const double* omega,
                               double* ff, double* fb, cudaStream_t s) {
  const long long n = (long long)npc * g.V * g.nb * 4 * g.n;
  const unsigned blocks = (unsigned)((n + 127) / 128);
  if (g.n == 2)
    k_build_chain<2><<<blocks, 128, 0, s>>>(g, npc, fac, omega, ff, fb);
  else if (g.n == 4)
    k_build_chain<4><<<blocks, 128, 0, s>>>(g, npc, fac, omega, ff, fb);
  else if (g.n == 8)
    k_build_chain<8><<<blocks, 128, 0, s>>>(g, npc, fac, omega, ff, fb);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

template <int NS, bool INNER, int P, int MT, bool TF = false, bool BGX = false>
static cudaError_t chain_launch(const Geo& g, const ChainOps& co, const double* rhs,
                                const double* th, double* out, const double* rdot, int sm_count,
                                double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  constexpr size_t smem =
      (size_t)(P + 1) * Ch<NS, INNER, MT, false, BGX>::SLOT * sizeof(double) + (TF ? (P + 1) * 8 : 0);
  const int n_items = g.V * (MT == 1 ? co.nseg : co.nseg16);
  static int cache[64] = {0};
  int per_sm = 1;
  cudaError_t e = kernel_occupancy(k_chain<NS, INNER, P, MT, TF, false, BGX>, 32, smem, cache, per_sm);
  if (e != cudaSuccess) return e;
  const int blocks = std::max(1, std::min(n_items, per_sm * sm_count));
  const int smc = sm_count;   // n = 8 item grouping
  k_chain<NS, INNER, P, MT, TF, false, BGX><<<blocks, 32, smem, s>>>(g, co, rhs, th, out, rdot, n_items,
                                                      partials, st, dotmode, nullptr, nullptr,
                                                      smc);
  return cudaGetLastError();
}

template <int NS, bool INNER>
static cudaError_t chain_p(const Geo& g, const ChainOps& co, const double* rhs, const double* th,
                           double* out, const double* rdot, int sm_count, double* partials,
                           PcgState* st, int dotmode, cudaStream_t s) {
  // ring depth (blocks in flight per warp), measured at n = 2 (round 1): outer P 3 -> 7 took
  // the outer sweep 0.216 -> 0.182 ms, inner P 3 -> 4 took 0.304 -> 0.287 ms; deeper inner
  // rings lose (P 5: 0.331).  n = 4 slots are 2.5x larger: P = 3.
  if constexpr (NS == 2) {
    if (INNER) return chain_launch<NS, INNER, 4, 1>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
    return chain_launch<NS, INNER, 7, 1>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
  }
  return chain_launch<NS, INNER, 3, 1>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
}

cudaError_t launch_chain(const Geo& g, const ChainOps& co, bool inner, const double* rhs,
                         const double* th, double* out, const double* rdot, int sm_count,
                         double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  // large n = 2 grids: the inner sweeps (with or without the fused dot) run on the twelve-warp
  // kernel (0.236 / 0.255 against 0.262 / 0.273 ms at the headline); its plain outer form
  // measured slower than this file's (0.166 against 0.161 ms) and is only reached with
  // GQ_CHAINM=2
  if (chainm_supported(g, sm_count) && (inner || chainm_all()))
    return launch_chainm(g, co, inner, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
  if (g.n == 2)
    return inner ? chain_p<2, true>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s)
                 : chain_p<2, false>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
  if (g.n == 4)
    return inner ? chain_p<4, true>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s)
                 : chain_p<4, false>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
  if (g.n == 8 && co.grp != nullptr && chain8c_enabled())
    return launch_chain8c(g, co, inner, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
  if (g.n == 8) {
    // P = 2 (10 KB inner / 5 KB outer record slots; factor tiles are not staged)
    // measured on config 5 (tools/c5time.py): inner P = 1 (smaller rings leave more of the
    // SM's L1 to the factor tiles: 4.1 -> 3.55 ms), outer P = 2 (2.36 vs 2.6 ms at P = 1)
    if (inner) return chain_launch<8, true, 1, 1>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
    return chain_launch<8, false, 2, 1>(g, co, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
  }
  return cudaErrorInvalidValue;
}

// outer sweep fused with the PCG residual update: r -= alpha y is applied to the staged
// right-hand-side records, written back to r, and its max-norm reduced (pcg.py:111-121)
template <int NS, int P>
static cudaError_t chain_fr_launch(const Geo& g, const ChainOps& co, double* r, const double* y,
                                   double* out, int sm_count, double* partials, PcgState* st,
                                   cudaStream_t s) {
  constexpr size_t smem = (size_t)(P + 1) * Ch<NS, false, 1, true>::SLOT * sizeof(double);
  const int n_items = g.V * co.nseg;
  static int cache[64] = {0};
  int per_sm = 1;
  cudaError_t e = kernel_occupancy(k_chain<NS, false, P, 1, false, true>, 32, smem, cache, per_sm);
  if (e != cudaSuccess) return e;
  const int blocks = std::max(1, std::min(n_items, per_sm * sm_count));
  k_chain<NS, false, P, 1, false, true><<<blocks, 32, smem, s>>>(
      g, co, r, nullptr, out, nullptr, n_items, partials, st, kDotNone, y, r, sm_count);
  return cudaGetLastError();
}

cudaError_t launch_chain_fr(const Geo& g, const ChainOps& co, double* r, const double* y,
                            double* out, int sm_count, double* partials, PcgState* st,
                            cudaStream_t s) {
  if (chainm_supported(g, sm_count))   // 0.256 against 0.277 ms at the headline
    return launch_chainm_fr(g, co, r, y, out, sm_count, partials, st, s);
  if (g.n == 2)
    return chain_fr_launch<2, 7>(g, co, r, y, out, sm_count, partials, st, s);
  if (g.n == 4) return chain_fr_launch<4, 3>(g, co, r, y, out, sm_count, partials, st, s);
  if (g.n == 8) return chain_fr_launch<8, 3>(g, co, r, y, out, sm_count, partials, st, s);
  return cudaErrorInvalidValue;
}

long long chain_fr_max_blocks(const Geo& g, int nseg, int sm_count) {
  return std::min<long long>((long long)g.V * nseg, 64LL * sm_count);
}

long long chain_max_blocks(const Geo& g, int nseg, int sm_count) {
  return std::min<long long>((long long)g.V * nseg, 32LL * sm_count);
}

}  // namespace gq
