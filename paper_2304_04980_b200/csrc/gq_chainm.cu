// Pair-chain sweeps on the fp64 tensor cores for n = 2 grids that fill the machine.
//
// Same recurrences and the same arithmetic as gq_chain.cu (block_linalg.py:336-358,
// nested_jacobi.py:85-103):
//
//   forward   w_k = L_k^-1 tau_k  - (L_k^-1 Omega~_k) theta  - G_k w_{k-1}
//   backward  x_k = L_k^-T w_k    - H_k x_{k+1}
//
// with 8 consecutive stages of one column pair on the M dimension of m8n8k4 DMMAs, records
// and factor tiles staged per warp by cp.async P blocks ahead.  What differs from the per-warp
// kernel of gq_chain.cu:
//
//   * The theta records of the two middle columns at rows 2k+1, 2k+2 are the rows -1, 0 of the
//     next block: their A fragments are carried in registers, so an inner sweep fetches eight
//     theta records per block instead of twelve (record order in gq_chain.cuh).  The ring slot
//     shrinks from 5.0 to 4.4 KB, and with P = 3 twelve warps fit on an SM instead of eight:
//     the 3328 items of the headline run in two full rounds of 1776 warps instead of three
//     rounds of 1184 (inner sweep 0.257 -> 0.236 ms).
//   * A CTA is W = 12 independent warps (one CTA per SM, no barrier inside the sweep); the last
//     round spreads its items evenly over the CTAs.
//   * w is parked and x written with L1 no-allocate stores.
//
// Measured and dropped on the way (round 2, all parity-green): B fragments read straight from
// global memory through L1 with the warps of an SM on one pair (L2 traffic -40%, but L1TEX
// returns the hits behind the outstanding record copies: 0.31 ms; with a register ring P
// blocks deep the loads share too few scoreboards: 0.44 ms), L1-allocating factor copies
// (cp.async.ca: same time as the per-warp kernel, the L1 data pipe carries every tile three
// times), and a CTA-shared factor-tile ring fed by bulk copies on full/empty mbarriers
// (0.32 ms: 137 instructions per block and warp).
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
// factor tiles: plain 16-byte global -> shared copy (L1 bypassed)
__device__ __forceinline__ void ldgsts_f(unsigned dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
// ... of `sz` (16 or 0) bytes: size 0 zero-fills the destination without touching memory
__device__ __forceinline__ void ldgsts_fz(unsigned dst, const double* src, unsigned sz) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz)
               : "memory");
}
// vector data read once (prologue fragments): bypass L1
__device__ __forceinline__ double2 ldcg2(const double* p) {
  return __ldcg(reinterpret_cast<const double2*>(p));
}

template <int NS, bool INNER, bool FR, bool DOT>
struct Cm {
  static constexpr int Q = 4 * NS, QQ = Q * Q, NT = Q / 8;
  static constexpr int TC = 12 * NS;                  // theta feature count of the M tile
  static constexpr int KT = TC / 8;                   // its k-pairs ...
  static constexpr int KC = KT / 3;                   // ... of which the first KC are carried
  static constexpr int FFS = 2 * QQ + Q * TC;         // forward factor doubles per block
  static constexpr int FB = 2 * QQ;                   // backward factor doubles per block
  static constexpr int REC = 8 * NS;                  // record: 8 stages x NS
  // records are whole 128-byte rows of the ring (a padded stride would split every 128-byte
  // cp.async row write in two); the 16-byte stage chunks of record r sit at chunk ^ 2 (r & 3),
  // which keeps the A-fragment reads of a quarter warp (4 records x 2 stages) conflict-free
  static constexpr int RSTR = REC;
  static constexpr int CPR = REC / 2;                 // 16-byte chunks per record
  static constexpr int RPI = 32 / CPR;                // records per warp copy instruction
  // forward records: tau (4), then theta records 4..11 (inner) or y (4, fused r update)
  static constexpr int NRF = INNER ? 12 : (FR ? 8 : 4);
  static constexpr int NRB = DOT ? 8 : 4;             // backward: w (4) [+ r (4) for q.r]
  static constexpr int JF = NRF / RPI, JB = NRB / RPI;
  static constexpr int FF = INNER ? FFS : 2 * QQ;     // forward factor doubles staged
  static constexpr int CFF = FF / 64, CFB = FB / 64;  // factor copy instructions (32 x 16 B)
  static constexpr int SLOT = (NRF * RSTR + FF) > (NRB * RSTR + FB) ? (NRF * RSTR + FF)
                                                                     : (NRB * RSTR + FB);
  static_assert(NS == 2, "record swizzle: one 16-byte chunk per stage");
};

template <int NS, bool INNER, int P, bool FR, bool DOT>
__device__ __forceinline__ void chainm_item(const Geo& g, const ChainOps& co,
                                            const double* __restrict__ rhs,
                                            const double* __restrict__ th, double* out,
                                            const double* __restrict__ rdot, double* ring, int v,
                                            int t0, int nvalid, int cls, bool diag,
                                            uint64_t pol_k, double& dot, const double* __restrict__ yv,
                                            double* rupd, double alpha, double& rmax) {
  using C = Cm<NS, INNER, FR, DOT>;
  constexpr int QQ = C::QQ, NT = C::NT, KT = C::KT, KC = C::KC, REC = C::RSTR, R = P + 1;
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
  // A-fragment offset of feature pair f0 = 8p + 2qd of chain rw inside a slot
  auto aofs = [&](int f0) {
    return (f0 / NS) * REC + ((rw ^ (2 * ((f0 / NS) & 3))) * NS) + (f0 % NS);
  };

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
    fsrc[j] = (r < 4 ? rhs : (FR ? yv : th)) + col_a + (long long)(colok ? dc : 0) * cs +
              (long long)dr * rs + wofs;
  }
  // per-lane shared destination, kept in a vector register (no [R + UR] LDGSTS forms)
  const unsigned rec_dst = lane_opaque(
      ring_u + (unsigned)(((lane / C::CPR) * REC + 2 * (wch ^ (2 * ((lane / C::CPR) & 3)))) * 8));
  const unsigned facf_dst = lane_opaque(ring_u + (unsigned)(C::NRF * REC * 8 + 16 * lane));
  const unsigned facb_dst = lane_opaque(ring_u + (unsigned)(C::NRB * REC * 8 + 16 * lane));
  const double* ffb = co.ff + ((long long)cls * g.V + v) * nb * C::FFS + 2 * lane;
  // a class whose coupling tiles (G, L^-1 Omega~, H) are all zero -- stage 0, where Psi_0 =
  // Q_0^-1 is block diagonal -- stages only L^-1 and L^-T; the other tiles are zero-filled
  const unsigned offsz = diag ? 0u : 16u;

  // last block (and the prologue): rows outside [0, K) zero-fill
  auto issue_f_chk = [&](int k, int slot) {
    const unsigned sb = lane_opaque((unsigned)(slot * C::SLOT * 8));
#pragma unroll
    for (int j = 0; j < C::JF; ++j) {
      const bool ok = fsz[j] && 2 * k + frow[j] < K;
      ldgsts(rec_dst + sb + j * C::RPI * REC * 8, ok ? fsrc[j] + k * rs2 : rhs, ok ? 16 : 0, 0);
    }
    const double* fp = ffb + (long long)k * C::FFS;
    ldgsts_f(facf_dst + sb, fp);
#pragma unroll
    for (int i = 1; i < C::CFF; ++i) ldgsts_fz(facf_dst + sb + 512 * i, fp + 64 * i, offsz);
  };

  double2 wd[NT];
#pragma unroll
  for (int h = 0; h < NT; ++h) wd[h] = make_double2(0.0, 0.0);

  // output fragment addressing: lane holds features 8h + 2qd, +1 of chain (stage) rw
  long long oofs[NT];
  bool ook[NT];
  int orow[NT];
#pragma unroll
  for (int h = 0; h < NT; ++h) {
    const int f0 = 8 * h + 2 * qd, nd = f0 / NS, cc = f0 % NS;
    orow[h] = nd >> 1;
    oofs[h] = col_a + (long long)(nd & 1) * cs + (long long)(nd >> 1) * rs + rw * NS + cc;
    ook[h] = rw < nvalid && ((nd & 1) ? okb : true);
  }

  // carried theta fragments of block 0: rows -1 (zero) and 0 of the two middle columns
  double2 carry[KC > 0 ? KC : 1];
  if constexpr (INNER) {
#pragma unroll
    for (int p = 0; p < KC; ++p) {
      const int f0 = 8 * p + 2 * qd, rec = f0 / NS, cc = f0 % NS;
      const int dc = th_dc(rec), dr = th_dr(rec);
      const bool ok = dr == 0 && a + dc >= 0 && a + dc < g.N && rw < nvalid;
      carry[p] = ok ? ldcg2(th + col_a + (long long)dc * cs + rw * NS + cc)
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
  const double* fpc = ffb + (long long)P * C::FFS;

  int slot = 0, islot = P % R;
#pragma unroll 1
  for (int k = 0; k < nb; ++k) {
    const int kk = k + P;
    if (kk < nb) {
      if (kk == nb - 1) {
        issue_f_chk(kk, islot);
      } else {
        const unsigned sb = lane_opaque((unsigned)(islot * C::SLOT * 8));
#pragma unroll
        for (int j = 0; j < C::JF; ++j)
          ldgsts(rec_dst + sb + j * C::RPI * REC * 8, fcur[j], fsz[j], 0);
        ldgsts_f(facf_dst + sb, fpc);
#pragma unroll
        for (int i = 1; i < C::CFF; ++i) ldgsts_fz(facf_dst + sb + 512 * i, fpc + 64 * i, offsz);
      }
    }
    commit();
#pragma unroll
    for (int j = 0; j < C::JF; ++j)
      if (fsz[j]) fcur[j] += rs2;
    fpc += C::FFS;
    wait_groups<P>();
    __syncwarp();

    const double* sl = ring + slot * C::SLOT;
    const double* sf = sl + C::NRF * REC + rw * 8 + 2 * qd;
    // loop-carried products first: -G w_{k-1}
    double2 g0[NT], g1[NT];
#pragma unroll
    for (int h = 0; h < NT; ++h) {
      g0[h] = g1[h] = make_double2(0.0, 0.0);
#pragma unroll
      for (int p = 0; p < NT; ++p) {
        const double2 b = lds2(sf + QQ + (h * NT + p) * 64);
        dmma(g0[h], wd[p].x, b.x);
        dmma(g1[h], wd[p].y, b.y);
      }
    }
    double2 tv[NT];
#pragma unroll
    for (int p = 0; p < NT; ++p) tv[p] = lds2(sl + aofs(8 * p + 2 * qd));
    if constexpr (FR) {
      // r -= alpha y (pcg.py:111) on the staged records; the updated residual is this sweep's
      // right-hand side, is written back, and feeds max|r| (pcg.py:113)
      const bool lastk_ = k == nb - 1;
#pragma unroll
      for (int p = 0; p < NT; ++p) {
        const double2 yy = lds2(sl + 4 * REC + aofs(8 * p + 2 * qd));
        tv[p].x = __dsub_rn(tv[p].x, __dmul_rn(alpha, yy.x));
        tv[p].y = __dsub_rn(tv[p].y, __dmul_rn(alpha, yy.y));
        if (ook[p] && !(lastk_ && 2 * k + orow[p] >= K)) {
          stg2_out(rupd + oofs[p] + (long long)k * rs2, tv[p]);
          rmax = nmax(rmax, nmax(fabs(tv[p].x), fabs(tv[p].y)));
        }
      }
    }
    double2 tq[INNER ? KT : 1];
    if constexpr (INNER) {
#pragma unroll
      for (int p = 0; p < KC; ++p) tq[p] = carry[p];
#pragma unroll
      for (int p = KC; p < KT; ++p) tq[p] = lds2(sl + aofs(8 * p + 2 * qd));
#pragma unroll
      for (int p = 0; p < KC; ++p) carry[p] = tq[KC + p];
    }
#pragma unroll
    for (int h = 0; h < NT; ++h) {
      double2 a0 = make_double2(0.0, 0.0), a1 = a0, m0 = a0, m1 = a0, m2 = a0, m3 = a0;
#pragma unroll
      for (int p = 0; p < NT; ++p) {
        const double2 b = lds2(sf + (h * NT + p) * 64);
        dmma(a0, tv[p].x, b.x);
        dmma(a1, tv[p].y, b.y);
      }
      if constexpr (INNER) {
#pragma unroll
        for (int p = 0; p < KT; ++p) {
          const double2 b = lds2(sf + 2 * QQ + (h * KT + p) * 64);
          if (p & 1) {
            dmma(m2, tq[p].x, b.x);
            dmma(m3, tq[p].y, b.y);
          } else {
            dmma(m0, tq[p].x, b.x);
            dmma(m1, tq[p].y, b.y);
          }
        }
      }
      double2 sm = add2(a0, a1);
      if constexpr (INNER) sm = add2(sm, add2(add2(m0, m1), add2(m2, m3)));
      wd[h] = add2(sm, add2(g0[h], g1[h]));
    }
    const bool lastk = k == nb - 1;
#pragma unroll
    for (int h = 0; h < NT; ++h)
      if (ook[h] && !(lastk && 2 * k + orow[h] >= K))
        stg2_park(out + oofs[h] + (long long)k * rs2, wd[h], pol_k);
    slot = slot + 1 == R ? 0 : slot + 1;
    islot = islot + 1 == R ? 0 : islot + 1;
    __syncwarp();
  }
  wait_groups<0>();
  // w was stored by other lanes of this warp: order the stores before the copies that read
  // them back.  CTA scope is enough (same SM, L1 bypassed both ways), and a GPU-scope fence
  // would invalidate the L1 lines of the factor tiles for every warp of the SM.
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
    bsrc[j] = (r < 4 ? (const double*)out : rdot) + col_a + (long long)(dc && okb ? 1 : 0) * cs +
              (long long)dr * rs + wofs;
  }
  const double* fbb = co.fb + ((long long)cls * g.V + v) * nb * C::FB + 2 * lane;
  auto issue_b_chk = [&](int k, int slot_) {
    const unsigned sb = lane_opaque((unsigned)(slot_ * C::SLOT * 8));
#pragma unroll
    for (int j = 0; j < C::JB; ++j) {
      const bool ok = bsz[j] && 2 * k + brow[j] < K;
      ldgsts(rec_dst + sb + j * C::RPI * REC * 8, ok ? bsrc[j] + k * rs2 : rhs, ok ? 16 : 0, 0);
    }
    const double* fp = fbb + (long long)k * C::FB;
    ldgsts_f(facb_dst + sb, fp);
#pragma unroll
    for (int i = 1; i < C::CFB; ++i) ldgsts_fz(facb_dst + sb + 512 * i, fp + 64 * i, offsz);
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
  const double* fbc = fbb + (long long)(nb - 1 - P) * C::FB;

  double2 xd[NT];
#pragma unroll
  for (int h = 0; h < NT; ++h) xd[h] = make_double2(0.0, 0.0);
  slot = 0;
  islot = P % R;
#pragma unroll 1
  for (int k = nb - 1; k >= 0; --k) {
    const int kk = k - P;
    if (kk >= 0) {
      const unsigned sb = lane_opaque((unsigned)(islot * C::SLOT * 8));
#pragma unroll
      for (int j = 0; j < C::JB; ++j)
        ldgsts(rec_dst + sb + j * C::RPI * REC * 8, bcur[j], bsz[j], 0);
      ldgsts_f(facb_dst + sb, fbc);
#pragma unroll
      for (int i = 1; i < C::CFB; ++i) ldgsts_fz(facb_dst + sb + 512 * i, fbc + 64 * i, offsz);
    }
    commit();
#pragma unroll
    for (int j = 0; j < C::JB; ++j)
      if (bsz[j]) bcur[j] -= rs2;
    fbc -= C::FB;
    wait_groups<P>();
    __syncwarp();

    const double* sl = ring + slot * C::SLOT;
    const double* sf = sl + C::NRB * REC + rw * 8 + 2 * qd;
    // loop-carried products first: -H x_{k+1}
    double2 g0[NT], g1[NT];
#pragma unroll
    for (int h = 0; h < NT; ++h) {
      g0[h] = g1[h] = make_double2(0.0, 0.0);
#pragma unroll
      for (int p = 0; p < NT; ++p) {
        const double2 b = lds2(sf + QQ + (h * NT + p) * 64);
        dmma(g0[h], xd[p].x, b.x);
        dmma(g1[h], xd[p].y, b.y);
      }
    }
    double2 wv[NT];
#pragma unroll
    for (int p = 0; p < NT; ++p) wv[p] = lds2(sl + aofs(8 * p + 2 * qd));
#pragma unroll
    for (int h = 0; h < NT; ++h) {
      double2 a0 = make_double2(0.0, 0.0), a1 = a0;
#pragma unroll
      for (int p = 0; p < NT; ++p) {
        const double2 b = lds2(sf + (h * NT + p) * 64);
        dmma(a0, wv[p].x, b.x);
        dmma(a1, wv[p].y, b.y);
      }
      xd[h] = add2(add2(a0, a1), add2(g0[h], g1[h]));
    }
    const bool lastk = k == nb - 1;
#pragma unroll
    for (int h = 0; h < NT; ++h)
      if (ook[h] && !(lastk && 2 * k + orow[h] >= K)) {
        stg2_out(out + oofs[h] + (long long)k * rs2, xd[h]);
        if constexpr (DOT) {
          const double2 rv = lds2(sl + 4 * REC + aofs(8 * h + 2 * qd));
          dot = fma(xd[h].x, rv.x, dot);
          dot = fma(xd[h].y, rv.y, dot);
        }
      }
    slot = slot + 1 == R ? 0 : slot + 1;
    islot = islot + 1 == R ? 0 : islot + 1;
    __syncwarp();
  }
  wait_groups<0>();
  __syncwarp();
}

// Deterministic CTA + grid reduction for W-warp CTAs: lane sums/maxes by butterfly, warp
// partials folded in warp order by thread 0, CTA partials folded by the last CTA.
template <bool MAX>
__device__ bool cta_grid_reduce(double v, double* red, double* partials, unsigned int* counter,
                                double& outv) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = MAX ? warp_max(v) : warp_sum(v);
  // the flag lives in the dynamic array: a static __shared__ variable would move the rings
  // off their 128-byte alignment, and every cp.async into them would split in two
  int& is_last = *reinterpret_cast<int*>(red + 24);
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

template <int NS, bool INNER, int P, int W, bool FR, bool DOT>
__global__ void __launch_bounds__(32 * W, 1)
    k_chainm(Geo g, ChainOps co, const double* __restrict__ rhs, const double* __restrict__ th,
             double* out, const double* __restrict__ rdot, int n_items, double* partials,
             PcgState* st, int dotmode, const double* __restrict__ yv, double* rupd) {
  extern __shared__ __align__(128) double ring_all[];
  using C = Cm<NS, INNER, FR, DOT>;
  if (halted(st)) return;
  const int warp = threadIdx.x >> 5;
  double* ring = ring_all + (size_t)warp * (P + 1) * C::SLOT;
  double* red = ring_all + (size_t)W * (P + 1) * C::SLOT;
  const double alpha = FR ? st->alpha : 0.0;
  double rmax = 0.0, dot = 0.0;
  const uint64_t pol_k = pol_last();
  const int nseg = co.nseg;
  // rounds of gridDim.x * W items; the last round spreads what is left evenly over the CTAs
  // (consecutive items, i.e. chunks of one pair, stay on one CTA)
  const int G = gridDim.x;
#pragma unroll 1
  for (int base = 0; base < n_items; base += G * W) {
    const int left = n_items - base;
    const int per = left >= G * W ? W : (left + G - 1) / G;
    const int u = base + blockIdx.x * per + warp;
    if (warp >= per || u >= n_items) continue;
    const int v = u / nseg;
    const int4 sg = co.seg[u - v * nseg];
    chainm_item<NS, INNER, P, FR, DOT>(g, co, rhs, th, out, rdot, ring, v, sg.x, sg.y, sg.z,
                                       sg.w != 0, pol_k, dot, yv, rupd, alpha, rmax);
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

// flags[cls] = 1 if any coupling tile of the class (forward: everything after L^-1, backward:
// everything after L^-T) has a nonzero entry
__global__ void k_tiles_nonzero(long long blocks_per_cls, int npc, const double* __restrict__ ff,
                                const double* __restrict__ fb, int* flags) {
  using C = Cm<2, true, false, false>;
  const long long total = (long long)npc * blocks_per_cls;
  for (long long b = blockIdx.x; b < total; b += gridDim.x) {
    const double* f = ff + b * C::FFS;
    const double* h = fb + b * C::FB;
    bool nz = false;
    for (int e = C::QQ + threadIdx.x; e < C::FFS; e += blockDim.x) nz = nz || f[e] != 0.0;
    for (int e = C::QQ + threadIdx.x; e < C::FB; e += blockDim.x) nz = nz || h[e] != 0.0;
    if (nz) flags[b / blocks_per_cls] = 1;
  }
}
__global__ void k_seg_mark(int4* seg, int nseg, const int* __restrict__ flags) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nseg) seg[i].w = flags[seg[i].z] ? 0 : 1;
}

int env_or(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

template <int NS, bool INNER, int P, int W, bool FR, bool DOT>
cudaError_t chainm_launch(const Geo& g, const ChainOps& co, const double* rhs, const double* th,
                          double* out, const double* rdot, int sm_count, double* partials,
                          PcgState* st, int dotmode, const double* yv, double* rupd,
                          cudaStream_t s) {
  using C = Cm<NS, INNER, FR, DOT>;
  constexpr size_t smem = ((size_t)W * (P + 1) * C::SLOT + 32) * sizeof(double);
  static bool configured[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 63;
  auto kern = k_chainm<NS, INNER, P, W, FR, DOT>;
  if (!configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured[dev] = true;
  }
  const int n_items = g.V * co.nseg;
  const int blocks = std::max(1, std::min((n_items + W - 1) / W, sm_count));
  kern<<<blocks, 32 * W, smem, s>>>(g, co, rhs, th, out, rdot, n_items, partials, st, dotmode,
                                    yv, rupd);
  return cudaGetLastError();
}

}  // namespace

bool chainm_supported(const Geo& g, int sm_count) {
  // twelve-warp CTAs, one per SM: worth it when the items fill the machine; smaller grids
  // stay on the per-warp kernel (GQ_CHAINM=1 forces this one, the variant tests use it)
  if (g.n != 2 || env_or("GQ_NO_CHAINM", 0)) return false;
  return env_or("GQ_CHAINM", 0) >= 1 || (long long)g.V * ((g.T1 + 7) / 8) >= 8LL * sm_count;
}

bool chainm_all() { return env_or("GQ_CHAINM", 0) == 2; }

cudaError_t launch_chainm_mark(const Geo& g, int npc, const ChainOps& co, int4* seg, int nseg,
                               int* flags, cudaStream_t s) {
  if (g.n != 2 || env_or("GQ_NO_ZTILES", 0)) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(flags, 0, (size_t)npc * sizeof(int), s);
  if (e != cudaSuccess) return e;
  const long long per = (long long)g.V * g.nb;
  k_tiles_nonzero<<<(unsigned)std::min<long long>(npc * per, 4096), 128, 0, s>>>(per, npc, co.ff,
                                                                               co.fb, flags);
  k_seg_mark<<<(nseg + 127) / 128, 128, 0, s>>>(seg, nseg, flags);
  return cudaGetLastError();
}

cudaError_t launch_chainm(const Geo& g, const ChainOps& co, bool inner, const double* rhs,
                          const double* th, double* out, const double* rdot, int sm_count,
                          double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  // ring depth: inner P = 3 (4 slots x 4.4 KB x 12 warps = 215 KB), outer P = 6
  const bool dot = dotmode != kDotNone;
  if (inner) {
    if (dot)
      return chainm_launch<2, true, 3, 12, false, true>(g, co, rhs, th, out, rdot, sm_count,
                                                        partials, st, dotmode, nullptr, nullptr, s);
    return chainm_launch<2, true, 3, 12, false, false>(g, co, rhs, th, out, rdot, sm_count,
                                                       partials, st, dotmode, nullptr, nullptr, s);
  }
  if (dot)
    return chainm_launch<2, false, 7, 12, false, true>(g, co, rhs, th, out, rdot, sm_count,
                                                       partials, st, dotmode, nullptr, nullptr, s);
  return chainm_launch<2, false, 7, 12, false, false>(g, co, rhs, th, out, rdot, sm_count,
                                                      partials, st, dotmode, nullptr, nullptr, s);
}

cudaError_t launch_chainm_fr(const Geo& g, const ChainOps& co, double* r, const double* y,
                             double* out, int sm_count, double* partials, PcgState* st,
                             cudaStream_t s) {
  // ring depth 6 (headline: 0.2482 ms; 5: 0.2485, 7: 0.2516, 8: 0.2539)
  return chainm_launch<2, false, 6, 12, true, false>(g, co, r, nullptr, out, nullptr, sm_count,
                                                     partials, st, kDotNone, y, r, s);
}

}  // namespace gq
