// Pipelined hot kernels for problems whose stage classes are warp-compatible
// (at most two Psi classes among the stages a warp covers and a single Xi class -- every
// time-invariant problem, with or without a distinct terminal weight).  Everything else
// runs the generic v1 kernels in gq_stencil.cu / gq_sweep.cu.
//
// Both kernels keep the v1 mapping (lane = stage, warp = 30/32 consecutive stages of one
// node column / pair) but never consume a load in the iteration that issues it: each warp
// owns a ring of P+1 shared-memory slots filled by cp.async (LDGSTS) P rows / blocks
// ahead.  A slot holds the lane-private vector records the row/block needs (zero-filled
// through src-size 0 when the neighbour is off-grid, which also removes every bounds
// test from the arithmetic) and the warp-uniform operator data (Psi/Xi rows or the pair
// factor block) for the warp's stage classes, so all math reads shared memory.
//
// Sweep: a persistent grid processes (pair, 32-stage chunk) items so that only a bounded
// number of chains is in flight; the forward iterate w is parked in `out` with an L2
// evict_last policy and streamed back by the same ring for the backward sweep, so it
// stays in L2 instead of round-tripping HBM (v1 measured +0.35 GB/sweep of spill).
#include <algorithm>
#include <cstdlib>

#include "gq_internal.h"

namespace gq {

// ---- async-copy helpers -----------------------------------------------------------------

__device__ __forceinline__ unsigned su32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cpa16(void* dst, const void* src, bool valid, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(su32(dst)),
               "l"(src), "r"(valid ? 16 : 0), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cpa8(void* dst, const void* src, bool valid, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2, %3;\n" ::"r"(su32(dst)),
               "l"(src), "r"(valid ? 8 : 0), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// lane-private record: the NS doubles of this lane's stage at one node
template <int NS>
__device__ __forceinline__ void cp_rec(double* dst, const double* src, bool valid, uint64_t pol) {
  if constexpr (NS % 2 == 0) {
#pragma unroll
    for (int k = 0; k < NS; k += 2) cpa16(dst + k, src + k, valid, pol);
  } else {
#pragma unroll
    for (int k = 0; k < NS; ++k) cpa8(dst + k, src + k, valid, pol);
  }
}

// warp-cooperative copy of `nd` doubles of uniform data (8- or 16-byte chunks)
template <int NS>
__device__ __forceinline__ void warp_copy(double* dst, const double* src, int nd, bool valid,
                                          int lane, uint64_t pol) {
  if constexpr (NS % 2 == 0) {
    for (int o = 2 * lane; o < nd; o += 64) cpa16(dst + o, src + o, valid, pol);
  } else {
    for (int o = lane; o < nd; o += 32) cpa8(dst + o, src + o, valid, pol);
  }
}

template <int NS>
__device__ __forceinline__ Vec<NS> lds_rec(const double* p) {
  Vec<NS> r;
  if constexpr (NS % 2 == 0) {
#pragma unroll
    for (int k = 0; k < NS; k += 2) {
      const double2 t = *reinterpret_cast<const double2*>(p + k);
      r.v[k] = t.x;
      r.v[k + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < NS; ++k) r.v[k] = p[k];
  }
  return r;
}

// acc += M x with M from shared memory (fma accumulate)
template <int NS>
__device__ __forceinline__ void macs(Vec<NS>& acc, const double* M, const Vec<NS>& x) {
#pragma unroll
  for (int a = 0; a < NS; ++a) {
#pragma unroll
    for (int b = 0; b < NS; b += (NS % 2 == 0 ? 2 : 1)) {
      if constexpr (NS % 2 == 0) {
        const double2 m = *reinterpret_cast<const double2*>(M + a * NS + b);
        acc.v[a] = fma(m.x, x.v[b], acc.v[a]);
        acc.v[a] = fma(m.y, x.v[b + 1], acc.v[a]);
      } else {
        acc.v[a] = fma(M[a * NS + b], x.v[b], acc.v[a]);
      }
    }
  }
}

template <int NS>
__device__ __forceinline__ void st_rec_pol(double* p, const Vec<NS>& x, uint64_t pol) {
  if constexpr (NS % 2 == 0) {
#pragma unroll
    for (int k = 0; k < NS; k += 2)
      asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p + k),
                   "d"(x.v[k]), "d"(x.v[k + 1]), "l"(pol)
                   : "memory");
  } else {
#pragma unroll
    for (int k = 0; k < NS; ++k)
      asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p + k), "d"(x.v[k]),
                   "l"(pol)
                   : "memory");
  }
}

__device__ __forceinline__ int first_lane(unsigned mask) { return mask ? __ffs(mask) - 1 : 0; }
__device__ __forceinline__ int last_lane(unsigned mask) { return mask ? 31 - __clz(mask) : 0; }


constexpr int kStencilP = 5;   // rows in flight per warp
constexpr int kSweepP = 4;     // blocks in flight per warp

template <int N>
struct Even {
  static constexpr int v = (N + 1) / 2 * 2;
};

// ---- setup: fast-path operator layouts ----------------------------------------------------
// oprow[pc][node] = Psi(13) | Xi_0(5) | Xi_0'(5) blocks: one contiguous row per node so a warp
// stages everything the stencil needs with a single run of 16-byte copies.
// omega[pc][node] = the five cross-pair Psi blocks in the order the sweep applies them.
// fac3[pc][v][k] = G_k = L_k^-1 C_k | L_k^-1 | H_k = L_k^-T C_{k+1}^T, so the chain
// recurrences read w_k = L_k^-1 b_k - G_k w_{k-1} and x_k = L_k^-T w_k - H_k x_{k+1}:
// the same solve as block_linalg.py:336-358 with the dependent path halved.
template <int NS>
__global__ void k_build_rows(Geo g, int npc, const double* __restrict__ psi,
                             const double* __restrict__ xi, const double* __restrict__ xit,
                             double* __restrict__ oprow, double* __restrict__ omega) {
  constexpr int B2 = NS * NS;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)npc * g.nk) return;
  const long long node = idx % g.nk;
  const int j = (int)(node / g.K);
  const double* P = psi + idx * 13 * B2;
  double* O = oprow + idx * 23 * B2;
  for (int e = 0; e < 13 * B2; ++e) O[e] = P[e];
  for (int e = 0; e < 5 * B2; ++e) O[13 * B2 + e] = xi[node * 5 * B2 + e];
  for (int e = 0; e < 5 * B2; ++e) O[18 * B2 + e] = xit[node * 5 * B2 + e];
  const int ev[5] = {7, 9, 3, 11, 8};
  const int od[5] = {7, 10, 4, 12, 8};
  double* W = omega + idx * 5 * B2;
  for (int u = 0; u < 5; ++u) {
    const int o = (j & 1) ? od[u] : ev[u];
    for (int e = 0; e < B2; ++e) W[u * B2 + e] = P[o * B2 + e];
  }
}

template <int NS>
__global__ void k_build_fac3(Geo g, int npc, const double* __restrict__ fac,
                             double* __restrict__ fac3) {
  constexpr int Q = 4 * NS, QQ = Q * Q;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)npc * g.V * g.nb) return;
  const int k = (int)(idx % g.nb);
  const double* L = fac + idx * 2 * QQ;
  const double* C = L + QQ;
  const double* Cn = (k + 1 < g.nb) ? fac + (idx + 1) * 2 * QQ + QQ : nullptr;
  double* G = fac3 + idx * 3 * QQ;
  double* Lo = G + QQ;
  double* H = Lo + QQ;
  for (int p = 0; p < Q; ++p)
    for (int c = 0; c < Q; ++c) {
      double s = 0.0;
      for (int m = 0; m <= p; ++m) s = fma(L[p * Q + m], C[m * Q + c], s);
      G[p * Q + c] = s;
      Lo[p * Q + c] = L[p * Q + c];
      double h = 0.0;
      if (Cn)
        for (int m = p; m < Q; ++m) h = fma(L[m * Q + p], Cn[c * Q + m], h);
      H[p * Q + c] = h;
    }
}

// ---- stencil v3 ----------------------------------------------------------------------------
// modes: kDelta (y = Delta x, optional y.x) and kOuterRhs (y = r + Xi~ x)

template <int NS, int MODE>
struct St3 {
  static constexpr int B2 = NS * NS;
  static constexpr int OPR = 23 * B2;
  static constexpr int OPOFF = (MODE == kDelta) ? 0 : 13 * B2;
  static constexpr int OPN = OPR - OPOFF;
  static constexpr int OPNP = Even<OPN>::v;
  static constexpr int NREC = (MODE == kDelta) ? 5 : 6;
  static constexpr int REC = 32 * NS;
  static constexpr int SLOT = NREC * REC + 2 * OPNP;
  static constexpr int R = kStencilP + 1;
};

template <int NS, int MODE>
__global__ void __launch_bounds__(128) k_stencil3(Geo g, FastOps fo, const double* __restrict__ x,
                                                  const double* __restrict__ rin,
                                                  double* __restrict__ y, int nchunk, int nstrip,
                                                  int rows, double* partials, PcgState* st,
                                                  int dotmode) {
  using C = St3<NS, MODE>;
  constexpr int B2 = C::B2, REC = C::REC;
  extern __shared__ __align__(128) double smem[];
  if (st != nullptr) {
    if (dotmode == kDotStep) {
      const bool stop = st->done || st->step >= st->max_steps;
      if (blockIdx.x == 0 && threadIdx.x == 0) st->skip = stop ? 1 : 0;
      if (stop) return;
    } else if (halted(st)) {
      return;
    }
  }
  const int lane = threadIdx.x & 31;
  double* ring = smem + (size_t)(threadIdx.x >> 5) * C::R * C::SLOT;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const bool active = gw < (long long)g.N * nchunk * nstrip;
  int strip = 0, chunk = 0, j = 0;
  if (active) {
    strip = (int)(gw % nstrip);
    const long long rest = gw / nstrip;
    chunk = (int)(rest % nchunk);
    j = (int)(rest / nchunk);
  }
  const int t = chunk * kHaloChunk + lane - 1;
  const bool tv = active && t >= 0 && t < g.T1;
  const bool useful = tv && lane >= 1 && lane <= kHaloChunk &&
                      (MODE != kDelta || slab_owned(g, t));
  const unsigned vmask = __ballot_sync(0xffffffffu, tv);
  const int pc = tv ? fo.psi_cls[t] : 0;
  const int cA = __shfl_sync(0xffffffffu, pc, first_lane(vmask));
  const int cB = __shfl_sync(0xffffffffu, pc, last_lane(vmask));
  // off-range lanes read class A's operator slot (always staged); their zero-filled
  // records keep every product finite and the masks below select them away
  const int psel = (tv && pc != cA) ? 1 : 0;
  const bool ke = tv && t < g.T;    // e_t exists (Xi_t, t < T)
  const bool kf = tv && t >= 1;     // f_t exists (Xi_{t-1})
  const bool ku = t >= 1;           // receives e_{t-1}
  const bool kd = t < g.T;          // receives f_{t+1}
  const uint64_t pol = policy_evict_first();
  const uint64_t pol_op = policy_evict_last();
  double dot = 0.0;

  if (active) {
    const int i0 = strip * rows;
    const int i1 = min(g.K, i0 + rows);
    const long long rs = (long long)g.TS * NS;
    const int dj[5] = {0, -1, 1, -2, 2};
    const double* cx[5];
    bool cok[5];
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      const int jj = j + dj[m];
      cok[m] = tv && jj >= 0 && jj < g.N;
      cx[m] = cok[m] ? x + ((long long)jj * g.K * g.TS + t) * NS : x;
    }
    const double* cr = (MODE == kOuterRhs && tv) ? rin + ((long long)j * g.K * g.TS + t) * NS : rin;
    const double* oA = fo.oprow + ((long long)cA * g.nk + (long long)j * g.K) * C::OPR + C::OPOFF;
    const double* oB = fo.oprow + ((long long)cB * g.nk + (long long)j * g.K) * C::OPR + C::OPOFF;
    const bool two = cB != cA;
    auto issue = [&](int i, double* sl) {
      if (i < i1) {
        const bool r2 = i + 2 < g.K, r1 = i + 1 < g.K;
        cp_rec<NS>(sl + 0 * REC + lane * NS, r2 ? cx[0] + (i + 2) * rs : x, cok[0] && r2, pol);
        cp_rec<NS>(sl + 1 * REC + lane * NS, r1 ? cx[1] + (i + 1) * rs : x, cok[1] && r1, pol);
        cp_rec<NS>(sl + 2 * REC + lane * NS, r1 ? cx[2] + (i + 1) * rs : x, cok[2] && r1, pol);
        cp_rec<NS>(sl + 3 * REC + lane * NS, cx[3] + i * rs, cok[3], pol);
        cp_rec<NS>(sl + 4 * REC + lane * NS, cx[4] + i * rs, cok[4], pol);
        if (MODE == kOuterRhs) cp_rec<NS>(sl + 5 * REC + lane * NS, cr + i * rs, tv, pol);
        double* so = sl + C::NREC * REC;
        warp_copy<NS>(so, oA + (long long)i * C::OPR, C::OPN, true, lane, pol_op);
        if (two) warp_copy<NS>(so + C::OPNP, oB + (long long)i * C::OPR, C::OPN, true, lane, pol_op);
      }
      cp_commit();
    };
    auto LD = [&](int m, int ii) -> Vec<NS> {
      if (cok[m] && ii >= 0 && ii < g.K) return ldv_nc<NS>(cx[m] + ii * rs);
      return vzero<NS>();
    };
    Vec<NS> c0[5], cm[3], cp[3], cm2, cp2;
    c0[0] = LD(0, i0 - 2);
    c0[1] = LD(0, i0 - 1);
    c0[2] = LD(0, i0);
    c0[3] = LD(0, i0 + 1);
    cm[0] = LD(1, i0 - 1);
    cm[1] = LD(1, i0);
    cp[0] = LD(2, i0 - 1);
    cp[1] = LD(2, i0);
    int sc = 0, si = 0;   // consume / issue slots
#pragma unroll 1
    for (int p = 0; p < kStencilP; ++p) {
      issue(i0 + p, ring + si * C::SLOT);
      si = (si + 1 == C::R) ? 0 : si + 1;
    }
#pragma unroll 1
    for (int i = i0; i < i1; ++i) {
      issue(i + kStencilP, ring + si * C::SLOT);
      si = (si + 1 == C::R) ? 0 : si + 1;
      cp_wait<kStencilP>();
      __syncwarp();
      const double* sl = ring + sc * C::SLOT;
      sc = (sc + 1 == C::R) ? 0 : sc + 1;
      c0[4] = lds_rec<NS>(sl + 0 * REC + lane * NS);
      cm[2] = lds_rec<NS>(sl + 1 * REC + lane * NS);
      cp[2] = lds_rec<NS>(sl + 2 * REC + lane * NS);
      cm2 = lds_rec<NS>(sl + 3 * REC + lane * NS);
      cp2 = lds_rec<NS>(sl + 4 * REC + lane * NS);
      const double* P = sl + C::NREC * REC + psel * C::OPNP;
      Vec<NS> acc = vzero<NS>();
      const double* E;
      if (MODE == kDelta) {
        macs<NS>(acc, P + 0 * B2, c0[2]);
        macs<NS>(acc, P + 1 * B2, c0[1]);
        macs<NS>(acc, P + 2 * B2, c0[3]);
        macs<NS>(acc, P + 3 * B2, cm[1]);
        macs<NS>(acc, P + 4 * B2, cp[1]);
        macs<NS>(acc, P + 5 * B2, c0[0]);
        macs<NS>(acc, P + 6 * B2, c0[4]);
        macs<NS>(acc, P + 7 * B2, cm2);
        macs<NS>(acc, P + 8 * B2, cp2);
        macs<NS>(acc, P + 9 * B2, cm[0]);
        macs<NS>(acc, P + 10 * B2, cp[0]);
        macs<NS>(acc, P + 11 * B2, cm[2]);
        macs<NS>(acc, P + 12 * B2, cp[2]);
        E = P + 13 * B2;
      } else {
        E = P;
      }
      Vec<NS> e = vzero<NS>(), f = vzero<NS>();
      macs<NS>(e, E + 0 * B2, c0[2]);
      macs<NS>(e, E + 1 * B2, c0[1]);
      macs<NS>(e, E + 2 * B2, c0[3]);
      macs<NS>(e, E + 3 * B2, cm[1]);
      macs<NS>(e, E + 4 * B2, cp[1]);
      macs<NS>(f, E + 5 * B2, c0[2]);
      macs<NS>(f, E + 6 * B2, c0[1]);
      macs<NS>(f, E + 7 * B2, c0[3]);
      macs<NS>(f, E + 8 * B2, cm[1]);
      macs<NS>(f, E + 9 * B2, cp[1]);
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        e.v[k] = ke ? e.v[k] : 0.0;
        f.v[k] = kf ? f.v[k] : 0.0;
      }
      Vec<NS> eu = shfl_up<NS>(e, 1);
      Vec<NS> fd = shfl_down<NS>(f, 1);
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        eu.v[k] = ku ? eu.v[k] : 0.0;
        fd.v[k] = kd ? fd.v[k] : 0.0;
      }
      if (MODE == kDelta) {
#pragma unroll
        for (int k = 0; k < NS; ++k) acc.v[k] = (acc.v[k] + eu.v[k]) + fd.v[k];
      } else {   // y = r + (-(Xi_{t-1} x_{t-1}) - Xi_t' x_{t+1})
        const Vec<NS> rv = lds_rec<NS>(sl + 5 * REC + lane * NS);
#pragma unroll
        for (int k = 0; k < NS; ++k) acc.v[k] = rv.v[k] + ((0.0 - eu.v[k]) - fd.v[k]);
      }
      if (useful) {
        stv<NS>(y + ((long long)j * g.K * g.TS + t) * NS + i * rs, acc);
        if (dotmode != kDotNone) {
#pragma unroll
          for (int k = 0; k < NS; ++k) dot = fma(acc.v[k], c0[2].v[k], dot);
        }
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 4; ++r) c0[r] = c0[r + 1];
      cm[0] = cm[1];
      cm[1] = cm[2];
      cp[0] = cp[1];
      cp[1] = cp[2];
    }
    cp_wait<0>();
  }
  if (dotmode != kDotNone) {
    double c;
    if (grid_reduce<false>(dot, partials, &st->counter[0], c) && threadIdx.x == 0) {
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

// ---- sweep v3 ------------------------------------------------------------------------------

template <int NS, bool INNER>
struct Sw3 {
  static constexpr int Q = 4 * NS, QQ = Q * Q, B2 = NS * NS, REC = 32 * NS;
  static constexpr int NRF = INNER ? 16 : 4;
  static constexpr int NR = NRF > 8 ? NRF : 8;      // backward: w (4) + r (4)
  static constexpr int FAC = 2 * QQ;                // G|L (forward) or L|H (backward)
  static constexpr int OMG = INNER ? Even<4 * 5 * B2>::v : 0;
  static constexpr int SLOT = NR * REC + 2 * FAC + 2 * OMG;
  static constexpr int R = kSweepP + 1;
};

template <int NS, bool INNER>
__global__ void __launch_bounds__(32) k_sweep3(Geo g, FastOps fo, const double* __restrict__ rhs,
                                               const double* __restrict__ th, double* out,
                                               const double* __restrict__ rdot, int n_items,
                                               int nchunk, double* partials, PcgState* st,
                                               int dotmode) {
  using C = Sw3<NS, INNER>;
  constexpr int Q = C::Q, QQ = C::QQ, B2 = C::B2, REC = C::REC;
  extern __shared__ __align__(128) double smem[];
  if (halted(st)) return;
  const int lane = threadIdx.x & 31;
  double* ring = smem;
  const uint64_t pol = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  const long long rs = (long long)g.TS * NS;            // next row, same column and stage
  const long long cs = (long long)g.K * g.TS * NS;      // next column
  double dot = 0.0;

#pragma unroll 1
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int v = item / nchunk, chunk = item % nchunk;
    const int t = chunk * 32 + lane;
    const bool tv = t < g.T1;
    const unsigned vmask = __ballot_sync(0xffffffffu, tv);
    const int pc = tv ? fo.psi_cls[t] : 0;
    const int cA = __shfl_sync(0xffffffffu, pc, first_lane(vmask));
    const int cB = __shfl_sync(0xffffffffu, pc, last_lane(vmask));
    const int psel = (tv && pc != cA) ? 1 : 0;
    const bool two = cB != cA;
    const int a = 2 * v;
    const bool okb = a + 1 < g.N;
    const long long lane_off = (long long)(tv ? t : 0) * NS;
    const long long col_a = (long long)a * g.K * g.TS * NS + lane_off;   // (a, row 0, t)
    const double* FA = fo.fac3 + ((long long)cA * g.V + v) * g.nb * 3 * QQ;
    const double* FB = fo.fac3 + ((long long)cB * g.V + v) * g.nb * 3 * QQ;
    const double* OA = fo.omega + ((long long)cA * g.nk + (long long)a * g.K) * 5 * B2;
    const double* OB = fo.omega + ((long long)cB * g.nk + (long long)a * g.K) * 5 * B2;

    // ---- forward: w_k = L_k^-1 tau_k - G_k w_{k-1} ----
    auto issue_f = [&](int k, double* sl) {
      if (k < g.nb) {
        const int i0 = 2 * k;
        const bool ok1 = i0 + 1 < g.K;
        const long long r0 = col_a + i0 * rs;
        cp_rec<NS>(sl + 0 * REC + lane * NS, rhs + r0, tv, pol);
        cp_rec<NS>(sl + 1 * REC + lane * NS, okb ? rhs + r0 + cs : rhs, tv && okb, pol);
        cp_rec<NS>(sl + 2 * REC + lane * NS, ok1 ? rhs + r0 + rs : rhs, tv && ok1, pol);
        cp_rec<NS>(sl + 3 * REC + lane * NS, ok1 && okb ? rhs + r0 + rs + cs : rhs,
                   tv && ok1 && okb, pol);
        if (INNER) {
          // theta at (col offset, row offset): a-2:{0,1} a-1:{-1,0,1,2} b+1:{-1,0,1,2} b+2:{0,1}
          const int tc[12] = {-2, -2, -1, -1, -1, -1, 2, 2, 2, 2, 3, 3};
          const int tr[12] = {0, 1, -1, 0, 1, 2, -1, 0, 1, 2, 0, 1};
#pragma unroll
          for (int m = 0; m < 12; ++m) {
            const int jj = a + tc[m], ii = i0 + tr[m];
            const bool ok = tv && jj >= 0 && jj < g.N && ii >= 0 && ii < g.K;
            cp_rec<NS>(sl + (4 + m) * REC + lane * NS, ok ? th + r0 + tc[m] * cs + tr[m] * rs : th,
                       ok, pol);
          }
          double* so = sl + C::NR * REC + 2 * C::FAC;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const bool ok = (s & 1 ? okb : true) && (s >> 1 ? ok1 : true);
            const long long off = ((long long)(s & 1) * g.K + i0 + (s >> 1)) * 5 * B2;
            warp_copy<NS>(so + s * 5 * B2, ok ? OA + off : OA, 5 * B2, ok, lane, pol_keep);
            if (two)
              warp_copy<NS>(so + C::OMG + s * 5 * B2, ok ? OB + off : OB, 5 * B2, ok, lane, pol_keep);
          }
        }
        double* sf = sl + C::NR * REC;
        warp_copy<NS>(sf, FA + (long long)k * 3 * QQ, 2 * QQ, true, lane, pol_keep);
        if (two) warp_copy<NS>(sf + C::FAC, FB + (long long)k * 3 * QQ, 2 * QQ, true, lane, pol_keep);
      }
      cp_commit();
    };
    double wp[Q];
#pragma unroll
    for (int p = 0; p < Q; ++p) wp[p] = 0.0;
    int sc = 0, si = 0;
#pragma unroll 1
    for (int p = 0; p < kSweepP; ++p) {
      issue_f(p, ring + si * C::SLOT);
      si = (si + 1 == C::R) ? 0 : si + 1;
    }
#pragma unroll 1
    for (int k = 0; k < g.nb; ++k) {
      issue_f(k + kSweepP, ring + si * C::SLOT);
      si = (si + 1 == C::R) ? 0 : si + 1;
      cp_wait<kSweepP>();
      __syncwarp();
      const double* sl = ring + sc * C::SLOT;
      sc = (sc + 1 == C::R) ? 0 : sc + 1;
      double bb[Q];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        Vec<NS> rv = lds_rec<NS>(sl + s * REC + lane * NS);
        if (INNER) {
          const double* om = sl + C::NR * REC + 2 * C::FAC + psel * C::OMG + s * 5 * B2;
          auto T = [&](int m) { return lds_rec<NS>(sl + (4 + m) * REC + lane * NS); };
          const int ri = s >> 1;
          Vec<NS> sacc = vzero<NS>();
          if ((s & 1) == 0) {
            macs<NS>(sacc, om + 0 * B2, T(0 + ri));
            macs<NS>(sacc, om + 1 * B2, T(2 + ri));
            macs<NS>(sacc, om + 2 * B2, T(3 + ri));
            macs<NS>(sacc, om + 3 * B2, T(4 + ri));
            macs<NS>(sacc, om + 4 * B2, T(7 + ri));
          } else {
            macs<NS>(sacc, om + 0 * B2, T(3 + ri));
            macs<NS>(sacc, om + 1 * B2, T(6 + ri));
            macs<NS>(sacc, om + 2 * B2, T(7 + ri));
            macs<NS>(sacc, om + 3 * B2, T(8 + ri));
            macs<NS>(sacc, om + 4 * B2, T(10 + ri));
          }
#pragma unroll
          for (int kk = 0; kk < NS; ++kk) rv.v[kk] -= sacc.v[kk];
        }
#pragma unroll
        for (int kk = 0; kk < NS; ++kk) bb[s * NS + kk] = rv.v[kk];
      }
      const double* G = sl + C::NR * REC + psel * C::FAC;
      const double* Lk = G + QQ;
      double w[Q];
#pragma unroll
      for (int p = 0; p < Q; ++p) {
        double s0 = 0.0;
#pragma unroll
        for (int c = 0; c <= p; ++c) s0 = fma(Lk[p * Q + c], bb[c], s0);
        w[p] = s0;
      }
#pragma unroll
      for (int p = 0; p < Q; ++p) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int c = 0; c < Q; c += 2) {
          const double2 m = *reinterpret_cast<const double2*>(G + p * Q + c);
          s0 = fma(m.x, wp[c], s0);
          s1 = fma(m.y, wp[c + 1], s1);
        }
        w[p] -= s0 + s1;
      }
#pragma unroll
      for (int p = 0; p < Q; ++p) wp[p] = w[p];
      if (tv) {
        const long long r0 = col_a + 2 * k * rs;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const bool ok = (s & 1 ? okb : true) && (s >> 1 ? 2 * k + 1 < g.K : true);
          if (ok) {
            Vec<NS> wv;
#pragma unroll
            for (int kk = 0; kk < NS; ++kk) wv.v[kk] = w[s * NS + kk];
            st_rec_pol<NS>(out + r0 + (s & 1) * cs + (s >> 1) * rs, wv, pol_keep);
          }
        }
      }
      __syncwarp();
    }
    cp_wait<0>();
    __threadfence();
    __syncwarp();

    // ---- backward: x_k = L_k^-T w_k - H_k x_{k+1} ----
    auto issue_b = [&](int k, double* sl) {
      if (k >= 0) {
        const bool ok1 = 2 * k + 1 < g.K;
        const long long r0 = col_a + 2 * k * rs;
        cp_rec<NS>(sl + 0 * REC + lane * NS, out + r0, tv, pol);
        cp_rec<NS>(sl + 1 * REC + lane * NS, okb ? out + r0 + cs : out, tv && okb, pol);
        cp_rec<NS>(sl + 2 * REC + lane * NS, ok1 ? out + r0 + rs : out, tv && ok1, pol);
        cp_rec<NS>(sl + 3 * REC + lane * NS, ok1 && okb ? out + r0 + rs + cs : out,
                   tv && ok1 && okb, pol);
        if (dotmode != kDotNone) {
          cp_rec<NS>(sl + 4 * REC + lane * NS, rdot + r0, tv, pol);
          cp_rec<NS>(sl + 5 * REC + lane * NS, okb ? rdot + r0 + cs : rdot, tv && okb, pol);
          cp_rec<NS>(sl + 6 * REC + lane * NS, ok1 ? rdot + r0 + rs : rdot, tv && ok1, pol);
          cp_rec<NS>(sl + 7 * REC + lane * NS, ok1 && okb ? rdot + r0 + rs + cs : rdot,
                     tv && ok1 && okb, pol);
        }
        double* sf = sl + C::NR * REC;
        warp_copy<NS>(sf, FA + (long long)k * 3 * QQ + QQ, 2 * QQ, true, lane, pol_keep);
        if (two)
          warp_copy<NS>(sf + C::FAC, FB + (long long)k * 3 * QQ + QQ, 2 * QQ, true, lane, pol_keep);
      }
      cp_commit();
    };
    double xn[Q];
#pragma unroll
    for (int p = 0; p < Q; ++p) xn[p] = 0.0;
    sc = 0;
    si = 0;
#pragma unroll 1
    for (int p = 0; p < kSweepP; ++p) {
      issue_b(g.nb - 1 - p, ring + si * C::SLOT);
      si = (si + 1 == C::R) ? 0 : si + 1;
    }
#pragma unroll 1
    for (int k = g.nb - 1; k >= 0; --k) {
      issue_b(k - kSweepP, ring + si * C::SLOT);
      si = (si + 1 == C::R) ? 0 : si + 1;
      cp_wait<kSweepP>();
      __syncwarp();
      const double* sl = ring + sc * C::SLOT;
      sc = (sc + 1 == C::R) ? 0 : sc + 1;
      double wv[Q];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const Vec<NS> r = lds_rec<NS>(sl + s * REC + lane * NS);
#pragma unroll
        for (int kk = 0; kk < NS; ++kk) wv[s * NS + kk] = r.v[kk];
      }
      const double* Lk = sl + C::NR * REC + psel * C::FAC;
      const double* H = Lk + QQ;
      double x[Q];
#pragma unroll
      for (int p = 0; p < Q; ++p) x[p] = 0.0;
#pragma unroll
      for (int c = 0; c < Q; ++c) {
#pragma unroll
        for (int p = 0; p <= c; ++p) x[p] = fma(Lk[c * Q + p], wv[c], x[p]);
      }
#pragma unroll
      for (int p = 0; p < Q; ++p) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int c = 0; c < Q; c += 2) {
          const double2 m = *reinterpret_cast<const double2*>(H + p * Q + c);
          s0 = fma(m.x, xn[c], s0);
          s1 = fma(m.y, xn[c + 1], s1);
        }
        x[p] -= s0 + s1;
      }
#pragma unroll
      for (int p = 0; p < Q; ++p) xn[p] = x[p];
      if (tv) {
        const long long r0 = col_a + 2 * k * rs;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const bool ok = (s & 1 ? okb : true) && (s >> 1 ? 2 * k + 1 < g.K : true);
          if (ok) {
            Vec<NS> xv;
#pragma unroll
            for (int kk = 0; kk < NS; ++kk) xv.v[kk] = x[s * NS + kk];
            stv<NS>(out + r0 + (s & 1) * cs + (s >> 1) * rs, xv);
            if (dotmode != kDotNone) {
              const Vec<NS> r = lds_rec<NS>(sl + (4 + s) * REC + lane * NS);
#pragma unroll
              for (int kk = 0; kk < NS; ++kk) dot = fma(xv.v[kk], r.v[kk], dot);
            }
          }
        }
      }
      __syncwarp();
    }
    cp_wait<0>();
    __syncwarp();
  }
  if (dotmode != kDotNone) {
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


// ---- sweep v4: pair-chain recurrence on the fp64 tensor cores (DMMA m8n8k4) -------------
//
// A warp owns 16 chains (16 consecutive stages of one column pair) = two M-tiles of 8.
// With chains on the MMA M dimension and the 4n features of a block on N, the block
// recurrences are GEMMs  W_k^T = B_k^T L_k^-T - W_{k-1}^T G_k^T  (forward) and
// X_k^T = W_k^T L_k^-1 - X_{k+1}^T H_k^T (backward).  Features are split across k-steps
// as {8s + 2l + (s&1)} so the D fragment of one block (lane l holds columns 2(l%4), +1 of
// its chain row) is exactly the A fragment of the next: the recurrence never leaves
// registers.  B fragments (factor matrices) are read with one LDS.128 per lane per
// (N-tile, k-pair).  M-tiles that mix two stage classes (t = 0 of a time-invariant
// problem) run the MMAs once per class with the other class's rows masked.
// Omega~ theta (inner sweeps) stays on the fp64 FMA pipe: each lane applies the cross-pair
// blocks to the two features it owns.

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}


template <int NS>
struct Sw4P {
  static constexpr int v = NS == 2 ? 6 : 3;   // blocks in flight per warp
};

template <int NS, bool INNER, int MT_ = 2>
struct Sw4 {
  static constexpr int MT = MT_;                     // M-tiles (8 chains each) per warp
  static constexpr int Q = 4 * NS, QQ = Q * Q, B2 = NS * NS;
  static constexpr int NT = Q / 8;                   // N-tiles == k-pairs
  static constexpr int CH = 8 * MT;                  // chains per warp
  static constexpr int REC = CH * NS;                // doubles per record (CH stages)
  static constexpr int NRF = INNER ? 16 : 4;         // forward: tau (4) + theta (12)
  static constexpr int NR = NRF > 8 ? NRF : 8;       // backward: w (4) + r (4)
  static constexpr int FAC = 2 * QQ;                 // per class: L|-G or L^T|-H
  static constexpr int OMG = INNER ? 4 * 5 * B2 : 0; // per class: omega rows of 4 nodes
  static constexpr int SLOT = NR * REC + 2 * FAC + 2 * OMG;
  static constexpr int P = NS == 2 ? (INNER ? (MT == 1 ? 4 : 6) : (MT == 1 ? 6 : 10)) : 3;
  static constexpr int R = P + 1;
};

// copy NREC records (16 stages x NS doubles, used by the v4 layout notes, contiguous in the stage-inner layout) into
// consecutive smem records; src[r] == nullptr -> zero fill; stages >= nvalid zero-filled.
template <int NS, int NREC>
__device__ __forceinline__ void cp_records(double* dst, const double* const (&src)[NREC],
                                           int nvalid, int lane, const double* dummy,
                                           uint64_t pol) {
  static_assert(NS == 2 || NS == 4, "records of 16 stages need NS in {2,4}");
  constexpr int CPR = 8 * NS;                     // 16-byte chunks per record
#pragma unroll
  for (int i = 0; i < NREC * CPR / 32; ++i) {
    const int c = lane + 32 * i;
    const double* s;
    int w;
    if (NS == 2) {
      s = (lane >> 4) ? src[2 * i + 1] : src[2 * i];
      w = lane & 15;
    } else {
      s = src[i];
      w = lane;
    }
    const int stage = w / (NS / 2);
    const bool ok = s != nullptr && stage < nvalid;
    cpa16(dst + (c / CPR) * 16 * NS + 2 * w, ok ? s + 2 * w : dummy, ok, pol);
  }
}

// ---- sweep v6: lean DMMA chain solver ------------------------------------------------------
// Same math and fragment layout as described above, restructured for issue efficiency:
//  * every address is computed once per item; per block only row offsets advance and only
//    the first/last block (grid boundary rows) test validity;
//  * the L*tau products and the two G/H k-steps use separate accumulators, so a single
//    DMMA (~86-cycle latency) sits on the loop-carried path;
//  * MT M-tiles (8 chains each) per warp: MT=1 lets two warps share an SMSP (a DMMA blocks
//    its issuing warp ~17 cycles) while keeping the chains in flight, and so the parked
//    forward iterates, inside L2;
//  * tiles holding one stage class skip the class masking (TWO=false instantiation).
template <int NS, bool INNER, int MT, bool TWO>
__device__ __forceinline__ void sweep6_item(
    const Geo& g, const FastOps& fo, const double* __restrict__ rhs,
    const double* __restrict__ th, double* out, const double* __restrict__ rdot, int dotmode,
    double* ring, int lane, int v, int t0, int nvalid, int cA, int cB, const int (&cls)[MT],
    const bool (&tvm)[MT], uint64_t pol, uint64_t pol_keep, double& dot) {
  using C = Sw4<NS, INNER, MT>;
  constexpr int Q = C::Q, QQ = C::QQ, B2 = C::B2, NT = C::NT, REC = C::REC, P = C::P, R = C::R;
  constexpr int SLOT = C::SLOT, CH = C::CH;
  constexpr int CPR = CH * NS / 2;                 // 16-byte chunks per record
  constexpr int RPI = 32 / CPR;                    // records per warp instruction
  const int qd = lane & 3, rw = lane >> 2;
  const long long rs = (long long)g.TS * NS;
  const long long cs = (long long)g.K * g.TS * NS;
  const long long rs2 = 2 * rs;
  const int a = 2 * v;
  const bool okb = a + 1 < g.N;
  const int nb = g.nb;
  const long long col_a = (long long)a * g.K * g.TS * NS + (long long)t0 * NS;
  const double* FA = fo.fac4 + ((long long)cA * g.V + v) * nb * 4 * QQ;
  const double* FB = fo.fac4 + ((long long)cB * g.V + v) * nb * 4 * QQ;
  const double* OA = fo.omega + ((long long)cA * g.nk + (long long)a * g.K) * 5 * B2;
  const double* OB = fo.omega + ((long long)cB * g.nk + (long long)a * g.K) * 5 * B2;
  double* const ring_end = ring + R * SLOT;

  const int my_w = lane % CPR;
  const bool stage_ok = my_w / (NS / 2) < nvalid;
  constexpr int JF = C::NRF / RPI;
  const double* fsrc[JF];
  int fsz[JF], fdst[JF], frow[JF];
#pragma unroll
  for (int j = 0; j < JF; ++j) {
    const int r = j * RPI + lane / CPR;
    int dc, dr;
    if (r < 4) {
      dc = r & 1;
      dr = r >> 1;
    } else {
      const int tc[12] = {-2, -2, -1, -1, -1, -1, 2, 2, 2, 2, 3, 3};
      const int tr[12] = {0, 1, -1, 0, 1, 2, -1, 0, 1, 2, 0, 1};
      dc = tc[r - 4];
      dr = tr[r - 4];
    }
    const int jj = a + dc;
    const bool colok = stage_ok && jj >= 0 && jj < g.N;
    fsz[j] = colok ? 16 : 0;
    frow[j] = dr;
    fsrc[j] = colok ? (r < 4 ? rhs : th) + col_a + (long long)dc * cs + (long long)dr * rs + 2 * my_w
                    : rhs;
    fdst[j] = r * REC + 2 * my_w;
  }
  constexpr int FCH = QQ;                          // 16-byte chunks of one factor pair
  constexpr int OCHN = 5 * B2 / 2;
  constexpr int OCH = 4 * OCHN;
  constexpr int OCU = (OCH + 31) / 32;
  int odst[OCU], osz[OCU], orow[OCU], ooff[OCU];
#pragma unroll
  for (int u = 0; u < OCU; ++u) {
    const int c = lane + 32 * u;
    const int s = c / OCHN, w = c % OCHN;
    const bool ok = INNER && c < OCH && ((s & 1) ? okb : true);
    osz[u] = ok ? 16 : 0;
    orow[u] = s >> 1;
    ooff[u] = ok ? (((s & 1) * g.K + (s >> 1)) * 5 * B2 + 2 * w) : 0;
    odst[u] = C::NR * REC + 2 * C::FAC + (c < OCH ? c : 0) * 2;
  }
  const long long odelta = 2LL * 5 * B2;

  auto issue_f = [&](int k, double* sl) {
    if (k < nb) {
      const long long roff = (long long)k * rs2;
      const bool edge = (k == 0) || (k == nb - 1);
#pragma unroll
      for (int j = 0; j < JF; ++j) {
        int sz = fsz[j];
        if (edge) {
          const int row = 2 * k + frow[j];
          if (row < 0 || row >= g.K) sz = 0;
        }
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(
                         su32(sl + fdst[j])),
                     "l"(sz ? fsrc[j] + roff : rhs), "r"(sz), "l"(pol)
                     : "memory");
      }
      const double* fa = FA + (long long)k * 4 * QQ;
#pragma unroll
      for (int c = lane; c < FCH; c += 32) cpa16(sl + C::NR * REC + 2 * c, fa + 2 * c, true, pol_keep);
      if (TWO) {
        const double* fb = FB + (long long)k * 4 * QQ;
#pragma unroll
        for (int c = lane; c < FCH; c += 32)
          cpa16(sl + C::NR * REC + C::FAC + 2 * c, fb + 2 * c, true, pol_keep);
      }
      if (INNER) {
#pragma unroll
        for (int u = 0; u < OCU; ++u) {
          if (lane + 32 * u < OCH) {
            int sz = osz[u];
            if (edge && 2 * k + orow[u] >= g.K) sz = 0;
            const long long o = sz ? ooff[u] + k * odelta : 0;
            cpa16(sl + odst[u], OA + o, sz != 0, pol_keep);
            if (TWO) cpa16(sl + odst[u] + C::OMG, OB + o, sz != 0, pol_keep);
          }
        }
      }
    }
    cp_commit();
  };

  int nd[NT], co[NT];
#pragma unroll
  for (int h = 0; h < NT; ++h) {
    nd[h] = (8 * h + 2 * qd) / NS;
    co[h] = (8 * h + 2 * qd) % NS;
  }
  double* optr[MT][NT];
  bool ostore[MT][NT], olast[MT][NT];
  int bofs[MT][NT];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int h = 0; h < NT; ++h) {
      optr[m][h] = out + col_a + (nd[h] & 1) * cs + (nd[h] >> 1) * rs + (8 * m + rw) * NS + co[h];
      ostore[m][h] = tvm[m] && ((nd[h] & 1) ? okb : true);
      olast[m][h] = (nd[h] >> 1) && (2 * (nb - 1) + 1 >= g.K);
      bofs[m][h] = nd[h] * REC + (8 * m + rw) * NS + co[h];
    }
  int fofs[NT][NT];
#pragma unroll
  for (int h = 0; h < NT; ++h)
#pragma unroll
    for (int sg = 0; sg < NT; ++sg) fofs[h][sg] = (8 * h + rw) * Q + 8 * sg + 2 * qd;
  int selm[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) selm[m] = (TWO && cls[m] == cB) ? 1 : 0;

  // DMMA halves of a block update (rows masked per class pass when TWO):
  //   lmma: d = X0 L0 + X1 L1 (independent of the recurrence)
  //   gmma: e = Y0 G0 + Y1 G1 (loop-carried through Y)
  auto lmma = [&](const double* sf, const double (&xa)[MT][NT][2], double (&d)[MT][NT][2]) {
    double d1[MT][NT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h)
#pragma unroll
        for (int z = 0; z < 2; ++z) d[m][h][z] = d1[m][h][z] = 0.0;
#pragma unroll
    for (int pass = 0; pass < (TWO ? 2 : 1); ++pass) {
      const double* L = sf + pass * C::FAC;
      const int cx = pass ? cB : cA;
#pragma unroll
      for (int h = 0; h < NT; ++h)
#pragma unroll
        for (int sg = 0; sg < NT; ++sg) {
          const double2 lb = *reinterpret_cast<const double2*>(L + fofs[h][sg]);
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            const bool on = !TWO || cls[m] == cx;
            dmma(d[m][h][0], d[m][h][1], on ? xa[m][sg][0] : 0.0, lb.x);
            dmma(d1[m][h][0], d1[m][h][1], on ? xa[m][sg][1] : 0.0, lb.y);
          }
        }
    }
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h)
#pragma unroll
        for (int z = 0; z < 2; ++z) d[m][h][z] += d1[m][h][z];
  };
  // G fragments of one block (both classes when TWO)
  auto gfrag = [&](const double* sf, double2 (&gb)[TWO ? 2 : 1][NT][NT]) {
#pragma unroll
    for (int pass = 0; pass < (TWO ? 2 : 1); ++pass)
#pragma unroll
      for (int h = 0; h < NT; ++h)
#pragma unroll
        for (int sg = 0; sg < NT; ++sg)
          gb[pass][h][sg] = *reinterpret_cast<const double2*>(sf + pass * C::FAC + QQ + fofs[h][sg]);
  };
  auto gmma = [&](const double2 (&gb)[TWO ? 2 : 1][NT][NT], const double (&ya)[MT][NT][2],
                  double (&e0)[MT][NT][2], double (&e1)[MT][NT][2]) {
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h)
#pragma unroll
        for (int z = 0; z < 2; ++z) e0[m][h][z] = e1[m][h][z] = 0.0;
#pragma unroll
    for (int pass = 0; pass < (TWO ? 2 : 1); ++pass) {
      const int cx = pass ? cB : cA;
#pragma unroll
      for (int h = 0; h < NT; ++h)
#pragma unroll
        for (int sg = 0; sg < NT; ++sg)
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            const bool on = !TWO || cls[m] == cx;
            dmma(e0[m][h][0], e0[m][h][1], on ? ya[m][sg][0] : 0.0, gb[pass][h][sg].x);
            dmma(e1[m][h][0], e1[m][h][1], on ? ya[m][sg][1] : 0.0, gb[pass][h][sg].y);
          }
    }
  };
  // tau pairs of a forward slot (rhs minus Omega~ theta for inner sweeps)
  auto load_tau = [&](const double* sl, double (&bp)[MT][NT][2]) {
    const double* sf = sl + C::NR * REC;
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        const double2 bv = *reinterpret_cast<const double2*>(sl + bofs[m][h]);
        bp[m][h][0] = bv.x;
        bp[m][h][1] = bv.y;
      }
    if (INNER) {
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        const int ri = nd[h] >> 1;
        const bool odd = nd[h] & 1;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          const double* om = sf + 2 * C::FAC + selm[m] * C::OMG + nd[h] * 5 * B2 + co[h] * NS;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int u = 0; u < 5; ++u) {
            const int tix = odd ? (u == 0 ? 3 : u == 1 ? 6 : u == 2 ? 7 : u == 3 ? 8 : 10)
                                : (u == 0 ? 0 : u == 1 ? 2 : u == 2 ? 3 : u == 3 ? 4 : 7);
#pragma unroll
            for (int c = 0; c < NS; c += 2) {
              const double2 m0 = *reinterpret_cast<const double2*>(om + u * B2 + c);
              const double2 m1 = *reinterpret_cast<const double2*>(om + u * B2 + NS + c);
              const double2 tv2 = *reinterpret_cast<const double2*>(
                  sl + (4 + tix + ri) * REC + (8 * m + rw) * NS + c);
              s0 = fma(m0.x, tv2.x, s0);
              s2 = fma(m0.y, tv2.y, s2);
              s1 = fma(m1.x, tv2.x, s1);
              s3 = fma(m1.y, tv2.y, s3);
            }
          }
          bp[m][h][0] -= s0 + s2;
          bp[m][h][1] -= s1 + s3;
        }
      }
    }
  };

  // ---------------- forward: w_k = L_k^-1 tau_k - G_k w_{k-1} ----------------
  // software-pipelined by one block: the loop-carried G_k w_{k-1} DMMAs of block k overlap
  // the fragment loads and L_{k+1} tau_{k+1} DMMAs of block k+1.
  double wd[MT][NT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int h = 0; h < NT; ++h) wd[m][h][0] = wd[m][h][1] = 0.0;
  double* scp = ring;   // slot of the next block to consume
  double* sip = ring;
#pragma unroll 1
  for (int p = 0; p < P; ++p) {
    issue_f(p, sip);
    sip += SLOT;
    if (sip == ring_end) sip = ring;
  }
  double dl[MT][NT][2];
  double2 gcur[TWO ? 2 : 1][NT][NT];
  {
    cp_wait<P - 1>();
    __syncwarp();
    double bp[MT][NT][2];
    load_tau(scp, bp);
    lmma(scp + C::NR * REC, bp, dl);
    gfrag(scp + C::NR * REC, gcur);
    scp += SLOT;
    if (scp == ring_end) scp = ring;
  }
#pragma unroll 1
  for (int k = 0; k < nb; ++k) {
    issue_f(k + P, sip);
    sip += SLOT;
    if (sip == ring_end) sip = ring;
    double e0[MT][NT][2], e1[MT][NT][2];
    gmma(gcur, wd, e0, e1);
    double dln[MT][NT][2];
    double2 gnext[TWO ? 2 : 1][NT][NT];
    if (k + 1 < nb) {
      cp_wait<P - 1>();
      __syncwarp();
      double bp[MT][NT][2];
      load_tau(scp, bp);
      lmma(scp + C::NR * REC, bp, dln);
      gfrag(scp + C::NR * REC, gnext);
      scp += SLOT;
      if (scp == ring_end) scp = ring;
    }
    const bool lastk = k == nb - 1;
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        wd[m][h][0] = dl[m][h][0] + (e0[m][h][0] + e1[m][h][0]);
        wd[m][h][1] = dl[m][h][1] + (e0[m][h][1] + e1[m][h][1]);
        if (ostore[m][h] && !(lastk && olast[m][h])) {
          asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(optr[m][h] + k * rs2),
                         "d"(wd[m][h][0]), "d"(wd[m][h][1]), "l"(pol_keep)
                         : "memory");
        }
      }
    if (k + 1 < nb) {
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int h = 0; h < NT; ++h) {
          dl[m][h][0] = dln[m][h][0];
          dl[m][h][1] = dln[m][h][1];
        }
#pragma unroll
      for (int pass = 0; pass < (TWO ? 2 : 1); ++pass)
#pragma unroll
        for (int h = 0; h < NT; ++h)
#pragma unroll
          for (int sg = 0; sg < NT; ++sg) gcur[pass][h][sg] = gnext[pass][h][sg];
    }
    __syncwarp();
  }
  cp_wait<0>();
  __threadfence();
  __syncwarp();

  // ---------------- backward: x_k = L_k^-T w_k - H_k x_{k+1} ----------------
  constexpr int JB = 8 / RPI;
  const double* bsrc[JB];
  int bsz[JB], bdst[JB], brow[JB];
#pragma unroll
  for (int j = 0; j < JB; ++j) {
    const int r = j * RPI + lane / CPR;
    const int dc = r & 1, dr = (r >> 1) & 1;
    const bool ok = stage_ok && (dc ? okb : true) && (r < 4 || dotmode != kDotNone);
    bsz[j] = ok ? 16 : 0;
    brow[j] = dr;
    bsrc[j] = ok ? (r < 4 ? (const double*)out : rdot) + col_a + (long long)dc * cs +
                       (long long)dr * rs + 2 * my_w
                 : rhs;
    bdst[j] = r * REC + 2 * my_w;
  }
  auto issue_b = [&](int k, double* sl) {
    if (k >= 0) {
      const long long roff = (long long)k * rs2;
      const bool edge = (k == nb - 1);
#pragma unroll
      for (int j = 0; j < JB; ++j) {
        int sz = bsz[j];
        if (edge && 2 * k + brow[j] >= g.K) sz = 0;
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(
                         su32(sl + bdst[j])),
                     "l"(sz ? bsrc[j] + roff : rhs), "r"(sz), "l"(pol)
                     : "memory");
      }
      const double* fa = FA + (long long)k * 4 * QQ + 2 * QQ;
#pragma unroll
      for (int c = lane; c < FCH; c += 32) cpa16(sl + C::NR * REC + 2 * c, fa + 2 * c, true, pol_keep);
      if (TWO) {
        const double* fb = FB + (long long)k * 4 * QQ + 2 * QQ;
#pragma unroll
        for (int c = lane; c < FCH; c += 32)
          cpa16(sl + C::NR * REC + C::FAC + 2 * c, fb + 2 * c, true, pol_keep);
      }
    }
    cp_commit();
  };
  auto load_w = [&](const double* sl, double (&wp)[MT][NT][2], double (&rp)[MT][NT][2]) {
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        const double2 wv = *reinterpret_cast<const double2*>(sl + bofs[m][h]);
        wp[m][h][0] = wv.x;
        wp[m][h][1] = wv.y;
        const double2 rv = *reinterpret_cast<const double2*>(sl + 4 * REC + bofs[m][h]);
        rp[m][h][0] = rv.x;
        rp[m][h][1] = rv.y;
      }
  };
  double xd[MT][NT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int h = 0; h < NT; ++h) xd[m][h][0] = xd[m][h][1] = 0.0;
  scp = ring;
  sip = ring;
#pragma unroll 1
  for (int p = 0; p < P; ++p) {
    issue_b(nb - 1 - p, sip);
    sip += SLOT;
    if (sip == ring_end) sip = ring;
  }
  double rcur[MT][NT][2];
  {
    cp_wait<P - 1>();
    __syncwarp();
    double wp[MT][NT][2];
    load_w(scp, wp, rcur);
    lmma(scp + C::NR * REC, wp, dl);
    gfrag(scp + C::NR * REC, gcur);
    scp += SLOT;
    if (scp == ring_end) scp = ring;
  }
#pragma unroll 1
  for (int k = nb - 1; k >= 0; --k) {
    issue_b(k - P, sip);
    sip += SLOT;
    if (sip == ring_end) sip = ring;
    double e0[MT][NT][2], e1[MT][NT][2];
    gmma(gcur, xd, e0, e1);
    double dln[MT][NT][2], rnext[MT][NT][2];
    double2 gnext[TWO ? 2 : 1][NT][NT];
    if (k > 0) {
      cp_wait<P - 1>();
      __syncwarp();
      double wp[MT][NT][2];
      load_w(scp, wp, rnext);
      lmma(scp + C::NR * REC, wp, dln);
      gfrag(scp + C::NR * REC, gnext);
      scp += SLOT;
      if (scp == ring_end) scp = ring;
    }
    const bool lastk = k == nb - 1;
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        xd[m][h][0] = dl[m][h][0] + (e0[m][h][0] + e1[m][h][0]);
        xd[m][h][1] = dl[m][h][1] + (e0[m][h][1] + e1[m][h][1]);
        if (ostore[m][h] && !(lastk && olast[m][h])) {
          *reinterpret_cast<double2*>(optr[m][h] + k * rs2) = make_double2(xd[m][h][0], xd[m][h][1]);
          if (dotmode != kDotNone) {
            dot = fma(xd[m][h][0], rcur[m][h][0], dot);
            dot = fma(xd[m][h][1], rcur[m][h][1], dot);
          }
        }
      }
    if (k > 0) {
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int h = 0; h < NT; ++h)
#pragma unroll
          for (int z = 0; z < 2; ++z) {
            dl[m][h][z] = dln[m][h][z];
            rcur[m][h][z] = rnext[m][h][z];
          }
#pragma unroll
      for (int pass = 0; pass < (TWO ? 2 : 1); ++pass)
#pragma unroll
        for (int h = 0; h < NT; ++h)
#pragma unroll
          for (int sg = 0; sg < NT; ++sg) gcur[pass][h][sg] = gnext[pass][h][sg];
    }
    __syncwarp();
  }
  cp_wait<0>();
  __syncwarp();
}

template <int NS, bool INNER, int MT>
__global__ void __launch_bounds__(32) k_sweep6(Geo g, FastOps fo, const double* __restrict__ rhs,
                                               const double* __restrict__ th, double* out,
                                               const double* __restrict__ rdot, int n_items,
                                               int nchunk, double* partials, PcgState* st,
                                               int dotmode) {
  extern __shared__ __align__(128) double smem[];
  if (halted(st)) return;
  const int lane = threadIdx.x & 31;
  const int rw = lane >> 2;
  uint64_t pol = policy_evict_first();
  uint64_t pol_keep = policy_evict_last();
  double dot = 0.0;
#pragma unroll 1
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int v = item / nchunk, chunk = item % nchunk;
    const int t0 = chunk * 8 * MT;
    const int nvalid = min(8 * MT, g.T1 - t0);
    int cls[MT];
    bool tvm[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int t = t0 + 8 * m + rw;
      tvm[m] = t < g.T1;
      cls[m] = tvm[m] ? fo.psi_cls[t] : -1;
    }
    const int cA = fo.psi_cls[t0];
    const int cB = fo.psi_cls[t0 + nvalid - 1];
    if (cA == cB)
      sweep6_item<NS, INNER, MT, false>(g, fo, rhs, th, out, rdot, dotmode, smem, lane, v, t0,
                                        nvalid, cA, cB, cls, tvm, pol, pol_keep, dot);
    else
      sweep6_item<NS, INNER, MT, true>(g, fo, rhs, th, out, rdot, dotmode, smem, lane, v, t0,
                                       nvalid, cA, cB, cls, tvm, pol, pol_keep, dot);
  }
  if (dotmode != kDotNone) {
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


template <int NS>
__global__ void k_build_fac4(Geo g, int npc, const double* __restrict__ fac,
                             double* __restrict__ fac4) {
  constexpr int Q = 4 * NS, QQ = Q * Q;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)npc * g.V * g.nb) return;
  const int k = (int)(idx % g.nb);
  const double* L = fac + idx * 2 * QQ;
  const double* Cm = L + QQ;
  const double* Cn = (k + 1 < g.nb) ? fac + (idx + 1) * 2 * QQ + QQ : nullptr;
  double* Lo = fac4 + idx * 4 * QQ;
  double* G = Lo + QQ;
  double* LT = G + QQ;
  double* H = LT + QQ;
  for (int p = 0; p < Q; ++p)
    for (int c = 0; c < Q; ++c) {
      double s = 0.0;
      for (int m = 0; m <= p; ++m) s = fma(L[p * Q + m], Cm[m * Q + c], s);
      G[p * Q + c] = -s;
      Lo[p * Q + c] = L[p * Q + c];
      LT[p * Q + c] = L[c * Q + p];
      double h = 0.0;
      if (Cn)
        for (int m = p; m < Q; ++m) h = fma(L[m * Q + p], Cn[c * Q + m], h);
      H[p * Q + c] = -h;
    }
}

// ---- host side -----------------------------------------------------------------------------

static int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return s ? atoi(s) : dflt;
}

static constexpr size_t kSmemBudget = 220 * 1024;

template <int NS, int MODE>
static constexpr size_t st3_warp_bytes() {
  return (size_t)St3<NS, MODE>::R * St3<NS, MODE>::SLOT * sizeof(double);
}
template <int NS, bool INNER>
static constexpr size_t sw3_warp_bytes() {
  return (size_t)Sw3<NS, INNER>::R * Sw3<NS, INNER>::SLOT * sizeof(double);
}

template <int NS>
static cudaError_t stencil3_n(const Geo& g, const FastOps& fo, int mode, const double* x,
                              const double* rin, double* y, const StencilShape& sh,
                              double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  const long long warps = (long long)g.N * sh.nchunk * sh.nstrip;
  cudaError_t e;
  if (mode == kDelta) {
    constexpr size_t per = st3_warp_bytes<NS, kDelta>();
    const int wpb = (int)std::max<size_t>(1, std::min<size_t>(4, kSmemBudget / per));
    const unsigned blocks = (unsigned)((warps + wpb - 1) / wpb);
    e = cudaFuncSetAttribute(k_stencil3<NS, kDelta>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(wpb * per));
    if (e != cudaSuccess) return e;
    k_stencil3<NS, kDelta><<<blocks, 32 * wpb, wpb * per, s>>>(g, fo, x, rin, y, sh.nchunk,
                                                               sh.nstrip, sh.rows, partials, st,
                                                               dotmode);
  } else {
    constexpr size_t per = st3_warp_bytes<NS, kOuterRhs>();
    const int wpb = (int)std::max<size_t>(1, std::min<size_t>(4, kSmemBudget / per));
    const unsigned blocks = (unsigned)((warps + wpb - 1) / wpb);
    e = cudaFuncSetAttribute(k_stencil3<NS, kOuterRhs>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(wpb * per));
    if (e != cudaSuccess) return e;
    k_stencil3<NS, kOuterRhs><<<blocks, 32 * wpb, wpb * per, s>>>(g, fo, x, rin, y, sh.nchunk,
                                                                  sh.nstrip, sh.rows, partials,
                                                                  st, kDotNone);
  }
  return cudaGetLastError();
}

cudaError_t launch_stencil3(const Geo& g, const FastOps& fo, int mode, const double* x,
                            const double* rin, double* y, const StencilShape& sh,
                            double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  switch (g.n) {
    case 1: return stencil3_n<1>(g, fo, mode, x, rin, y, sh, partials, st, dotmode, s);
    case 2: return stencil3_n<2>(g, fo, mode, x, rin, y, sh, partials, st, dotmode, s);
    case 3: return stencil3_n<3>(g, fo, mode, x, rin, y, sh, partials, st, dotmode, s);
    case 4: return stencil3_n<4>(g, fo, mode, x, rin, y, sh, partials, st, dotmode, s);
    default: return cudaErrorInvalidValue;
  }
}

int sweep3_warps(const Geo& g, int sm_count) {
  const int nchunk = (g.T1 + 31) / 32;
  const int n_items = g.V * nchunk;
  const int wsm = 4;   // warps per SM (measured round 1)
  return std::min(n_items, wsm * sm_count);
}

// persistent grid: never more warps than can be co-resident (items are strided by block)
template <typename K>
static unsigned resident_blocks(K kernel, size_t smem, int want, int sm_count) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 32, smem);
  per_sm = std::max(per_sm, 1);
  return (unsigned)std::max(1, std::min(want, per_sm * sm_count));
}

template <int NS>
static cudaError_t sweep3_n(const Geo& g, const FastOps& fo, bool inner, const double* rhs,
                            const double* th, double* out, const double* rdot, int sm_count,
                            double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  const int nchunk = (g.T1 + 31) / 32;
  const int n_items = g.V * nchunk;
  const int want = sweep3_warps(g, sm_count);
  cudaError_t e;
  unsigned blocks;
  if (inner) {
    constexpr size_t per = sw3_warp_bytes<NS, true>();
    e = cudaFuncSetAttribute(k_sweep3<NS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)per);
    if (e != cudaSuccess) return e;
    blocks = resident_blocks(k_sweep3<NS, true>, per, want, sm_count);
    k_sweep3<NS, true><<<blocks, 32, per, s>>>(g, fo, rhs, th, out, rdot, n_items, nchunk,
                                               partials, st, dotmode);
  } else {
    constexpr size_t per = sw3_warp_bytes<NS, false>();
    e = cudaFuncSetAttribute(k_sweep3<NS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)per);
    if (e != cudaSuccess) return e;
    blocks = resident_blocks(k_sweep3<NS, false>, per, want, sm_count);
    k_sweep3<NS, false><<<blocks, 32, per, s>>>(g, fo, rhs, th, out, rdot, n_items, nchunk,
                                                partials, st, dotmode);
  }
  return cudaGetLastError();
}

template <int NS, bool INNER, int MT>
static constexpr size_t sw6_warp_bytes() {
  return (size_t)Sw4<NS, INNER, MT>::R * Sw4<NS, INNER, MT>::SLOT * sizeof(double);
}

template <int NS, bool INNER, int MT>
static cudaError_t sweep6_launch(const Geo& g, const FastOps& fo, const double* rhs,
                                 const double* th, double* out, const double* rdot, int sm_count,
                                 double* partials, PcgState* st, int dotmode, cudaStream_t s,
                                 int wsm) {
  const int nchunk = (g.T1 + 8 * MT - 1) / (8 * MT);
  const int n_items = g.V * nchunk;
  const int want = std::min(n_items, std::max(1, wsm) * sm_count);
  constexpr size_t per = sw6_warp_bytes<NS, INNER, MT>();
  cudaError_t e = cudaFuncSetAttribute(k_sweep6<NS, INNER, MT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
  if (e != cudaSuccess) return e;
  const unsigned blocks = resident_blocks(k_sweep6<NS, INNER, MT>, per, want, sm_count);
  k_sweep6<NS, INNER, MT><<<blocks, 32, per, s>>>(g, fo, rhs, th, out, rdot, n_items, nchunk,
                                                  partials, st, dotmode);
  return cudaGetLastError();

}

template <int NS>
static cudaError_t sweep4_n(const Geo& g, const FastOps& fo, bool inner, const double* rhs,
                            const double* th, double* out, const double* rdot, int sm_count,
                            double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  // n = 4: the MT = 1 instantiation (255 registers + spills) faults with an illegal
  // instruction on B200; the two-tile variant is used instead.
  const int mt = NS == 4 ? 2 : 1;
  const int wsm = mt == 1 ? 8 : 4;
  if (mt == 2) {
    if (inner) return sweep6_launch<NS, true, 2>(g, fo, rhs, th, out, rdot, sm_count, partials, st, dotmode, s, wsm);
    return sweep6_launch<NS, false, 2>(g, fo, rhs, th, out, rdot, sm_count, partials, st, dotmode, s, wsm);
  }
  if constexpr (NS == 2) {
    if (inner) return sweep6_launch<NS, true, 1>(g, fo, rhs, th, out, rdot, sm_count, partials, st, dotmode, s, wsm);
    return sweep6_launch<NS, false, 1>(g, fo, rhs, th, out, rdot, sm_count, partials, st, dotmode, s, wsm);
  }
  return cudaErrorInvalidValue;
}


bool tc_supported(int n) { return (n == 2 || n == 4) && env_int("GQ_NO_DMMA", 0) == 0; }

cudaError_t launch_sweep3(const Geo& g, const FastOps& fo, bool inner, const double* rhs,
                          const double* th, double* out, const double* rdot, int sm_count,
                          double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  if (fo.fac4 != nullptr) {
    if (g.n == 2) return sweep4_n<2>(g, fo, inner, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
    if (g.n == 4) return sweep4_n<4>(g, fo, inner, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
  }
  switch (g.n) {
    case 1: return sweep3_n<1>(g, fo, inner, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
    case 2: return sweep3_n<2>(g, fo, inner, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
    case 3: return sweep3_n<3>(g, fo, inner, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
    case 4: return sweep3_n<4>(g, fo, inner, rhs, th, out, rdot, sm_count, partials, st, dotmode, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int NS>
static cudaError_t build_fast_n(const Geo& g, int npc, const Ops& op, double* oprow,
                                double* omega, double* fac3, double* fac4, cudaStream_t s) {
  const long long c1 = (long long)npc * g.nk;
  k_build_rows<NS><<<(unsigned)((c1 + 127) / 128), 128, 0, s>>>(g, npc, op.psi, op.xi, op.xit,
                                                                  oprow, omega);
  const long long c2 = (long long)npc * g.V * g.nb;
  if (fac3) k_build_fac3<NS><<<(unsigned)((c2 + 127) / 128), 128, 0, s>>>(g, npc, op.fac, fac3);
  if (fac4) k_build_fac4<NS><<<(unsigned)((c2 + 127) / 128), 128, 0, s>>>(g, npc, op.fac, fac4);
  return cudaGetLastError();
}

cudaError_t launch_build_fast(const Geo& g, int npc, const Ops& op, double* oprow, double* omega,
                              double* fac3, double* fac4, cudaStream_t s) {
  switch (g.n) {
    case 1: return build_fast_n<1>(g, npc, op, oprow, omega, fac3, nullptr, s);
    case 2: return build_fast_n<2>(g, npc, op, oprow, omega, fac3, fac4, s);
    case 3: return build_fast_n<3>(g, npc, op, oprow, omega, fac3, nullptr, s);
    case 4: return build_fast_n<4>(g, npc, op, oprow, omega, fac3, fac4, s);
    default: return cudaErrorInvalidValue;
  }
}

bool fast_supported(int n) {
  if (n == 1 || n == 2 || n == 3) return true;
  if (n == 4) return sw3_warp_bytes<4, true>() <= kSmemBudget && st3_warp_bytes<4, kDelta>() <= kSmemBudget;
  return false;
}

long long fast_max_blocks(const Geo& g, const StencilShape& sh, int sm_count) {
  const long long warps = (long long)g.N * sh.nchunk * sh.nstrip;
  const long long w4 = (long long)g.V * ((g.T1 + 7) / 8);
  return std::max<long long>({warps, (long long)sweep3_warps(g, sm_count), w4});
}

}  // namespace gq
