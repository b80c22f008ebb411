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
  extern __shared__ __align__(16) double smem[];
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
  const bool useful = tv && lane >= 1 && lane <= kHaloChunk;
  const unsigned vmask = __ballot_sync(0xffffffffu, tv);
  const int pc = tv ? fo.psi_cls[t] : 0;
  const int cA = __shfl_sync(0xffffffffu, pc, first_lane(vmask));
  const int cB = __shfl_sync(0xffffffffu, pc, last_lane(vmask));
  const double msel = (pc == cA) ? 0.0 : 1.0;
  const int psel = (pc == cA) ? 0 : 1;
  const double ke = (tv && t < g.T) ? 1.0 : 0.0;   // e_t exists (Xi_t, t < T)
  const double kf = (tv && t >= 1) ? 1.0 : 0.0;    // f_t exists (Xi_{t-1})
  const double ku = (t >= 1) ? 1.0 : 0.0;          // receives e_{t-1}
  const double kd = (t < g.T) ? 1.0 : 0.0;         // receives f_{t+1}
  (void)msel;
  const uint64_t pol = policy_evict_first();
  const uint64_t pol_op = policy_evict_last();
  double dot = 0.0;

  if (active) {
    const int i0 = strip * rows;
    const int i1 = min(g.K, i0 + rows);
    const long long rs = (long long)g.T1 * NS;
    const int dj[5] = {0, -1, 1, -2, 2};
    const double* cx[5];
    bool cok[5];
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      const int jj = j + dj[m];
      cok[m] = tv && jj >= 0 && jj < g.N;
      cx[m] = cok[m] ? x + ((long long)jj * g.K * g.T1 + t) * NS : x;
    }
    const double* cr = (MODE == kOuterRhs && tv) ? rin + ((long long)j * g.K * g.T1 + t) * NS : rin;
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
        e.v[k] *= ke;
        f.v[k] *= kf;
      }
      const Vec<NS> eu = shfl_up<NS>(e, 1);
      const Vec<NS> fd = shfl_down<NS>(f, 1);
      if (MODE == kDelta) {
#pragma unroll
        for (int k = 0; k < NS; ++k) acc.v[k] = (acc.v[k] + ku * eu.v[k]) + kd * fd.v[k];
      } else {   // y = r + (-(Xi_{t-1} x_{t-1}) - Xi_t' x_{t+1})
        const Vec<NS> rv = lds_rec<NS>(sl + 5 * REC + lane * NS);
#pragma unroll
        for (int k = 0; k < NS; ++k) acc.v[k] = rv.v[k] + ((0.0 - ku * eu.v[k]) - kd * fd.v[k]);
      }
      if (useful) {
        stv<NS>(y + ((long long)j * g.K * g.T1 + t) * NS + i * rs, acc);
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
  extern __shared__ __align__(16) double smem[];
  if (halted(st)) return;
  const int lane = threadIdx.x & 31;
  double* ring = smem;
  const uint64_t pol = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  const long long rs = (long long)g.T1 * NS;            // next row, same column and stage
  const long long cs = (long long)g.K * g.T1 * NS;      // next column
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
    const int psel = (pc == cA) ? 0 : 1;
    const bool two = cB != cA;
    const int a = 2 * v;
    const bool okb = a + 1 < g.N;
    const long long lane_off = (long long)(tv ? t : 0) * NS;
    const long long col_a = (long long)a * g.K * g.T1 * NS + lane_off;   // (a, row 0, t)
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

template <int NS, bool INNER>
struct Sw4 {
  static constexpr int Q = 4 * NS, QQ = Q * Q, B2 = NS * NS;
  static constexpr int NT = Q / 8;                   // N-tiles == k-pairs
  static constexpr int CH = 16;                      // chains per warp
  static constexpr int REC = CH * NS;                // doubles per record (16 stages)
  static constexpr int NRF = INNER ? 16 : 4;         // forward: tau (4) + theta (12)
  static constexpr int NR = NRF > 8 ? NRF : 8;       // backward: w (4) + r (4)
  static constexpr int FAC = 2 * QQ;                 // per class: L|-G or L^T|-H
  static constexpr int OMG = INNER ? 4 * 5 * B2 : 0; // per class: omega rows of 4 nodes
  static constexpr int SLOT = NR * REC + 2 * FAC + 2 * OMG;
  static constexpr int P = Sw4P<NS>::v;
  static constexpr int R = P + 1;
};

// copy NREC records (16 stages x NS doubles, contiguous in the stage-inner layout) into
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

template <int NS, bool INNER>
__global__ void __launch_bounds__(32) k_sweep4(Geo g, FastOps fo, const double* __restrict__ rhs,
                                               const double* __restrict__ th, double* out,
                                               const double* __restrict__ rdot, int n_items,
                                               int nchunk, double* partials, PcgState* st,
                                               int dotmode) {
  using C = Sw4<NS, INNER>;
  constexpr int Q = C::Q, QQ = C::QQ, B2 = C::B2, NT = C::NT, REC = C::REC;
  extern __shared__ __align__(16) double smem[];
  if (halted(st)) return;
  const int lane = threadIdx.x & 31;
  const int qd = lane & 3, rw = lane >> 2;
  double* ring = smem;
  const uint64_t pol = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  const long long rs = (long long)g.T1 * NS;
  const long long cs = (long long)g.K * g.T1 * NS;
  double dot = 0.0;

#pragma unroll 1
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int v = item / nchunk, chunk = item % nchunk;
    const int t0 = chunk * 16;
    const int nvalid = min(16, g.T1 - t0);
    // chain (stage) of this lane in M-tile m: t0 + 8m + rw
    int cls[2];
    bool tvm[2];
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int t = t0 + 8 * m + rw;
      tvm[m] = t < g.T1;
      cls[m] = tvm[m] ? fo.psi_cls[t] : -1;
    }
    const int cA = fo.psi_cls[t0];
    const int cB = fo.psi_cls[t0 + nvalid - 1];
    const bool two = cB != cA;
    // per M-tile: classes present (warp-uniform)
    bool tileA[2], tileB[2];
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      tileA[m] = __any_sync(0xffffffffu, cls[m] == cA);
      tileB[m] = two && __any_sync(0xffffffffu, cls[m] == cB);
    }
    const int a = 2 * v;
    const bool okb = a + 1 < g.N;
    const long long col_a = (long long)a * g.K * g.T1 * NS + (long long)t0 * NS;
    const double* FA = fo.fac4 + ((long long)cA * g.V + v) * g.nb * 4 * QQ;
    const double* FB = fo.fac4 + ((long long)cB * g.V + v) * g.nb * 4 * QQ;
    const double* OA = fo.omega + ((long long)cA * g.nk + (long long)a * g.K) * 5 * B2;
    const double* OB = fo.omega + ((long long)cB * g.nk + (long long)a * g.K) * 5 * B2;
    // features owned by this lane in N-tile h: 8h + 2qd + {0,1}
    //   -> node slot nd(h) = (8h + 2qd) / NS, components c0(h) = (8h + 2qd) % NS
    auto nd_of = [&](int h) { return (8 * h + 2 * qd) / NS; };
    auto co_of = [&](int h) { return (8 * h + 2 * qd) % NS; };

    // ---------------- forward ----------------
    auto issue_f = [&](int k, double* sl) {
      if (k < g.nb) {
        const int i0 = 2 * k;
        const bool ok1 = i0 + 1 < g.K;
        const long long r0 = col_a + i0 * rs;
        const double* src[C::NRF];
        src[0] = rhs + r0;
        src[1] = okb ? rhs + r0 + cs : nullptr;
        src[2] = ok1 ? rhs + r0 + rs : nullptr;
        src[3] = (ok1 && okb) ? rhs + r0 + rs + cs : nullptr;
        if constexpr (INNER) {
          const int tc[12] = {-2, -2, -1, -1, -1, -1, 2, 2, 2, 2, 3, 3};
          const int tr[12] = {0, 1, -1, 0, 1, 2, -1, 0, 1, 2, 0, 1};
#pragma unroll
          for (int m = 0; m < 12; ++m) {
            const int jj = a + tc[m], ii = i0 + tr[m];
            src[4 + m] = (jj >= 0 && jj < g.N && ii >= 0 && ii < g.K)
                             ? th + r0 + tc[m] * cs + tr[m] * rs : nullptr;
          }
        }
        cp_records<NS, C::NRF>(sl, src, nvalid, lane, rhs, pol);
        double* sf = sl + C::NR * REC;
        warp_copy<NS>(sf, FA + (long long)k * 4 * QQ, 2 * QQ, true, lane, pol_keep);
        if (two) warp_copy<NS>(sf + C::FAC, FB + (long long)k * 4 * QQ, 2 * QQ, true, lane, pol_keep);
        if (INNER) {
          double* so = sf + 2 * C::FAC;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const bool ok = (s & 1 ? okb : true) && (s >> 1 ? ok1 : true);
            const long long off = ((long long)(s & 1) * g.K + i0 + (s >> 1)) * 5 * B2;
            warp_copy<NS>(so + s * 5 * B2, ok ? OA + off : OA, 5 * B2, ok, lane, pol_keep);
            if (two)
              warp_copy<NS>(so + C::OMG + s * 5 * B2, ok ? OB + off : OB, 5 * B2, ok, lane, pol_keep);
          }
        }
      }
      cp_commit();
    };
    // running W_{k-1} fragments: [m][h] = 2 doubles
    double wd[2][NT][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h) wd[m][h][0] = wd[m][h][1] = 0.0;
    int sc = 0, si = 0;
#pragma unroll 1
    for (int p = 0; p < C::P; ++p) {
      issue_f(p, ring + si * C::SLOT);
      si = (si + 1 == C::R) ? 0 : si + 1;
    }
#pragma unroll 1
    for (int k = 0; k < g.nb; ++k) {
      issue_f(k + C::P, ring + si * C::SLOT);
      si = (si + 1 == C::R) ? 0 : si + 1;
      cp_wait<C::P>();
      __syncwarp();
      const double* sl = ring + sc * C::SLOT;
      sc = (sc + 1 == C::R) ? 0 : sc + 1;
      // tau pairs (A fragments of the rhs) per M-tile and k-pair
      double bp[2][NT][2];
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int srow = 8 * m + rw;   // stage row inside the records
#pragma unroll
        for (int h = 0; h < NT; ++h) {
          const double2 bv =
              *reinterpret_cast<const double2*>(sl + nd_of(h) * REC + srow * NS + co_of(h));
          bp[m][h][0] = bv.x;
          bp[m][h][1] = bv.y;
          if (INNER) {
            // minus the cross-pair blocks (rows co, co+1 of node nd) times theta
            const int nd = nd_of(h), ri = nd >> 1, col_odd = nd & 1;
            const int sel = (cls[m] == cB && two) ? 1 : 0;
            const double* om = sl + C::NR * REC + 2 * C::FAC + sel * C::OMG + nd * 5 * B2;
            const int tix0[5] = {0, 2, 3, 4, 7};
            const int tix1[5] = {3, 6, 7, 8, 10};
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int u = 0; u < 5; ++u) {
              const int ti = (col_odd ? tix1[u] : tix0[u]) + ri;
              const double* tr = sl + (4 + ti) * REC + srow * NS;
              const double* M = om + u * B2 + co_of(h) * NS;
#pragma unroll
              for (int c = 0; c < NS; ++c) {
                s0 = fma(M[c], tr[c], s0);
                s1 = fma(M[NS + c], tr[c], s1);
              }
            }
            bp[m][h][0] -= s0;
            bp[m][h][1] -= s1;
          }
        }
      }
      // D = tau^T L^T - W^T G^T, per class present in the tile
      double dn[2][NT][2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int h = 0; h < NT; ++h) dn[m][h][0] = dn[m][h][1] = 0.0;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const double* L = sl + C::NR * REC + pass * C::FAC;
        const double* Gm = L + QQ;
        const int cx = pass ? cB : cA;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          if (pass == 0 ? !tileA[m] : !tileB[m]) continue;
          const bool on = cls[m] == cx;
#pragma unroll
          for (int h = 0; h < NT; ++h) {
#pragma unroll
            for (int sg = 0; sg < NT; ++sg) {
              const double2 lb =
                  *reinterpret_cast<const double2*>(L + (8 * h + rw) * Q + 8 * sg + 2 * qd);
              const double2 gb =
                  *reinterpret_cast<const double2*>(Gm + (8 * h + rw) * Q + 8 * sg + 2 * qd);
              dmma(dn[m][h][0], dn[m][h][1], on ? bp[m][sg][0] : 0.0, lb.x);
              dmma(dn[m][h][0], dn[m][h][1], on ? bp[m][sg][1] : 0.0, lb.y);
              dmma(dn[m][h][0], dn[m][h][1], on ? wd[m][sg][0] : 0.0, gb.x);
              dmma(dn[m][h][0], dn[m][h][1], on ? wd[m][sg][1] : 0.0, gb.y);
            }
          }
        }
      }
      // park w_k (evict_last) and carry it
      const long long r0 = col_a + 2 * k * rs;
      const bool ok1 = 2 * k + 1 < g.K;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
#pragma unroll
        for (int h = 0; h < NT; ++h) {
          wd[m][h][0] = dn[m][h][0];
          wd[m][h][1] = dn[m][h][1];
          const int nd = nd_of(h);
          const bool ok = tvm[m] && (nd & 1 ? okb : true) && (nd >> 1 ? ok1 : true);
          if (ok) {
            double* p = out + r0 + (nd & 1) * cs + (nd >> 1) * rs + (8 * m + rw) * NS + co_of(h);
            asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p),
                         "d"(dn[m][h][0]), "d"(dn[m][h][1]), "l"(pol_keep)
                         : "memory");
          }
        }
      }
      __syncwarp();
    }
    cp_wait<0>();
    __threadfence();
    __syncwarp();

    // ---------------- backward ----------------
    auto issue_b = [&](int k, double* sl) {
      if (k >= 0) {
        const bool ok1 = 2 * k + 1 < g.K;
        const long long r0 = col_a + 2 * k * rs;
        const double* src[8];
        src[0] = out + r0;
        src[1] = okb ? out + r0 + cs : nullptr;
        src[2] = ok1 ? out + r0 + rs : nullptr;
        src[3] = (ok1 && okb) ? out + r0 + rs + cs : nullptr;
        const bool dm = dotmode != kDotNone;
        src[4] = dm ? rdot + r0 : nullptr;
        src[5] = dm && okb ? rdot + r0 + cs : nullptr;
        src[6] = dm && ok1 ? rdot + r0 + rs : nullptr;
        src[7] = dm && ok1 && okb ? rdot + r0 + rs + cs : nullptr;
        cp_records<NS, 8>(sl, src, nvalid, lane, out, pol);
        double* sf = sl + C::NR * REC;
        warp_copy<NS>(sf, FA + (long long)k * 4 * QQ + 2 * QQ, 2 * QQ, true, lane, pol_keep);
        if (two)
          warp_copy<NS>(sf + C::FAC, FB + (long long)k * 4 * QQ + 2 * QQ, 2 * QQ, true, lane, pol_keep);
      }
      cp_commit();
    };
    double xd[2][NT][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h) xd[m][h][0] = xd[m][h][1] = 0.0;
    sc = 0;
    si = 0;
#pragma unroll 1
    for (int p = 0; p < C::P; ++p) {
      issue_b(g.nb - 1 - p, ring + si * C::SLOT);
      si = (si + 1 == C::R) ? 0 : si + 1;
    }
#pragma unroll 1
    for (int k = g.nb - 1; k >= 0; --k) {
      issue_b(k - C::P, ring + si * C::SLOT);
      si = (si + 1 == C::R) ? 0 : si + 1;
      cp_wait<C::P>();
      __syncwarp();
      const double* sl = ring + sc * C::SLOT;
      sc = (sc + 1 == C::R) ? 0 : sc + 1;
      double wp[2][NT][2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int h = 0; h < NT; ++h) {
          const double2 wv = *reinterpret_cast<const double2*>(
              sl + nd_of(h) * REC + (8 * m + rw) * NS + co_of(h));
          wp[m][h][0] = wv.x;
          wp[m][h][1] = wv.y;
        }
      double dn[2][NT][2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int h = 0; h < NT; ++h) dn[m][h][0] = dn[m][h][1] = 0.0;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const double* LT = sl + C::NR * REC + pass * C::FAC;
        const double* Hm = LT + QQ;
        const int cx = pass ? cB : cA;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          if (pass == 0 ? !tileA[m] : !tileB[m]) continue;
          const bool on = cls[m] == cx;
#pragma unroll
          for (int h = 0; h < NT; ++h) {
#pragma unroll
            for (int sg = 0; sg < NT; ++sg) {
              const double2 lb =
                  *reinterpret_cast<const double2*>(LT + (8 * h + rw) * Q + 8 * sg + 2 * qd);
              const double2 hb =
                  *reinterpret_cast<const double2*>(Hm + (8 * h + rw) * Q + 8 * sg + 2 * qd);
              dmma(dn[m][h][0], dn[m][h][1], on ? wp[m][sg][0] : 0.0, lb.x);
              dmma(dn[m][h][0], dn[m][h][1], on ? wp[m][sg][1] : 0.0, lb.y);
              dmma(dn[m][h][0], dn[m][h][1], on ? xd[m][sg][0] : 0.0, hb.x);
              dmma(dn[m][h][0], dn[m][h][1], on ? xd[m][sg][1] : 0.0, hb.y);
            }
          }
        }
      }
      const long long r0 = col_a + 2 * k * rs;
      const bool ok1 = 2 * k + 1 < g.K;
#pragma unroll
      for (int m = 0; m < 2; ++m) {
#pragma unroll
        for (int h = 0; h < NT; ++h) {
          xd[m][h][0] = dn[m][h][0];
          xd[m][h][1] = dn[m][h][1];
          const int nd = nd_of(h);
          const bool ok = tvm[m] && (nd & 1 ? okb : true) && (nd >> 1 ? ok1 : true);
          if (ok) {
            const long long off =
                r0 + (nd & 1) * cs + (nd >> 1) * rs + (8 * m + rw) * NS + co_of(h);
            *reinterpret_cast<double2*>(out + off) = make_double2(dn[m][h][0], dn[m][h][1]);
            if (dotmode != kDotNone) {
              const double2 rv = *reinterpret_cast<const double2*>(
                  sl + (4 + nd) * REC + (8 * m + rw) * NS + co_of(h));
              dot = fma(dn[m][h][0], rv.x, dot);
              dot = fma(dn[m][h][1], rv.y, dot);
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
        st->mu = mu;
      } else {
        st->beta = mu / st->mu;
        st->mu = mu;
      }
    }
  }
}


// ---- sweep v5: lean DMMA chain solver -----------------------------------------------------
// Same math and fragment layout as v4 (see above), restructured for issue efficiency:
//  * every address is computed once per item; per block only row offsets advance;
//  * the Linv*tau products (independent of the recurrence) and the two G/H k-steps use
//    separate accumulators, so one DMMA (~90-cycle latency) sits on the critical path;
//  * tiles holding a single stage class (all but the t=0 tile of a time-invariant
//    problem) skip the class masking entirely (TWO=false instantiation).

template <int NS, bool INNER, bool TWO>
__device__ __forceinline__ void sweep5_item(
    const Geo& g, const FastOps& fo, const double* __restrict__ rhs,
    const double* __restrict__ th, double* out, const double* __restrict__ rdot, int dotmode,
    double* ring, int lane, int v, int t0, int nvalid, int cA, int cB, const int (&cls)[2],
    const bool (&tvm)[2], uint64_t pol, uint64_t pol_keep, double& dot) {
  using C = Sw4<NS, INNER>;
  constexpr int Q = C::Q, QQ = C::QQ, B2 = C::B2, NT = C::NT, REC = C::REC, P = C::P, R = C::R;
  const int qd = lane & 3, rw = lane >> 2;
  const long long rs = (long long)g.T1 * NS;
  const long long cs = (long long)g.K * g.T1 * NS;
  const int a = 2 * v;
  const bool okb = a + 1 < g.N;
  const long long col_a = (long long)a * g.K * g.T1 * NS + (long long)t0 * NS;
  const double* FA = fo.fac4 + ((long long)cA * g.V + v) * g.nb * 4 * QQ;
  const double* FB = fo.fac4 + ((long long)cB * g.V + v) * g.nb * 4 * QQ;
  const double* OA = fo.omega + ((long long)cA * g.nk + (long long)a * g.K) * 5 * B2;
  const double* OB = fo.omega + ((long long)cB * g.nk + (long long)a * g.K) * 5 * B2;

  // ---- record copy plan: chunk j of this lane -> (record, stage) ----
  // NS == 2: 16 chunks/record, chunk j covers record 2j + (lane >> 4), stage lane & 15
  // NS == 4: 32 chunks/record, chunk j covers record j, stage lane >> 1 (half lane & 1)
  const int my_stage = NS == 2 ? (lane & 15) : (lane >> 1);
  const int my_w = NS == 2 ? (lane & 15) : lane;          // chunk inside the record
  const bool stage_ok = my_stage < nvalid;
  // record geometry relative to (col a, row 2k): column offset, row offset
  constexpr int NRF = C::NRF;
  constexpr int JF = NRF * NS / 4;                          // chunks per lane, forward
  auto rec_geo = [&](int r, int& dc, int& dr) {
    const int base_c[4] = {0, 1, 0, 1}, base_r[4] = {0, 0, 1, 1};
    const int tc[12] = {-2, -2, -1, -1, -1, -1, 2, 2, 2, 2, 3, 3};
    const int tr[12] = {0, 1, -1, 0, 1, 2, -1, 0, 1, 2, 0, 1};
    if (r < 4) {
      dc = base_c[r];
      dr = base_r[r];
    } else {
      dc = tc[r - 4];
      dr = tr[r - 4];
    }
  };
  const double* fsrc[JF];
  int frow[JF];
  bool fcol[JF];
  int fdst[JF];
#pragma unroll
  for (int j = 0; j < JF; ++j) {
    const int r = NS == 2 ? 2 * j + (lane >> 4) : j;
    int dc, dr;
    rec_geo(r, dc, dr);
    const int jj = a + dc;
    fcol[j] = stage_ok && jj >= 0 && jj < g.N;
    frow[j] = dr;
    fsrc[j] = (r < 4 ? rhs : th) + col_a + (long long)dc * cs + 2 * my_w;
    fdst[j] = r * REC + 2 * my_w;
  }
  // factor / omega copy offsets (uniform data, 16-byte chunks)
  constexpr int FCH = 2 * QQ / 2;          // chunks of the forward/backward factor pair
  constexpr int OCH = 5 * B2 / 2;          // chunks of one node's omega rows

  // ---- owned features: N-tile h -> node nd(h), component co(h) ----
  int nd[NT], co[NT];
#pragma unroll
  for (int h = 0; h < NT; ++h) {
    nd[h] = (8 * h + 2 * qd) / NS;
    co[h] = (8 * h + 2 * qd) % NS;
  }
  // global offsets of owned pairs at block 0 (stage row 8m + rw)
  long long own[2][NT];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int h = 0; h < NT; ++h)
      own[m][h] = col_a + (nd[h] & 1) * cs + (nd[h] >> 1) * rs + (8 * m + rw) * NS + co[h];
  bool own_col[NT];
#pragma unroll
  for (int h = 0; h < NT; ++h) own_col[h] = (nd[h] & 1) ? okb : true;

  auto issue_f = [&](int k, double* sl) {
    if (k < g.nb) {
      const long long roff = 2LL * k * rs;
#pragma unroll
      for (int j = 0; j < JF; ++j) {
        const int row = 2 * k + frow[j];
        const bool ok = fcol[j] && row >= 0 && row < g.K;
        cpa16(sl + fdst[j], ok ? fsrc[j] + roff + (long long)frow[j] * rs : rhs, ok, pol);
      }
      double* sf = sl + C::NR * REC;
      const double* fa = FA + (long long)k * 4 * QQ;
#pragma unroll
      for (int c = lane; c < FCH; c += 32) cpa16(sf + 2 * c, fa + 2 * c, true, pol_keep);
      if (TWO) {
        const double* fb = FB + (long long)k * 4 * QQ;
#pragma unroll
        for (int c = lane; c < FCH; c += 32) cpa16(sf + C::FAC + 2 * c, fb + 2 * c, true, pol_keep);
      }
      if (INNER) {
        double* so = sf + 2 * C::FAC;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int row = 2 * k + (s >> 1);
          const bool ok = ((s & 1) ? okb : true) && row < g.K;
          const long long off = ((long long)(s & 1) * g.K + row) * 5 * B2;
#pragma unroll
          for (int c = lane; c < OCH; c += 32) {
            cpa16(so + s * 5 * B2 + 2 * c, ok ? OA + off + 2 * c : OA, ok, pol_keep);
            if (TWO) cpa16(so + C::OMG + s * 5 * B2 + 2 * c, ok ? OB + off + 2 * c : OB, ok, pol_keep);
          }
        }
      }
    }
    cp_commit();
  };

  double wd[2][NT][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int h = 0; h < NT; ++h) wd[m][h][0] = wd[m][h][1] = 0.0;
  int sc = 0, si = 0;
#pragma unroll 1
  for (int p = 0; p < P; ++p) {
    issue_f(p, ring + si * C::SLOT);
    si = (si + 1 == R) ? 0 : si + 1;
  }
#pragma unroll 1
  for (int k = 0; k < g.nb; ++k) {
    issue_f(k + P, ring + si * C::SLOT);
    si = (si + 1 == R) ? 0 : si + 1;
    cp_wait<P>();
    __syncwarp();
    const double* sl = ring + sc * C::SLOT;
    sc = (sc + 1 == R) ? 0 : sc + 1;
    const double* sf = sl + C::NR * REC;
    // tau pairs
    double bp[2][NT][2];
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int srow = 8 * m + rw;
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        const double2 bv = *reinterpret_cast<const double2*>(sl + nd[h] * REC + srow * NS + co[h]);
        bp[m][h][0] = bv.x;
        bp[m][h][1] = bv.y;
        if (INNER) {
          const int ri = nd[h] >> 1;
          const int sel = (TWO && cls[m] == cB) ? 1 : 0;
          const double* om = sf + 2 * C::FAC + sel * C::OMG + nd[h] * 5 * B2 + co[h] * NS;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int u = 0; u < 5; ++u) {
            const int tix = (nd[h] & 1) ? (u == 0 ? 3 : u == 1 ? 6 : u == 2 ? 7 : u == 3 ? 8 : 10)
                                        : (u == 0 ? 0 : u == 1 ? 2 : u == 2 ? 3 : u == 3 ? 4 : 7);
            const double* tr = sl + (4 + tix + ri) * REC + srow * NS;
#pragma unroll
            for (int c = 0; c < NS; c += 2) {
              const double2 tv2 = *reinterpret_cast<const double2*>(tr + c);
              const double2 m0 = *reinterpret_cast<const double2*>(om + u * B2 + c);
              const double2 m1 = *reinterpret_cast<const double2*>(om + u * B2 + NS + c);
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
    double dl[2][NT][2], dg0[2][NT][2], dg1[2][NT][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h)
        dl[m][h][0] = dl[m][h][1] = dg0[m][h][0] = dg0[m][h][1] = dg1[m][h][0] = dg1[m][h][1] = 0.0;
#pragma unroll
    for (int pass = 0; pass < (TWO ? 2 : 1); ++pass) {
      const double* L = sf + pass * C::FAC;
      const double* Gm = L + QQ;
      const int cx = pass ? cB : cA;
#pragma unroll
      for (int h = 0; h < NT; ++h) {
#pragma unroll
        for (int sg = 0; sg < NT; ++sg) {
          const double2 lb = *reinterpret_cast<const double2*>(L + (8 * h + rw) * Q + 8 * sg + 2 * qd);
          const double2 gb = *reinterpret_cast<const double2*>(Gm + (8 * h + rw) * Q + 8 * sg + 2 * qd);
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            const bool on = !TWO || cls[m] == cx;
            dmma(dl[m][h][0], dl[m][h][1], on ? bp[m][sg][0] : 0.0, lb.x);
            dmma(dl[m][h][0], dl[m][h][1], on ? bp[m][sg][1] : 0.0, lb.y);
            dmma(dg0[m][h][0], dg0[m][h][1], on ? wd[m][sg][0] : 0.0, gb.x);
            dmma(dg1[m][h][0], dg1[m][h][1], on ? wd[m][sg][1] : 0.0, gb.y);
          }
        }
      }
    }
    const long long roff = 2LL * k * rs;
    const bool ok1 = 2 * k + 1 < g.K;
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        wd[m][h][0] = dl[m][h][0] + (dg0[m][h][0] + dg1[m][h][0]);
        wd[m][h][1] = dl[m][h][1] + (dg0[m][h][1] + dg1[m][h][1]);
        const bool ok = tvm[m] && own_col[h] && ((nd[h] >> 1) ? ok1 : true);
        if (ok) {
          double* p = out + own[m][h] + roff;
          asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p),
                       "d"(wd[m][h][0]), "d"(wd[m][h][1]), "l"(pol_keep)
                       : "memory");
        }
      }
    __syncwarp();
  }
  cp_wait<0>();
  __threadfence();
  __syncwarp();

  // ---------------- backward ----------------
  constexpr int JB = 8 * NS / 4;             // w (4) + r (4) records
  const double* bsrc[JB];
  int brow[JB];
  bool bcol[JB];
  int bdst[JB];
#pragma unroll
  for (int j = 0; j < JB; ++j) {
    const int r = NS == 2 ? 2 * j + (lane >> 4) : j;
    const int dc = r & 1, dr = (r >> 1) & 1;
    bcol[j] = stage_ok && (dc ? okb : true) && (r < 4 || dotmode != kDotNone);
    brow[j] = dr;
    bsrc[j] = (r < 4 ? (const double*)out : rdot) + col_a + (long long)dc * cs + 2 * my_w;
    bdst[j] = r * REC + 2 * my_w;
  }
  auto issue_b = [&](int k, double* sl) {
    if (k >= 0) {
      const long long roff = 2LL * k * rs;
#pragma unroll
      for (int j = 0; j < JB; ++j) {
        const int row = 2 * k + brow[j];
        const bool ok = bcol[j] && row < g.K;
        cpa16(sl + bdst[j], ok ? bsrc[j] + roff + (long long)brow[j] * rs : rhs, ok, pol);
      }
      double* sf = sl + C::NR * REC;
      const double* fa = FA + (long long)k * 4 * QQ + 2 * QQ;
#pragma unroll
      for (int c = lane; c < FCH; c += 32) cpa16(sf + 2 * c, fa + 2 * c, true, pol_keep);
      if (TWO) {
        const double* fb = FB + (long long)k * 4 * QQ + 2 * QQ;
#pragma unroll
        for (int c = lane; c < FCH; c += 32) cpa16(sf + C::FAC + 2 * c, fb + 2 * c, true, pol_keep);
      }
    }
    cp_commit();
  };
  double xd[2][NT][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int h = 0; h < NT; ++h) xd[m][h][0] = xd[m][h][1] = 0.0;
  sc = 0;
  si = 0;
#pragma unroll 1
  for (int p = 0; p < P; ++p) {
    issue_b(g.nb - 1 - p, ring + si * C::SLOT);
    si = (si + 1 == R) ? 0 : si + 1;
  }
#pragma unroll 1
  for (int k = g.nb - 1; k >= 0; --k) {
    issue_b(k - P, ring + si * C::SLOT);
    si = (si + 1 == R) ? 0 : si + 1;
    cp_wait<P>();
    __syncwarp();
    const double* sl = ring + sc * C::SLOT;
    sc = (sc + 1 == R) ? 0 : sc + 1;
    const double* sf = sl + C::NR * REC;
    double wp[2][NT][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        const double2 wv = *reinterpret_cast<const double2*>(sl + nd[h] * REC + (8 * m + rw) * NS + co[h]);
        wp[m][h][0] = wv.x;
        wp[m][h][1] = wv.y;
      }
    double dl[2][NT][2], dg0[2][NT][2], dg1[2][NT][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h)
        dl[m][h][0] = dl[m][h][1] = dg0[m][h][0] = dg0[m][h][1] = dg1[m][h][0] = dg1[m][h][1] = 0.0;
#pragma unroll
    for (int pass = 0; pass < (TWO ? 2 : 1); ++pass) {
      const double* LT = sf + pass * C::FAC;
      const double* Hm = LT + QQ;
      const int cx = pass ? cB : cA;
#pragma unroll
      for (int h = 0; h < NT; ++h) {
#pragma unroll
        for (int sg = 0; sg < NT; ++sg) {
          const double2 lb = *reinterpret_cast<const double2*>(LT + (8 * h + rw) * Q + 8 * sg + 2 * qd);
          const double2 hb = *reinterpret_cast<const double2*>(Hm + (8 * h + rw) * Q + 8 * sg + 2 * qd);
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            const bool on = !TWO || cls[m] == cx;
            dmma(dl[m][h][0], dl[m][h][1], on ? wp[m][sg][0] : 0.0, lb.x);
            dmma(dl[m][h][0], dl[m][h][1], on ? wp[m][sg][1] : 0.0, lb.y);
            dmma(dg0[m][h][0], dg0[m][h][1], on ? xd[m][sg][0] : 0.0, hb.x);
            dmma(dg1[m][h][0], dg1[m][h][1], on ? xd[m][sg][1] : 0.0, hb.y);
          }
        }
      }
    }
    const long long roff = 2LL * k * rs;
    const bool ok1 = 2 * k + 1 < g.K;
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        xd[m][h][0] = dl[m][h][0] + (dg0[m][h][0] + dg1[m][h][0]);
        xd[m][h][1] = dl[m][h][1] + (dg0[m][h][1] + dg1[m][h][1]);
        const bool ok = tvm[m] && own_col[h] && ((nd[h] >> 1) ? ok1 : true);
        if (ok) {
          *reinterpret_cast<double2*>(out + own[m][h] + roff) = make_double2(xd[m][h][0], xd[m][h][1]);
          if (dotmode != kDotNone) {
            const double2 rv = *reinterpret_cast<const double2*>(sl + (4 + nd[h]) * REC + (8 * m + rw) * NS + co[h]);
            dot = fma(xd[m][h][0], rv.x, dot);
            dot = fma(xd[m][h][1], rv.y, dot);
          }
        }
      }
    __syncwarp();
  }
  cp_wait<0>();
  __syncwarp();
}

template <int NS, bool INNER>
__global__ void __launch_bounds__(32) k_sweep5(Geo g, FastOps fo, const double* __restrict__ rhs,
                                               const double* __restrict__ th, double* out,
                                               const double* __restrict__ rdot, int n_items,
                                               int nchunk, double* partials, PcgState* st,
                                               int dotmode) {
  extern __shared__ __align__(16) double smem[];
  if (halted(st)) return;
  const int lane = threadIdx.x & 31;
  const int rw = lane >> 2;
  const uint64_t pol = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  double dot = 0.0;
#pragma unroll 1
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int v = item / nchunk, chunk = item % nchunk;
    const int t0 = chunk * 16;
    const int nvalid = min(16, g.T1 - t0);
    int cls[2];
    bool tvm[2];
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int t = t0 + 8 * m + rw;
      tvm[m] = t < g.T1;
      cls[m] = tvm[m] ? fo.psi_cls[t] : -1;
    }
    const int cA = fo.psi_cls[t0];
    const int cB = fo.psi_cls[t0 + nvalid - 1];
    if (cA == cB)
      sweep5_item<NS, INNER, false>(g, fo, rhs, th, out, rdot, dotmode, smem, lane, v, t0, nvalid,
                                    cA, cB, cls, tvm, pol, pol_keep, dot);
    else
      sweep5_item<NS, INNER, true>(g, fo, rhs, th, out, rdot, dotmode, smem, lane, v, t0, nvalid,
                                   cA, cB, cls, tvm, pol, pol_keep, dot);
  }
  if (dotmode != kDotNone) {
    double mu;
    if (grid_reduce<false>(dot, partials, &st->counter[2], mu) && threadIdx.x == 0) {
      if (dotmode == kDotInit) {
        st->mu = mu;
      } else {
        st->beta = mu / st->mu;
        st->mu = mu;
      }
    }
  }
}

// fac4[pc][v][k] = L_k^-1 | -G_k | L_k^-T | -H_k  (row-major q x q each)
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
  const int wsm = std::max(1, env_int("GQ_SWEEP_WARPS_PER_SM", 4));
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

template <int NS, bool INNER>
static constexpr size_t sw4_warp_bytes() {
  return (size_t)Sw4<NS, INNER>::R * Sw4<NS, INNER>::SLOT * sizeof(double);
}

template <int NS>
static cudaError_t sweep4_n(const Geo& g, const FastOps& fo, bool inner, const double* rhs,
                            const double* th, double* out, const double* rdot, int sm_count,
                            double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  const int nchunk = (g.T1 + 15) / 16;
  const int n_items = g.V * nchunk;
  const int want = std::min(n_items, std::max(1, env_int("GQ_SWEEP_WARPS_PER_SM", 4)) * sm_count);
  cudaError_t e;
  unsigned blocks;
  if (inner) {
    constexpr size_t per = sw4_warp_bytes<NS, true>();
    e = cudaFuncSetAttribute(k_sweep5<NS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)per);
    if (e != cudaSuccess) return e;
    blocks = resident_blocks(k_sweep5<NS, true>, per, want, sm_count);
    k_sweep5<NS, true><<<blocks, 32, per, s>>>(g, fo, rhs, th, out, rdot, n_items, nchunk,
                                               partials, st, dotmode);
  } else {
    constexpr size_t per = sw4_warp_bytes<NS, false>();
    e = cudaFuncSetAttribute(k_sweep5<NS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)per);
    if (e != cudaSuccess) return e;
    blocks = resident_blocks(k_sweep5<NS, false>, per, want, sm_count);
    k_sweep5<NS, false><<<blocks, 32, per, s>>>(g, fo, rhs, th, out, rdot, n_items, nchunk,
                                                partials, st, dotmode);
  }
  return cudaGetLastError();
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
  const long long w4 = (long long)g.V * ((g.T1 + 15) / 16);
  return std::max<long long>({warps, (long long)sweep3_warps(g, sm_count), w4});
}

}  // namespace gq
