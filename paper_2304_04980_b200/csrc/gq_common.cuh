// Shared definitions for the B200 PCGM kernels (sm_100a, fp64).
//
// Device vector layout ("stage-inner"): every multiplier vector is stored as
//   v[j][i][t][k]   index = ((j*K + i)*TS + t)*n + k
// with the stage stride TS >= T1 a multiple of 8 and the vector pointer itself T0 stages past
// its 128-byte aligned allocation (Geo::TS, gq_api.cu), so that the 8-stage records of the
// chain sweeps (and every node's first record) are whole 128-byte lines.  The padding stages
// hold zeros and are never written.
// i.e. node-major with the stage index innermost.  A warp maps its 32 lanes onto 32
// consecutive stages of ONE grid node, so
//   * every vector load/store of a warp is one contiguous 32*n*8-byte segment, and
//   * all operator data (Psi/Xi blocks, pair factors), which is per node and per stage
//     CLASS (time-invariant problems have 2 classes), is warp-uniform -> broadcast loads.
// The reference order (t, j, i, k) (gridlq/grid_problem.py:143-144) is only used at the
// C-ABI boundary; gq_layout.cu converts with a tiled transpose.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gq {

constexpr int kWarp = 32;
constexpr int kHaloChunk = 30;   // useful stages per warp when t+-1 exchange is needed

// 13-point diamond (di, dj); the first five are the 5-point stencil
//   0 self, 1 north (-1,0), 2 south (+1,0), 3 west (0,-1), 4 east (0,+1),
//   5 (-2,0), 6 (+2,0), 7 (0,-2), 8 (0,+2), 9 (-1,-1), 10 (-1,+1), 11 (+1,-1), 12 (+1,+1)
__host__ __device__ __forceinline__ constexpr int odi(int o) {
  return (o == 1 || o == 9 || o == 10) ? -1
       : (o == 2 || o == 11 || o == 12) ? 1
       : (o == 5) ? -2 : (o == 6) ? 2 : 0;
}
__host__ __device__ __forceinline__ constexpr int odj(int o) {
  return (o == 3 || o == 9 || o == 11) ? -1
       : (o == 4 || o == 10 || o == 12) ? 1
       : (o == 7) ? -2 : (o == 8) ? 2 : 0;
}
// coupling direction (west=0, east=1, north=2, south=3) of 5-point slot u>=1
__host__ __device__ __forceinline__ constexpr int slot_dir(int u) {
  return u == 1 ? 2 : u == 2 ? 3 : u == 3 ? 0 : 1;
}
__host__ __device__ __forceinline__ constexpr int slot_opp(int u) {
  return u == 1 ? 2 : u == 2 ? 1 : u == 3 ? 4 : u == 4 ? 3 : 0;
}

struct Geo {
  int K, N, T, T1, n;
  int V, nb;          // column pairs, 2-row blocks per pair chain
  long long nk;       // K*N
  long long dim;      // K*N*n*T1
  int TS = 0;         // stage stride of the device vectors (stages per node, >= T1)
  int T0 = 0;         // zero stages between a vector's 128-byte aligned allocation and v[0]
  long long span = 0; // doubles from a vector's first to one past its last entry
  int hx0 = -1, hx1 = -1;   // stage-slab halo stages: Delta leaves them unwritten (-1: none)
};

// Delta output rows a slab owns (every row outside stage-slab mode)
__host__ __device__ __forceinline__ bool slab_owned(const Geo& g, int t) {
  return t != g.hx0 && t != g.hx1;
}

struct Ops {
  const double* psi;   // [npc][N][K][13][n][n]   Psi_t(a, a+off13[o])
  const double* xi;    // [nxc][N][K][5][n][n]    Xi_t(a, a+off5[u])
  const double* xit;   // [nxc][N][K][5][n][n]    Xi_t(a+off5[u], a)^T
  const double* fac;   // [npc][V][nb][2][q][q]   {L_k^-1, C_k = M_{k,k-1} L_{k-1}^-T}
  const int* psi_cls;  // [T1]
  const int* xi_cls;   // [T]
};

// PCG scalars and control flags, device resident; the captured step graph reads
// everything that changes between runs from here.
struct PcgState {
  double mu, curv, alpha, beta, res, tol;
  double mu_prev;   // stage-slab mode: mu of the previous step while q.r is reduced
  long long step, max_steps;
  double* hist;
  int done, converged, breakdown;
  int defer;        // stage-slab mode: max|r| kernels record the history but leave the
                    // convergence decision to k_slab_conv_beta (after the global max)
  int skip;   // set by the first kernel of a step when the step budget is exhausted
  int nonfinite;   // set by the rhs check of gq_pcg_start
  unsigned int counter[4];
};

// kernels after the first one of a step stop on convergence, breakdown or budget
__device__ __forceinline__ bool halted(const PcgState* st) {
  return st != nullptr && (st->done || st->skip);
}

enum DotMode { kDotNone = 0, kDotInit = 1, kDotStep = 2 };

template <int NS>
struct Vec {
  double v[NS];
};

template <int NS>
__device__ __forceinline__ Vec<NS> vzero() {
  Vec<NS> r;
#pragma unroll
  for (int k = 0; k < NS; ++k) r.v[k] = 0.0;
  return r;
}

// read-only (non-coherent) vector load: only for data not written by the same launch
template <int NS>
__device__ __forceinline__ Vec<NS> ldv_nc(const double* __restrict__ p) {
  Vec<NS> r;
  if constexpr (NS % 2 == 0) {
#pragma unroll
    for (int k = 0; k < NS; k += 2) {
      double2 t = __ldg(reinterpret_cast<const double2*>(p + k));
      r.v[k] = t.x;
      r.v[k + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < NS; ++k) r.v[k] = __ldg(p + k);
  }
  return r;
}

template <int NS>
__device__ __forceinline__ Vec<NS> ldv(const double* p) {
  Vec<NS> r;
  if constexpr (NS % 2 == 0) {
#pragma unroll
    for (int k = 0; k < NS; k += 2) {
      double2 t = *reinterpret_cast<const double2*>(p + k);
      r.v[k] = t.x;
      r.v[k + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < NS; ++k) r.v[k] = p[k];
  }
  return r;
}

template <int NS>
__device__ __forceinline__ void stv(double* p, const Vec<NS>& x) {
  if constexpr (NS % 2 == 0) {
#pragma unroll
    for (int k = 0; k < NS; k += 2)
      *reinterpret_cast<double2*>(p + k) = make_double2(x.v[k], x.v[k + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < NS; ++k) p[k] = x.v[k];
  }
}

// acc += M x, M an NS x NS row-major block read through the read-only path
// (warp-uniform addresses -> one broadcast transaction per load)
template <int NS>
__device__ __forceinline__ void mac(Vec<NS>& acc, const double* __restrict__ M, const Vec<NS>& x) {
#pragma unroll
  for (int a = 0; a < NS; ++a) {
    double row[NS];
    if constexpr (NS % 2 == 0) {
#pragma unroll
      for (int b = 0; b < NS; b += 2) {
        double2 t = __ldg(reinterpret_cast<const double2*>(M + a * NS + b));
        row[b] = t.x;
        row[b + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int b = 0; b < NS; ++b) row[b] = __ldg(M + a * NS + b);
    }
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < NS; ++b) s = fma(row[b], x.v[b], s);
    acc.v[a] += s;
  }
}

template <int NS>
__device__ __forceinline__ Vec<NS> shfl_up(const Vec<NS>& x, int d) {
  Vec<NS> r;
#pragma unroll
  for (int k = 0; k < NS; ++k) r.v[k] = __shfl_up_sync(0xffffffffu, x.v[k], d);
  return r;
}
template <int NS>
__device__ __forceinline__ Vec<NS> shfl_down(const Vec<NS>& x, int d) {
  Vec<NS> r;
#pragma unroll
  for (int k = 0; k < NS; ++k) r.v[k] = __shfl_down_sync(0xffffffffu, x.v[k], d);
  return r;
}

// ---- deterministic reductions ---------------------------------------------------------
// xor-butterfly: every lane ends with the bitwise-same value (fp add is commutative)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// NaN-propagating max (np.max semantics)
__device__ __forceinline__ double nmax(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a > b ? a : b;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = nmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// block-wide reduction; result valid in every thread. blockDim.x multiple of 32, <= 1024
template <bool MAX>
__device__ double block_reduce(double v) {
  __shared__ double red[32];
  __syncthreads();
  v = MAX ? warp_max(v) : warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = (l < nw) ? red[l] : (MAX ? -1.0 : 0.0);
  r = MAX ? warp_max(r) : warp_sum(r);
  return r;
}

// Grid reduction, last-block-done pattern with partials summed in a fixed order, so
// results are bitwise reproducible for a fixed launch shape.  Returns true in the last
// block; `out` then holds the reduced value in every thread of that block.
template <bool MAX>
__device__ bool grid_reduce(double v, double* partials, unsigned int* counter, double& out) {
  __shared__ int is_last;
  v = block_reduce<MAX>(v);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = v;
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  double acc = MAX ? -1.0 : 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    double p = __ldcg(partials + b);
    acc = MAX ? nmax(acc, p) : acc + p;
  }
  out = block_reduce<MAX>(acc);
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

__device__ __forceinline__ long long vidx(const Geo& g, int j, int i, int t) {
  return (((long long)j * g.K + i) * g.TS + t) * g.n;
}

}  // namespace gq
