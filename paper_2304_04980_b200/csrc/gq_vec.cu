// CG vector updates with fused reductions, plus the boundary layout transposes.
//
// Reference: pcg_solve loop body (gridlq/pcg.py:98-131).  The element-wise updates use
// explicitly rounded multiply and add (no FMA contraction) so that, given identical
// inputs, they reproduce numpy's `x += alpha*d`, `r - alpha*y`, `q + beta*d` bit for bit.
// Reductions are grid-wide with a fixed partial order (bitwise reproducible run to run).
#include <algorithm>
#include "gq_internal.h"

namespace gq {

int vec_blocks(int sm_count) { return sm_count * 8; }

// Streaming kernels: each thread keeps kVU independent 16-byte loads per operand in flight
// (a 210 MB vector pass is pure HBM bandwidth), 8 x 256-thread blocks per SM.
constexpr int kVU = 4;

__device__ __forceinline__ double2 ld_stream(const double* p) {
  return __ldcs(reinterpret_cast<const double2*>(p));
}

__global__ void __launch_bounds__(256) k_update(long long dim, double* __restrict__ x,
                                                double* __restrict__ r,
                                                const double* __restrict__ d,
                                                const double* __restrict__ y, double* partials,
                                                PcgState* st) {
  if (halted(st)) return;
  const double alpha = st->alpha;
  double m = 0.0;
  const long long n2 = dim >> 1;
  const long long nth = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long b = tid; b < n2; b += nth * kVU) {
    double2 xv[kVU], rv[kVU], dv[kVU], yv[kVU];
#pragma unroll
    for (int u = 0; u < kVU; ++u) {
      const long long e = 2 * (b + u * nth);
      if (b + u * nth < n2) {
        dv[u] = ld_stream(d + e);
        yv[u] = ld_stream(y + e);
        xv[u] = *reinterpret_cast<const double2*>(x + e);
        rv[u] = *reinterpret_cast<const double2*>(r + e);
      }
    }
#pragma unroll
    for (int u = 0; u < kVU; ++u) {
      const long long e = 2 * (b + u * nth);
      if (b + u * nth < n2) {
        xv[u].x = __dadd_rn(xv[u].x, __dmul_rn(alpha, dv[u].x));    // pcg.py:109
        xv[u].y = __dadd_rn(xv[u].y, __dmul_rn(alpha, dv[u].y));
        rv[u].x = __dsub_rn(rv[u].x, __dmul_rn(alpha, yv[u].x));    // pcg.py:111
        rv[u].y = __dsub_rn(rv[u].y, __dmul_rn(alpha, yv[u].y));
        __stcs(reinterpret_cast<double2*>(x + e), xv[u]);
        *reinterpret_cast<double2*>(r + e) = rv[u];
        m = nmax(m, nmax(fabs(rv[u].x), fabs(rv[u].y)));           // pcg.py:113
      }
    }
  }
  if ((dim & 1) && tid == 0) {
    const long long e = dim - 1;
    x[e] = __dadd_rn(x[e], __dmul_rn(alpha, d[e]));
    const double rn = __dsub_rn(r[e], __dmul_rn(alpha, y[e]));
    r[e] = rn;
    m = nmax(m, fabs(rn));
  }
  double res;
  if (grid_reduce<true>(m, partials, &st->counter[1], res) && threadIdx.x == 0) {
    st->res = res;
    st->hist[st->step] = res;
    st->step += 1;
    if (res < st->tol && !st->defer) {            // pcg.py:119-121
      st->converged = 1;
      st->done = 1;
    }
  }
}

// r = r - alpha y and ||r||_inf only (the x update runs on a parallel graph branch)
__global__ void __launch_bounds__(256) k_update_r(long long dim, double* __restrict__ r,
                                                  const double* __restrict__ y, double* partials,
                                                  PcgState* st) {
  if (halted(st)) return;
  const double alpha = st->alpha;
  double m = 0.0;
  const long long n2 = dim >> 1;
  const long long nth = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long b = tid; b < n2; b += nth * kVU) {
    double2 rv[kVU], yv[kVU];
#pragma unroll
    for (int u = 0; u < kVU; ++u) {
      const long long e = 2 * (b + u * nth);
      if (b + u * nth < n2) {
        yv[u] = ld_stream(y + e);
        rv[u] = *reinterpret_cast<const double2*>(r + e);
      }
    }
#pragma unroll
    for (int u = 0; u < kVU; ++u) {
      const long long e = 2 * (b + u * nth);
      if (b + u * nth < n2) {
        rv[u].x = __dsub_rn(rv[u].x, __dmul_rn(alpha, yv[u].x));    // pcg.py:111
        rv[u].y = __dsub_rn(rv[u].y, __dmul_rn(alpha, yv[u].y));
        *reinterpret_cast<double2*>(r + e) = rv[u];
        m = nmax(m, nmax(fabs(rv[u].x), fabs(rv[u].y)));           // pcg.py:113
      }
    }
  }
  if ((dim & 1) && tid == 0) {
    const long long e = dim - 1;
    const double rn = __dsub_rn(r[e], __dmul_rn(alpha, y[e]));
    r[e] = rn;
    m = nmax(m, fabs(rn));
  }
  double res;
  if (grid_reduce<true>(m, partials, &st->counter[1], res) && threadIdx.x == 0) {
    st->res = res;
    st->hist[st->step] = res;
    st->step += 1;
    if (res < st->tol && !st->defer) {            // pcg.py:119-121
      st->converged = 1;
      st->done = 1;
    }
  }
}

// x = x + alpha d (pcg.py:109).  Runs concurrently with the r update and the sweeps of the
// same step, so it must not look at `done` (the r update may set it for this very step,
// whose x update still belongs to the result); `skip` (set by the step's first kernel) and
// `breakdown` (set by the curvature reduction before alpha) are the only stops.
__global__ void __launch_bounds__(256) k_update_x(long long dim, double* __restrict__ x,
                                                  const double* __restrict__ d, PcgState* st) {
  if (st->skip || st->breakdown) return;
  const double alpha = st->alpha;
  const long long n2 = dim >> 1;
  const long long nth = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long b = tid; b < n2; b += nth * kVU) {
    double2 xv[kVU], dv[kVU];
#pragma unroll
    for (int u = 0; u < kVU; ++u) {
      const long long e = 2 * (b + u * nth);
      if (b + u * nth < n2) {
        dv[u] = ld_stream(d + e);
        xv[u] = ld_stream(x + e);
      }
    }
#pragma unroll
    for (int u = 0; u < kVU; ++u) {
      const long long e = 2 * (b + u * nth);
      if (b + u * nth < n2) {
        xv[u].x = __dadd_rn(xv[u].x, __dmul_rn(alpha, dv[u].x));
        xv[u].y = __dadd_rn(xv[u].y, __dmul_rn(alpha, dv[u].y));
        __stcs(reinterpret_cast<double2*>(x + e), xv[u]);
      }
    }
  }
  if ((dim & 1) && tid == 0) x[dim - 1] = __dadd_rn(x[dim - 1], __dmul_rn(alpha, d[dim - 1]));
}

__global__ void __launch_bounds__(256) k_dirupdate(long long dim, double* __restrict__ d,
                                                   const double* __restrict__ q, PcgState* st) {
  if (halted(st)) return;
  const double beta = st->beta;
  const long long n2 = dim >> 1;
  const long long nth = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long b = tid; b < n2; b += nth * kVU) {
    double2 dv[kVU], qv[kVU];
#pragma unroll
    for (int u = 0; u < kVU; ++u) {
      const long long e = 2 * (b + u * nth);
      if (b + u * nth < n2) {
        qv[u] = ld_stream(q + e);
        dv[u] = *reinterpret_cast<const double2*>(d + e);
      }
    }
#pragma unroll
    for (int u = 0; u < kVU; ++u) {
      const long long e = 2 * (b + u * nth);
      if (b + u * nth < n2) {
        dv[u].x = __dadd_rn(qv[u].x, __dmul_rn(beta, dv[u].x));    // pcg.py:129
        dv[u].y = __dadd_rn(qv[u].y, __dmul_rn(beta, dv[u].y));
        *reinterpret_cast<double2*>(d + e) = dv[u];
      }
    }
  }
  if ((dim & 1) && tid == 0) d[dim - 1] = __dadd_rn(q[dim - 1], __dmul_rn(beta, d[dim - 1]));
}

// d = q + beta d (pcg.py:129) fused with the iterate update x += alpha d_old (pcg.py:109) of
// the same step: one pass reads q, d, x and writes d, x.  Runs unless the step was skipped
// (budget) or broke down; after convergence (done) only x is updated, as the reference
// updates x in the step that converges and stops before the direction update.
__global__ void __launch_bounds__(256) k_dirupdate_x(long long dim, double* __restrict__ d,
                                                     const double* __restrict__ q,
                                                     double* __restrict__ x, PcgState* st) {
  if (st->skip || st->breakdown) return;
  const double alpha = st->alpha, beta = st->beta;
  const bool dir = !st->done;
  const long long n2 = dim >> 1;
  const long long nth = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // one 16-byte element per thread and pass over a large grid: five streams (3 reads, 2
  // writes) at 6.4 TB/s on B200; four elements per thread a grid apart ran at 5.1 TB/s
  for (long long b = tid; b < n2; b += nth) {
    const long long e = 2 * b;
    double2 dv = *reinterpret_cast<const double2*>(d + e);
    double2 xv = ld_stream(x + e);
    xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, dv.x));
    xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, dv.y));
    __stcs(reinterpret_cast<double2*>(x + e), xv);
    if (dir) {
      const double2 qv = ld_stream(q + e);
      dv.x = __dadd_rn(qv.x, __dmul_rn(beta, dv.x));
      dv.y = __dadd_rn(qv.y, __dmul_rn(beta, dv.y));
      *reinterpret_cast<double2*>(d + e) = dv;
    }
  }
  if ((dim & 1) && tid == 0) {
    const long long e = dim - 1;
    const double dold = d[e];
    x[e] = __dadd_rn(x[e], __dmul_rn(alpha, dold));
    if (dir) d[e] = __dadd_rn(q[e], __dmul_rn(beta, dold));
  }
}

// max |a - b| (b may be null: max |a|), the successive-iterate test of the standalone nested
// Jacobi iteration (nested_jacobi.py:145); result in *out, reduced in a fixed order
__global__ void __launch_bounds__(256) k_maxdiff(long long dim, const double* __restrict__ a,
                                                 const double* __restrict__ b, double* partials,
                                                 unsigned int* counter, double* out) {
  double m = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < dim; e += stride)
    m = nmax(m, fabs(b ? a[e] - b[e] : a[e]));
  double res;
  if (grid_reduce<true>(m, partials, counter, res) && threadIdx.x == 0) *out = res;
}

// out = a + b
__global__ void __launch_bounds__(256) k_add(long long dim, double* __restrict__ out,
                                             const double* __restrict__ a,
                                             const double* __restrict__ b) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < dim; e += stride)
    out[e] = a[e] + b[e];
}

__global__ void __launch_bounds__(256) k_dot(long long dim, const double* __restrict__ a,
                                             const double* __restrict__ b, double* partials,
                                             PcgState* st, int dotmode) {
  if (halted(st)) return;
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < dim; e += stride)
    s = fma(a[e], b[e], s);
  double mu;
  if (grid_reduce<false>(s, partials, &st->counter[3], mu) && threadIdx.x == 0) {
    if (dotmode == kDotInit) {
      st->mu = mu;
    } else {
      st->beta = mu / st->mu;
      st->mu = mu;
    }
  }
}

__global__ void __launch_bounds__(256) k_sub(long long dim, double* __restrict__ out,
                                             const double* __restrict__ a,
                                             const double* __restrict__ b) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < dim; e += stride)
    out[e] = __dsub_rn(a[e], b[e]);
}

cudaError_t launch_update(const Geo& g, double* x, double* r, const double* d, const double* y,
                          int blocks, double* partials, PcgState* st, cudaStream_t s) {
  const long long fp = (long long)g.T0 * g.n;
  k_update<<<blocks, 256, 0, s>>>(g.span + fp, x - fp, r - fp, d - fp, y - fp, partials, st);
  return cudaGetLastError();
}

// any non-finite entry -> st->nonfinite = 1 (pcg.py:65-66 check, done on the device so the
// host never scans the 210 MB right-hand side)
__global__ void __launch_bounds__(256) k_nonfinite(long long dim, const double* __restrict__ v,
                                                   PcgState* st) {
  bool bad = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < dim; e += stride)
    bad |= !isfinite(v[e]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) st->nonfinite = 1;
}

cudaError_t launch_nonfinite(const Geo& g, const double* v, int blocks, PcgState* st,
                             cudaStream_t s) {
  const long long fp = (long long)g.T0 * g.n;
  k_nonfinite<<<blocks, 256, 0, s>>>(g.span + fp, v - fp, st);
  return cudaGetLastError();
}

cudaError_t launch_update_r(const Geo& g, double* r, const double* y, int blocks,
                            double* partials, PcgState* st, cudaStream_t s) {
  const long long fp = (long long)g.T0 * g.n;
  k_update_r<<<blocks, 256, 0, s>>>(g.span + fp, r - fp, y - fp, partials, st);
  return cudaGetLastError();
}

cudaError_t launch_update_x(const Geo& g, double* x, const double* d, int blocks, PcgState* st,
                            cudaStream_t s) {
  const long long fp = (long long)g.T0 * g.n;
  k_update_x<<<blocks, 256, 0, s>>>(g.span + fp, x - fp, d - fp, st);
  return cudaGetLastError();
}

cudaError_t launch_dirupdate(const Geo& g, double* d, const double* q, int blocks, PcgState* st,
                             cudaStream_t s) {
  const long long fp = (long long)g.T0 * g.n;
  k_dirupdate<<<blocks, 256, 0, s>>>(g.span + fp, d - fp, q - fp, st);
  return cudaGetLastError();
}

cudaError_t launch_dirupdate_x(const Geo& g, double* d, const double* q, double* x, int blocks,
                               PcgState* st, cudaStream_t s) {
  const long long fp = (long long)g.T0 * g.n;
  const long long n2 = (g.span + fp) >> 1;
  // `blocks` is the streaming kernels' 8 per SM: up to 64 per SM here, one pass for small sizes
  const long long want = std::max<long long>(1, std::min<long long>((n2 + 255) / 256, 8LL * blocks));
  k_dirupdate_x<<<(unsigned)want, 256, 0, s>>>(g.span + fp, d - fp, q - fp, x - fp, st);
  return cudaGetLastError();
}

cudaError_t launch_maxdiff(const Geo& g, const double* a, const double* b, int blocks,
                          double* partials, unsigned int* counter, double* out, cudaStream_t s) {
  const long long fp = (long long)g.T0 * g.n;
  k_maxdiff<<<blocks, 256, 0, s>>>(g.span + fp, a - fp, b ? b - fp : nullptr, partials, counter, out);
  return cudaGetLastError();
}

cudaError_t launch_add(const Geo& g, double* out, const double* a, const double* b, int blocks,
                       cudaStream_t s) {
  const long long fp = (long long)g.T0 * g.n;
  k_add<<<blocks, 256, 0, s>>>(g.span + fp, out - fp, a - fp, b - fp);
  return cudaGetLastError();
}

cudaError_t launch_dot(const Geo& g, const double* a, const double* b, int blocks,
                       double* partials, PcgState* st, int dotmode, cudaStream_t s) {
  const long long fp = (long long)g.T0 * g.n;
  k_dot<<<blocks, 256, 0, s>>>(g.span + fp, a - fp, b - fp, partials, st, dotmode);
  return cudaGetLastError();
}

cudaError_t launch_sub(const Geo& g, double* out, const double* a, const double* b, int blocks,
                       cudaStream_t s) {
  const long long fp = (long long)g.T0 * g.n;
  k_sub<<<blocks, 256, 0, s>>>(g.span + fp, out - fp, a - fp, b - fp);
  return cudaGetLastError();
}

// ---- layout transposes ------------------------------------------------------------------
// reference order (t, node, k) <-> stage-inner order (node, t, k); a tile is TS stages x
// TN nodes of n-double records staged through shared memory so both sides are coalesced.
constexpr int kTS = 32;

template <bool TO_INTERNAL>
__global__ void __launch_bounds__(256) k_transpose(Geo g, int tn, const double* __restrict__ src,
                                                   double* __restrict__ dst) {
  extern __shared__ double tile[];   // [kTS][tn][n]
  const int n = g.n;
  const long long nodes = g.nk;
  const int t0 = blockIdx.y * kTS;
  const long long nd0 = (long long)blockIdx.x * tn;
  const int rec = tn * n;            // doubles per stage row of the tile
  const int total = kTS * rec;
  if (TO_INTERNAL) {
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int ts = e / rec, w = e % rec;
      const int t = t0 + ts;
      const long long nd = nd0 + w / n;
      if (t < g.T1 && nd < nodes) tile[e] = src[(long long)t * nodes * n + nd0 * n + w];
    }
    __syncthreads();
    const int rec2 = kTS * n;        // doubles per node row of the output
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int nl = e / rec2, w = e % rec2;
      const int ts = w / n, k = w % n;
      const long long nd = nd0 + nl;
      const int t = t0 + ts;
      if (t < g.T1 && nd < nodes) dst[(nd * g.TS + t) * n + k] = tile[ts * rec + nl * n + k];
    }
  } else {
    const int rec2 = kTS * n;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int nl = e / rec2, w = e % rec2;
      const int ts = w / n, k = w % n;
      const long long nd = nd0 + nl;
      const int t = t0 + ts;
      if (t < g.T1 && nd < nodes) tile[ts * rec + nl * n + k] = src[(nd * g.TS + t) * n + k];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int ts = e / rec, w = e % rec;
      const int t = t0 + ts;
      const long long nd = nd0 + w / n;
      if (t < g.T1 && nd < nodes) dst[(long long)t * nodes * n + nd0 * n + w] = tile[e];
    }
  }
}

static cudaError_t launch_transpose(const Geo& g, bool to_internal, const double* src,
                                    double* dst, cudaStream_t s) {
  const int tn = g.n <= 2 ? 32 : (g.n <= 4 ? 16 : 8);
  dim3 grid((unsigned)((g.nk + tn - 1) / tn), (unsigned)((g.T1 + kTS - 1) / kTS));
  const size_t smem = (size_t)kTS * tn * g.n * sizeof(double);
  if (to_internal)
    k_transpose<true><<<grid, 256, smem, s>>>(g, tn, src, dst);
  else
    k_transpose<false><<<grid, 256, smem, s>>>(g, tn, src, dst);
  return cudaGetLastError();
}

cudaError_t launch_to_internal(const Geo& g, const double* ref, double* dev, cudaStream_t s) {
  return launch_transpose(g, true, ref, dev, s);
}

cudaError_t launch_to_reference(const Geo& g, const double* dev, double* ref, cudaStream_t s) {
  return launch_transpose(g, false, dev, ref, s);
}

}  // namespace gq
