// Stage-slab mode kernels (host logic in gq_api.cu and slab.py).
//
// A slab context holds the stage window [a, b) of the global problem: its owned stages
// [own_lo, own_hi) plus one halo stage on each side that has a neighbour.  The step kernels
// run unchanged on the whole window; these kernels make the slab's scalars owned-only and
// turn the slab-local decisions of the step kernels into global ones once the host has
// reduced the partial scalars over all slabs (pcg.py:100-131):
//
// Delta itself leaves the halo rows of y unwritten in stage-slab mode (Geo::hx0/hx1); they
// are zeroed once at the start (k_stage_zero), so y.d covers the owned stages only and r --
// with it max|r| and q.r -- stays zero on the halo stages for the whole solve.
//   k_slab_alpha      after the curvature sum: breakdown test and alpha = mu / c
//   k_slab_savemu     before the sweep that forms q.r: keep mu
//   k_slab_conv_beta  after ONE reduction of (max|r|, q.r): history entry, convergence test
//                     and beta = mu' / mu.  The max|r| kernels run with PcgState::defer, so
//                     no slab stops on its own partial; a converged step computes q for
//                     nothing, which changes no result.
//   k_stage_pack / k_stage_unpack  one stage of a stage-inner vector <-> a contiguous halo
//                  buffer in (column, row, state) order
#include <algorithm>

#include "gq_internal.h"

namespace gq {

__global__ void k_slab_alpha(PcgState* st) {
  if (st->skip) return;
  const double c = st->curv;                // pcg.py:101-108, now the global curvature
  if (c <= 0.0) {
    st->breakdown = 1;
    st->done = 1;
  } else {
    st->breakdown = 0;
    st->done = 0;
    st->alpha = st->mu / c;
  }
}

__global__ void k_slab_savemu(PcgState* st) {
  if (halted(st)) return;
  st->mu_prev = st->mu;
}

// after the fused max|r| / q.r reduction: history entry and convergence test
// (pcg.py:113-121), then beta = mu' / mu (pcg.py:127-131) unless the step converged
__global__ void k_slab_conv_beta(PcgState* st) {
  if (st->skip || st->breakdown) return;
  const double res = st->res;               // the global max|r|
  st->hist[st->step - 1] = res;
  if (res < st->tol) {
    st->converged = 1;
    st->done = 1;
    return;
  }
  // safeguard: a kernel that decided on a slab-local max|r| (one missing the PcgState::defer
  // check) must not stop this slab while the global residual is still above tol
  st->converged = 0;
  st->done = 0;
  st->beta = st->mu / st->mu_prev;          // the global q.r
}

__global__ void __launch_bounds__(256) k_stage_pack(Geo g, int t, const double* __restrict__ v,
                                                    double* __restrict__ buf) {
  const long long per = g.nk * g.n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < per;
       e += (long long)gridDim.x * blockDim.x) {
    const long long node = e / g.n;
    buf[e] = v[(node * g.TS + t) * g.n + (e - node * g.n)];
  }
}

__global__ void __launch_bounds__(256) k_stage_zero(Geo g, int t, double* __restrict__ v) {
  const long long per = g.nk * g.n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < per;
       e += (long long)gridDim.x * blockDim.x) {
    const long long node = e / g.n;
    v[(node * g.TS + t) * g.n + (e - node * g.n)] = 0.0;
  }
}

__global__ void __launch_bounds__(256) k_stage_unpack(Geo g, int t, const double* __restrict__ buf,
                                                      double* __restrict__ v) {
  const long long per = g.nk * g.n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < per;
       e += (long long)gridDim.x * blockDim.x) {
    const long long node = e / g.n;
    v[(node * g.TS + t) * g.n + (e - node * g.n)] = buf[e];
  }
}

static unsigned stage_blocks(const Geo& g, int sm_count) {
  const long long per = g.nk * g.n;
  return (unsigned)std::max(1LL, std::min<long long>((per + 255) / 256, 4LL * sm_count));
}

cudaError_t launch_slab_scalar(int which, PcgState* st, cudaStream_t s) {
  switch (which) {
    case 0: k_slab_alpha<<<1, 1, 0, s>>>(st); break;
    case 2: k_slab_savemu<<<1, 1, 0, s>>>(st); break;
    default: k_slab_conv_beta<<<1, 1, 0, s>>>(st); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_stage_pack(const Geo& g, int t, const double* v, double* buf, int sm_count,
                              cudaStream_t s) {
  k_stage_pack<<<stage_blocks(g, sm_count), 256, 0, s>>>(g, t, v, buf);
  return cudaGetLastError();
}

cudaError_t launch_stage_zero(const Geo& g, int t, double* v, int sm_count, cudaStream_t s) {
  k_stage_zero<<<stage_blocks(g, sm_count), 256, 0, s>>>(g, t, v);
  return cudaGetLastError();
}

cudaError_t launch_stage_unpack(const Geo& g, int t, const double* buf, double* v, int sm_count,
                                cudaStream_t s) {
  k_stage_unpack<<<stage_blocks(g, sm_count), 256, 0, s>>>(g, t, buf, v);
  return cudaGetLastError();
}

}  // namespace gq
