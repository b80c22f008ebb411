// Reduced right-hand side omega~ on the device (kkt_assembly.py:275-301): the initial states
// at stage 0, and at stage t+1 the boundary terms sum_d C_d(t) sigma_d(t) of the edge nodes
// whose coupling toward an off-grid neighbour d has both blocks and a declared trajectory.
// One thread per (stage, node); the directions are added in the reference's order (north,
// south, west, east), so every entry is one fixed sequence of fused multiply-adds.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "gridlq_b200.h"

namespace gq {
int api_fail(int code, const std::string& msg);
}

namespace {

// direction order of the arrays: west, east, north, south (problem.py DIRECTIONS)
__global__ void k_offset(int K, int N, int T, int n, int L, int ncls,
                         const double* __restrict__ init, const double* __restrict__ blocks,
                         const int32_t* __restrict__ cls, const double* __restrict__ traj,
                         double* __restrict__ out) {
  const long long nk = (long long)K * N;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nk * (T + 1)) return;
  const int t1 = (int)(idx / nk);                 // output stage
  const long long node = idx - (long long)t1 * nk;   // j * K + i
  const int j = (int)(node / K), i = (int)(node - (long long)j * K);
  double* o = out + ((long long)t1 * nk + node) * n;
  if (t1 == 0) {
    for (int k = 0; k < n; ++k) o[k] = init[node * n + k];
    return;
  }
  const int t = t1 - 1;
  double acc[8];
  for (int k = 0; k < n; ++k) acc[k] = 0.0;
  // reference order: north (i == 0), south (i == K-1), west (j == 0), east (j == N-1)
  const int dir[4] = {2, 3, 0, 1};
  const bool edge[4] = {i == 0, i == K - 1, j == 0, j == N - 1};
  const int eidx[4] = {j, j, i, i};
  for (int q = 0; q < 4; ++q) {
    if (!edge[q]) continue;
    const long long de = (long long)dir[q] * L + eidx[q];
    const int c = cls[de * T + t];
    if (c < 0) continue;
    const double* Cb = blocks + (de * ncls + c) * n * n;
    const double* sg = traj + (de * T + t) * n;
    for (int k = 0; k < n; ++k) {
      double s = 0.0;
      for (int e = 0; e < n; ++e) s = fma(Cb[k * n + e], sg[e], s);
      acc[k] += s;
    }
  }
  for (int k = 0; k < n; ++k) o[k] = acc[k];
}

}  // namespace

extern "C" int gq_build_offset(int32_t K, int32_t N, int32_t T, int32_t n, int32_t ncls,
                               const double* init, const double* blocks, const int32_t* cls,
                               const double* traj, double* out, void* stream) {
  if (K < 1 || N < 1 || T < 1 || n < 1 || n > 8 || ncls < 1 || !init || !out)
    return gq::api_fail(GQ_INVALID_ARG, "gq_build_offset: bad sizes or null init/out");
  if (!blocks || !cls || !traj)
    return gq::api_fail(GQ_INVALID_ARG, "gq_build_offset: null boundary arrays");
  const int L = K > N ? K : N;
  const long long total = (long long)K * N * (T + 1);
  k_offset<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      K, N, T, n, L, ncls, init, blocks, cls, traj, out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return gq::api_fail(GQ_CUDA_ERROR, std::string("gq_build_offset: ") + cudaGetErrorString(e));
  return GQ_OK;
}
