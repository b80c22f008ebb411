// TMA box semantics probe for the CTA chain kernel's access pattern: every CTA walks blocks k,
// loads the tau / theta boxes through a ring of R slots (full/empty mbarriers, 5 consumer
// warps, warp 0 lane 0 producer) and every consumer lane compares the staged values it reads
// with a direct global load.  Reports mismatches.  nvcc -arch=sm_100a -o tma_probe tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstdint>

#define CW 5
#define PITCH 84
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void expect(uint64_t* b, unsigned n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ bool tryw(uint64_t* b, unsigned p) {
  unsigned ok; asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }" : "=r"(ok) : "r"(su(b)), "r"(p) : "memory"); return ok; }
__device__ __forceinline__ void waitb(uint64_t* b, unsigned p) { while (!tryw(b, p)) {} }
__device__ __forceinline__ void tma3(void* d, const CUtensorMap* m, int a, int b, int c, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
    ::"r"(su(d)), "l"((uint64_t)m), "r"(a), "r"(b), "r"(c), "r"(su(bar)) : "memory"); }
struct Maps { CUtensorMap t22, t41, t21; };

template <int R>
__global__ void __launch_bounds__(160) probe(const __grid_constant__ Maps mp, const double* x, int K, int N, int T1, int nb, int nch, unsigned long long* bad, int mode) {
  extern __shared__ unsigned char raw[];
  double* ring = (double*)(((uintptr_t)raw + 127) & ~(uintptr_t)127);
  const int SLOT = 1840;
  uint64_t* full = (uint64_t*)(ring + R * SLOT); uint64_t* empty = full + R;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, rw = lane >> 2, qd = lane & 3;
  if (threadIdx.x == 0) { for (int i = 0; i < R; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, CW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
  __syncthreads();
  int item = blockIdx.x, v = item / nch, c = item % nch, t0 = 1 + 40 * c, col = 2 * v;
  long long rs = (long long)T1 * 2, cs = (long long)K * rs;
  unsigned si = 0, su_ = 0;
  auto issue = [&](int k) {
    unsigned s = si++; int slot = s % R;
    if (s >= R) waitb(empty + slot, ((s / R) - 1) & 1);
    double* sl = ring + slot * SLOT;
    expect(full + slot, 16 * 672);
    tma3(sl, &mp.t22, 2 * t0, 2 * k, col, full + slot);
    tma3(sl + 4 * PITCH, &mp.t41, 2 * t0, 2 * k - 1, col - 1, full + slot);
    tma3(sl + 8 * PITCH, &mp.t41, 2 * t0, 2 * k - 1, col + 2, full + slot);
    tma3(sl + 12 * PITCH, &mp.t21, 2 * t0, 2 * k, col - 2, full + slot);
    tma3(sl + 16 * PITCH, &mp.t21, 2 * t0, 2 * k, col + 3, full + slot);
  };
  // record r -> (dcol, drow)
  auto dcol = [](int r) { return r < 4 ? (r >> 1) : r < 8 ? -1 : r < 12 ? 2 : r < 14 ? -2 : 3; };
  auto drow = [](int r) { return r < 4 ? (r & 1) : r < 8 ? r - 5 : r < 12 ? r - 9 : r < 14 ? r - 12 : r - 16; };
  const int P = R - 1;
  if (threadIdx.x == 0) for (int k = 0; k < P && k < nb; ++k) issue(k);
  unsigned long long nbad = 0;
  for (int k = 0; k < nb; ++k) {
    if (threadIdx.x == 0 && k + P < nb) issue(k + P);
    __syncwarp();
    unsigned s = su_++; int slot = s % R;
    waitb(full + slot, (s / R) & 1);
    __syncwarp();
    const double* sl = ring + slot * SLOT;
    // every lane checks its stage rw of every used record, both components
    for (int r = 0; r < 18; ++r) {
      if (r == 14 || r == 15) continue;
      int cc = col + dcol(r), rr = 2 * k + drow(r), t = t0 + 8 * warp + rw;
      double2 got = *(const double2*)(sl + r * PITCH + 2 * (8 * warp + rw));
      double2 want = make_double2(0, 0);
      if (cc >= 0 && cc < N && rr >= 0 && rr < K && t < T1) want = *(const double2*)(x + cc * cs + rr * rs + 2 * t);
      if (qd == 0 && (got.x != want.x || got.y != want.y)) ++nbad;
    }
    if (mode & 1) for (int i = 0; i < 2000; ++i) asm volatile("nanosleep.u32 1;");
    __syncwarp();
    if (lane == 0) arrive(empty + slot);
  }
  if (nbad) atomicAdd(bad, nbad);
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int K = 256, N = 256, T = 200;
  if (argc > 3) { K = atoi(argv[1]); N = atoi(argv[2]); T = atoi(argv[3]); }
  int T1 = T + 1, nb = K / 2, nch = (T + 39) / 40, V = N / 2;
  size_t dim = (size_t)K * N * T1 * 2;
  std::vector<double> h(dim); for (size_t i = 0; i < dim; ++i) h[i] = (double)(i % 100003) + 0.25;
  double* x; cudaMalloc(&x, dim * 8); cudaMemcpy(x, h.data(), dim * 8, cudaMemcpyHostToDevice);
  unsigned long long* bad; cudaMalloc(&bad, 8);
  void* fp; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  Maps mp;
  cuuint64_t dims[3] = {(cuuint64_t)T1 * 2, (cuuint64_t)K, (cuuint64_t)N}, st[2] = {(cuuint64_t)T1 * 16, (cuuint64_t)T1 * 16 * K};
  cuuint32_t es[3] = {1, 1, 1};
  cuuint32_t b22[3] = {PITCH, 2, 2}, b41[3] = {PITCH, 4, 1}, b21[3] = {PITCH, 2, 1};
  printf("enc %d %d %d\n", enc(&mp.t22, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims, st, b22, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
    enc(&mp.t41, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims, st, b41, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
    enc(&mp.t21, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims, st, b21, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  for (int R = 2; R <= 4; ++R) for (int mode = 0; mode < 2; ++mode) {
    size_t smem = R * 1840 * 8 + 2 * R * 8 + 128;
    cudaMemset(bad, 0, 8);
    if (R == 2) { cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); probe<2><<<V * nch, 160, smem>>>(mp, x, K, N, T1, nb, nch, bad, mode); }
    if (R == 3) { cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); probe<3><<<V * nch, 160, smem>>>(mp, x, K, N, T1, nb, nch, bad, mode); }
    if (R == 4) { cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); probe<4><<<V * nch, 160, smem>>>(mp, x, K, N, T1, nb, nch, bad, mode); }
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long hb; cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
    printf("R=%d mode=%d err=%s bad=%llu\n", R, mode, cudaGetErrorString(e), hb);
  }
  return 0;
}
