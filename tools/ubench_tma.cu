// TMA load throughput on B200 against box shape: every CTA streams 3-D boxes {b0 doubles,
// bR rows, bC columns} of a [C][R][D0] fp64 tensor (the stage-inner vector layout) through a
// ring of NS shared-memory slots (thread 0 issues, everyone waits on the slot's mbarrier, one
// __syncthreads hands the slot back).  Prints GB/s per shape.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tma tools/ubench_tma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tma3(unsigned d, const CUtensorMap* m, int a, int b, int c, unsigned bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               ::"r"(d), "l"((uint64_t)m), "r"(a), "r"(b), "r"(c), "r"(bar) : "memory");
}
__device__ __forceinline__ bool tryw(unsigned b, unsigned p) {
  unsigned ok;
  asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }"
               : "=r"(ok) : "r"(b), "r"(p) : "memory");
  return ok;
}

__global__ void stream(const __grid_constant__ CUtensorMap m, int nb0, int nbR, int nbC, int b0,
                       int bR, int bC, int ns, unsigned box_bytes, double* sink, int runs) {
  extern __shared__ unsigned char raw[];
  const unsigned base = (su(raw) + 1023u) & ~1023u;
  const unsigned slot_bytes = (box_bytes + 1023u) & ~1023u;
  const unsigned bars = base + ns * slot_bytes;
  if (threadIdx.x == 0)
    for (int s = 0; s < ns; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * s));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const long long total = (long long)nb0 * nbR * nbC;
  // my boxes: b = blockIdx.x + k * gridDim.x
  long long nmine = total > blockIdx.x ? (total - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // runs = 1: every CTA walks one contiguous run of the box sequence (stage axis fastest)
  const long long lo = total * blockIdx.x / gridDim.x, hi = total * (blockIdx.x + 1) / gridDim.x;
  if (runs) nmine = hi - lo;
  auto issue = [&](long long k) {
    if (threadIdx.x == 0 && k < nmine) {
      const long long b = runs ? lo + k : blockIdx.x + k * gridDim.x;
      const int c0 = (int)(b % nb0), r = (int)((b / nb0) % nbR), c = (int)(b / nb0 / nbR);
      const unsigned s = (unsigned)(k % ns);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bars + 8 * s), "r"(box_bytes) : "memory");
      tma3(base + s * slot_bytes, &m, c0 * b0, r * bR, c * bC, bars + 8 * s);
    }
  };
  for (int k = 0; k < ns - 1; ++k) issue(k);
  double acc = 0.0;
  for (long long k = 0; k < nmine; ++k) {
    const unsigned s = (unsigned)(k % ns);
    while (!tryw(bars + 8 * s, (unsigned)((k / ns) & 1))) {}
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + s * slot_bytes + 8 * (threadIdx.x % 64)));
    acc += v;
    __syncthreads();
    issue(k + ns - 1);
  }
  if (acc == 12345.678) sink[0] = acc;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                        CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int D0 = 416, R = 256, C = 1024;   // 4 x   // the headline vector: 2 T1 doubles x K x N
  double* x;
  cudaMalloc(&x, (size_t)D0 * R * C * 8);
  cudaMemset(x, 0, (size_t)D0 * R * C * 8);
  double* sink;
  cudaMalloc(&sink, 8);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = (Enc)p;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Shape { int b0, bR, bC, ns, per_sm, thr, runs; };
  const Shape shapes[] = {
      {8, 16, 8, 6, 2, 128, 1},  {16, 16, 8, 3, 2, 128, 1}, {16, 16, 8, 6, 2, 128, 1},
      {32, 16, 8, 3, 2, 128, 1}, {32, 16, 4, 6, 2, 128, 1}, {16, 16, 8, 3, 2, 128, 0},
      {32, 16, 8, 3, 2, 128, 0}, {16, 18, 10, 3, 2, 128, 1}, {16, 18, 10, 4, 2, 128, 1},
      {32, 18, 10, 2, 2, 128, 1},
  };


  for (const Shape& s : shapes) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {(cuuint64_t)D0, (cuuint64_t)R, (cuuint64_t)C};
    const cuuint64_t strides[2] = {(cuuint64_t)D0 * 8, (cuuint64_t)D0 * 8 * R};
    const cuuint32_t box[3] = {(cuuint32_t)s.b0, (cuuint32_t)s.bR, (cuuint32_t)s.bC};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUtensorMapSwizzle sw = s.b0 == 8 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : s.b0 == 16 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : s.b0 == 4 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d for b0=%d\n", (int)r, s.b0); continue; }
    const unsigned bytes = (unsigned)s.b0 * 8 * s.bR * s.bC;
    const unsigned slot = (bytes + 1023) & ~1023u;
    const size_t smem = 1024 + (size_t)s.ns * slot + 8 * s.ns;
    const int nb0 = (D0 + s.b0 - 1) / s.b0, nbR = (R + s.bR - 1) / s.bR, nbC = (C + s.bC - 1) / s.bC;
    const int grid = sms * s.per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
      cudaEventRecord(e0);
      stream<<<grid, s.thr, smem>>>(m, nb0, nbR, nbC, s.b0, s.bR, s.bC, s.ns, bytes, sink, s.runs);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0 && ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    const double moved = (double)nb0 * nbR * nbC * bytes;
    printf("%s box {%2d dbl = %3d B rows, %2d x %2d} ns %2d per_sm %d thr %3d smem %6zu: %7.1f GB/s (%.3f ms) %s\n",
           s.runs ? "runs" : "intl", s.b0, s.b0 * 8, s.bR, s.bC, s.ns, s.per_sm, s.thr, smem, moved / best / 1e6, best,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  return 0;
}
