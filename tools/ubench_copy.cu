// Streaming global->shared throughput per staging mechanism (B200).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// each warp streams its own contiguous region through a 4-stage smem ring
template <int MODE>
__global__ void stream(const double* __restrict__ src, long long n_per_warp, double* out, int chunk_bytes) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + w;
  const double* base = src + gw * n_per_warp;
  double* ring = sm + (size_t)w * 4 * 512;   // 4 x 4 KB per warp
  __shared__ uint64_t bars[32][4];
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (MODE == 3 && lane == 0)
    for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[w][s])));
  __syncwarp();
  double acc = 0;
  const int per = chunk_bytes / 8;            // doubles per chunk
  const long long nch = n_per_warp / per;
  for (long long c = 0; c < nch; ++c) {
    const double* s = base + c * per;
    double* d = ring + (c & 3) * 512;
    if (MODE == 0) {          // plain LDG.128 into registers
      for (int o = 2 * lane; o < per; o += 64) {
        double2 v = *reinterpret_cast<const double2*>(s + o);
        acc += v.x + v.y;
      }
    } else if (MODE == 1 || MODE == 2) {   // LDGSTS 16B/lane (1: no hint, 2: hint)
      for (int o = 2 * lane; o < per; o += 64) {
        if (MODE == 1)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(d + o)), "l"(s + o));
        else
          asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, 16, %2;" ::"r"(su32(d + o)), "l"(s + o), "l"(pol));
      }
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group 3;");
      __syncwarp();
      acc += d[lane];
    } else {                  // TMA bulk copy of one chunk, lane 0
      uint64_t* bar = &bars[w][c & 3];
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(chunk_bytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(chunk_bytes), "r"(su32(bar)));
      }
      if (c >= 3) {   // consume chunk c-3
        uint64_t* bw = &bars[w][(c - 3) & 3];
        const unsigned par = ((c - 3) >> 2) & 1;
        asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" ::"r"(su32(bw)), "r"(par));
        acc += ring[((c - 3) & 3) * 512 + lane];
      }
      __syncwarp();
    }
  }
  if (MODE == 3) {
    for (long long c = nch - 3 > 0 ? nch - 3 : 0; c < nch; ++c) {
      uint64_t* bw = &bars[w][c & 3];
      const unsigned par = (c >> 2) & 1;
      asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" ::"r"(su32(bw)), "r"(par));
    }
  }
  out[gw * 32 + lane] = acc;
}

int main() {
  const long long total = 1LL << 27;   // 1 GiB of doubles
  double *src, *out;
  cudaMalloc(&src, total * 8);
  cudaMalloc(&out, 1 << 24);
  cudaMemset(src, 0, total * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[4] = {"LDG.128 regs", "LDGSTS 16B", "LDGSTS 16B+L2hint", "TMA bulk"};
  for (int mode = 0; mode < 4; ++mode)
    for (int wpb : {4, 8}) {
      for (int cb : {512, 1024, 4096}) {
        if (mode != 3 && cb != 512 && cb != 4096) continue;
        const int blocks = 148 * (16 / wpb);
        const long long warps = (long long)blocks * wpb;
        const long long npw = (total / warps) / (cb / 8) * (cb / 8);
        const size_t smem = (size_t)wpb * 4 * 4096;
        auto launch = [&]() {
          if (mode == 0) stream<0><<<blocks, 32 * wpb, smem>>>(src, npw, out, cb);
          if (mode == 1) stream<1><<<blocks, 32 * wpb, smem>>>(src, npw, out, cb);
          if (mode == 2) stream<2><<<blocks, 32 * wpb, smem>>>(src, npw, out, cb);
          if (mode == 3) stream<3><<<blocks, 32 * wpb, smem>>>(src, npw, out, cb);
        };
        cudaFuncSetAttribute(stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        cudaFuncSetAttribute(stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        cudaFuncSetAttribute(stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        cudaFuncSetAttribute(stream<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        launch();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("%-20s warps/SM=%2d chunk=%5dB : %7.1f GB/s %s\n", names[mode], wpb * (16 / wpb), cb,
               warps * npw * 8.0 / (ms * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
      }
    }
  return 0;
}
