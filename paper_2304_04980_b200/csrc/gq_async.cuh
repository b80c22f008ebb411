// Small sm_100a helpers shared by the lean kernels: cp.async (LDGSTS) with L2 cache
// policies, commit/wait groups, fp64 m8n8k4 DMMA, 16-byte shared loads.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gq {
namespace as {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// Forces a uniform value (a shared-window base or ring-slot offset) into a vector register.
// ptxas for sm_100a may otherwise emit an LDGSTS whose shared destination is [R + UR]; that
// form faults with "illegal instruction" on B200 (build.py rejects any such SASS).
__device__ __forceinline__ unsigned lane_opaque(unsigned v) {
  return __shfl_sync(0xffffffffu, v, threadIdx.x & 31);
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 16-byte global -> shared copy; sz = 0 zero-fills without reading.  No L2 cache-policy
// operand: with one, ptxas (CUDA 12.9, sm_100a) sometimes encodes the copy with its shared
// address split as [R + UR] next to the policy descriptor, and that instruction faults with
// "illegal instruction" on B200 (build.py scans the SASS for the form).  The policy argument
// is kept for call-site symmetry.
__device__ __forceinline__ void ldgsts(unsigned dst, const double* src, int sz, uint64_t pol) {
  (void)pol;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_groups() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void dmma(double2& d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d.x), "+d"(d.y)
               : "d"(a), "d"(b));
}
// ---- mbarrier + bulk (TMA) copies ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// bytes % 16 == 0, both addresses 16-byte aligned; completes `bar`'s transaction count
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// bounded wait: a protocol bug traps (launch error) instead of hanging the device
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (long long i = 0; !mbar_try(bar, parity); ++i)
    if (i > (1LL << 28)) __trap();
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ double2 lds2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ double2 add2(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}

}  // namespace as
}  // namespace gq
