// fp64 tensor core (mma.sync m8n8k4 f64) throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dmma_tput(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[ILP][2];
#pragma unroll
  for (int k = 0; k < ILP; ++k) c[k][0] = c[k][1] = k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms = 148, iters = 4000;
  for (int wpsm : {1, 2, 4, 8, 16}) {
    for (int ilp : {1, 2, 4, 8}) {
      int threads = 32 * wpsm;
      cudaEventRecord(e0);
      if (ilp == 1) dmma_tput<1><<<sms, threads>>>(d, iters);
      if (ilp == 2) dmma_tput<2><<<sms, threads>>>(d, iters);
      if (ilp == 4) dmma_tput<4><<<sms, threads>>>(d, iters);
      if (ilp == 8) dmma_tput<8><<<sms, threads>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fma = (double)sms * wpsm * iters * ilp * 256.0;
      printf("DMMA warps/SM=%2d ILP=%d : %.2f TFLOP/s\n", wpsm, ilp, 2 * fma / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
