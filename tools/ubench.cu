// Micro-benchmarks for design decisions: fp64 FMA latency / throughput, broadcast LDS rate.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_lat(double* out, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 32; ++k) x = fma(x, a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / (iters * 32.0);
  out[1 + threadIdx.x] = x;
}

template <int ILP>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void lds_tput(double* out, int iters) {
  __shared__ double2 buf[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = make_double2(i, i + 1);
  __syncthreads();
  double s = 0, s2 = 0;
  int idx = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      double2 v = buf[(idx + k) & 255];   // warp-uniform address (broadcast)
      s += v.x;
      s2 += v.y;
    }
    idx += 3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + s2;
}

int main() {
  double* d;
  cudaMalloc(&d, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_lat<<<1, 32>>>(d, 1000, 1.0000001, 1e-9);
  double h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("dfma dependent latency: %.2f cycles\n", h[0]);
  int sms = 148;
  int iters = 2000;
  for (int wpsm : {1, 2, 4, 8, 16, 32}) {
    int threads = 32 * wpsm;
    if (threads > 1024) threads = 1024;
    int blocks = sms * (32 * wpsm / threads);
    for (int ilp : {1, 4, 8}) {
      cudaEventRecord(e0);
      if (ilp == 1) dfma_tput<1><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
      if (ilp == 4) dfma_tput<4><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
      if (ilp == 8) dfma_tput<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fmas = (double)blocks * threads * iters * 8 * ilp;
      printf("warps/SM=%2d ILP=%d : %.2f TFLOP/s fp64\n", wpsm, ilp, 2 * fmas / (ms * 1e-3) / 1e12);
    }
  }
  for (int wpsm : {1, 4, 8, 16}) {
    int threads = 32 * wpsm;
    cudaEventRecord(e0);
    lds_tput<<<sms, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double lds = (double)sms * wpsm * iters * 16;   // warp-level LDS.128 instructions
    printf("broadcast LDS.128 warps/SM=%2d : %.3f instr/cycle/SM (at 1.965 GHz)\n", wpsm,
           lds / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
