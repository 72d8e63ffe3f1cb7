// Measured fp64 peaks on this B200 (the roofline denominator for the
// "whichever binds" fp64 view): DFMA vector pipe and DMMA (mma.sync f64)
// tensor path, each alone and both interleaved.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double *out, int iters) {
  double a0 = threadIdx.x * 1e-7, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void dmma_loop(double *out, int iters, int mix) {
  double d[8][2] = {};
  const double a = 1e-3 * threadIdx.x, b = 0.5;
  double f0 = a, f1 = a + 1, f2 = a + 2, f3 = a + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(d[j][0], d[j][1], a, b);
    if (mix) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        f0 = fma(f0, b, a); f1 = fma(f1, b, a); f2 = fma(f2, b, a); f3 = fma(f3, b, a);
      }
    }
  }
  double s = f0 + f1 + f2 + f3;
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double *out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 4000;
  float ms;
  dfma_loop<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  dfma_loop<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma_tf = 2.0 * 128.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
  dmma_loop<<<blocks, threads>>>(out, 10, 0);
  cudaEventRecord(e0);
  dmma_loop<<<blocks, threads>>>(out, iters, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  // each mma.sync m8n8k4 = 8*8*4 FMA per warp
  const double dmma_tf = 2.0 * 256.0 * 8 * iters * (double)blocks * (threads / 32) / (ms * 1e-3) / 1e12;
  cudaEventRecord(e0);
  dmma_loop<<<blocks, threads>>>(out, iters, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double mix_tf = (2.0 * 256.0 * 8 * iters * (double)blocks * (threads / 32) +
                         2.0 * 32.0 * iters * (double)blocks * threads) / (ms * 1e-3) / 1e12;
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, "
         "\"dmma_plus_dfma_tflops\": %.3f}\n", sms, clk, dfma_tf, dmma_tf, mix_tf);
  return 0;
}
