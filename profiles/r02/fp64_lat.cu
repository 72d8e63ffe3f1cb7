// DFMA / DADD latency and per-warp issue rate vs ILP on one SM (clock64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_lat fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, int OP>
__global__ void chain(double *out, double a, double b, int iters, long long *cyc) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int i = 0; i < ILP; ++i) x[i] = OP == 0 ? fma(x[i], a, b) : x[i] + b;
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int ILP, int OP>
void run(int warps, double *out, long long *cyc) {
  const int iters = 1000;
  chain<ILP, OP><<<1, 32 * warps>>>(out, 1.0000001, 1e-9, iters, cyc);
  long long h;
  cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double n = 16.0 * iters * ILP;  // instructions per warp
  printf("%s ILP=%d warps=%d : %.2f cycles per instr per warp, SM rate %.2f warp-instr/clk\n",
         OP == 0 ? "DFMA" : "DADD", ILP, warps, h / n, warps * n / h);
}

int main() {
  double *out;
  long long *cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1024);
  for (int w : {1, 4, 8, 16}) {
    run<1, 0>(w, out, cyc); run<2, 0>(w, out, cyc); run<4, 0>(w, out, cyc); run<8, 0>(w, out, cyc);
    run<1, 1>(w, out, cyc); run<4, 1>(w, out, cyc);
  }
  return 0;
}
