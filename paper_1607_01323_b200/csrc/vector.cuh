// Vector kernels for the Krylov solvers (reference solvers.py), fp64.
// Reductions are deterministic: fixed grid, fixed per-thread stride order,
// fixed tree order, second pass over the partials in index order.
#pragma once
#include "common.cuh"

namespace dg {

constexpr int kRedBlocks = 592;   // 4 x 148 SMs
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  v = 0.0;
  if (w == 0) {
    v = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;
}

// partial[b] = sum over this block's strided slice of x*y (y == null -> sum x)
static __global__ void dot_partial_kernel(const double *__restrict__ x,
                                   const double *__restrict__ y, int64_t n,
                                   double *__restrict__ partial) {
  __shared__ double sh[32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    acc += y ? x[i] * y[i] : x[i];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// out[0] = sum(partial[0..m)) in fixed order (one block); long arrays (the
// per-CTA partials of the vector kernels: 16-32k) with four independent
// accumulators per thread (m <= blockDim: one element per thread, as before)
static __global__ void sum_partials_kernel(const double *__restrict__ partial, int m,
                                    double *__restrict__ out) {
  __shared__ double sh[32];
  const int bd = blockDim.x;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int i = threadIdx.x;
  for (; i + 3 * bd < m; i += 4 * bd) {
    a0 += partial[i];
    a1 += partial[i + bd];
    a2 += partial[i + 2 * bd];
    a3 += partial[i + 3 * bd];
  }
  for (; i < m; i += bd) a0 += partial[i];
  double acc = (a0 + a1) + (a2 + a3);
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) *out = acc;
}

}  // namespace dg
