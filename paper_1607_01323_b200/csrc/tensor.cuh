// Tensor-product cell operator  out_e = scale_e (A (x) A (x) A) u_e  for the
// consistent mass (A = M = S^T W S, scale = prod h/2) and its exact inverse
// (A = M^-1, scale = prod 2/h).  Replaces apply_mass / apply_inverse_mass
// (reference kernels.py:95-113); on affine cells JxW is a constant times the
// tensor weights, so S^-1 diag(1/JxW) S^-T = (M^-1)^(x)dim / det.
#pragma once
#include "common.cuh"
#include "laplace.cuh"

namespace dg {

template <int DIM, int N>
struct TensorCfg {
  static constexpr int RP = row_pitch<N>();
  static constexpr int LPC = (DIM == 3) ? N * N : N;
  static constexpr int CS = (DIM == 3) ? N * N * RP : N * RP;
  static constexpr int NC = (DIM == 3) ? (N <= 4 ? 16 : (N <= 6 ? 8 : 4)) : 32;
  static constexpr int NL = NC * LPC;
  static constexpr int THREADS = ((NL + 31) / 32) * 32;
  static constexpr size_t SMEM = sizeof(double) * NC * CS;
};

template <int DIM, int N>
__global__ void __launch_bounds__(TensorCfg<DIM, N>::THREADS)
tensor_apply_kernel(const double *__restrict__ u, double *__restrict__ out, const Geo g,
                    const TensorTab<N> T, const int64_t ncells, const int inverse) {
  using C = TensorCfg<DIM, N>;
  constexpr int RP = C::RP, LPC = C::LPC, CS = C::CS;
  constexpr int NP = (DIM == 3) ? N * N * N : N * N;
  __shared__ double buf[C::NC * C::CS];
  const int64_t c0 = (int64_t)blockIdx.x * C::NC;
  const int tid = threadIdx.x;
  for (int i = tid; i < C::NC * NP; i += blockDim.x) {
    const int c = i / NP, o = i % NP;
    const int x = o % N, y = (o / N) % N, z = (DIM == 3) ? o / (N * N) : 0;
    buf[c * CS + (z * N + y) * RP + x] = (c0 + c < ncells) ? u[(c0 + c) * NP + o] : 0.0;
  }
  __syncthreads();
  const int l = tid;
  const int c = l / LPC, t = l % LPC;
  const bool active = l < C::NL && c0 + c < ncells;
  const int ta = (DIM == 3) ? t / N : 0, tb = (DIM == 3) ? t % N : t;
  double v[N];
  // x sweep (line (ta,tb) = (z,y))
  if (active) {
    const int base = c * CS + (ta * N + tb) * RP;
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = buf[base + q];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double a = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) a += T.A[i * N + q] * v[q];
      buf[base + i] = a;
    }
  }
  __syncthreads();
  // y sweep (line (z, x))
  if (active) {
    const int base = c * CS + ta * N * RP + tb;
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = buf[base + q * RP];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double a = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) a += T.A[i * N + q] * v[q];
      buf[base + i * RP] = a;
    }
  }
  if (DIM == 3) {
    __syncthreads();
    if (active) {
      const int base = c * CS + ta * RP + tb;
#pragma unroll
      for (int q = 0; q < N; ++q) v[q] = buf[base + q * N * RP];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double a = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) a += T.A[i * N + q] * v[q];
        buf[base + i * N * RP] = a;
      }
    }
  }
  __syncthreads();
  // scale and store (coalesced)
  const int64_t ncell_geo = (int64_t)g.nx * g.ny * g.nz;
  for (int i = tid; i < C::NC * NP; i += blockDim.x) {
    const int cc = i / NP, o = i % NP;
    if (c0 + cc >= ncells) continue;
    const int64_t e = (c0 + cc) % ncell_geo;
    const int ix = (int)(e % g.nx), iy = (int)((e / g.nx) % g.ny), iz = (int)(e / ((int64_t)g.nx * g.ny));
    double s = 0.5 * g.hx[ix] * 0.5 * g.hy[iy];
    if (DIM == 3) s *= 0.5 * g.hz[iz];
    if (inverse) s = 1.0 / s;
    const int x = o % N, y = (o / N) % N, z = (DIM == 3) ? o / (N * N) : 0;
    out[(c0 + cc) * NP + o] = s * buf[cc * CS + (z * N + y) * RP + x];
  }
}

}  // namespace dg
