// Tensor-product cell operator out_e = scale_e (A (x) A (x) A) u_e on runs of
// contiguous cells (3D, odd n): TMA bulk load of the run into shared memory,
// three even-odd line sweeps, TMA bulk store.  No per-element index
// arithmetic on the global side.  Used for the consistent mass and its exact
// inverse (reference kernels.py:95-113, operators.py:167-181).
#pragma once
#include "laplace.cuh"

namespace dg {

template <int N>
struct EOTab {  // even-odd split of one centro-symmetric 1D matrix
  static constexpr int H = N / 2, NE = (N + 1) / 2;
  double Ae[NE * NE];
  double Ao[H * H > 0 ? H * H : 1];
};

__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <int N, int CPB>
__global__ void __launch_bounds__(((CPB * N * N + 31) / 32) * 32)
tensor_fast_kernel(const double *__restrict__ u, double *__restrict__ out, const Geo g,
                   const EOTab<N> T, const int64_t ncells_total, const int inverse) {
  constexpr int NP = N * N * N, LPC = N * N, H = N / 2, NE = (N + 1) / 2;
  constexpr int HO = H > 0 ? H : 1;
  static_assert(N & 1, "odd n: unpadded rows");
  __shared__ __align__(128) double buf[CPB * NP];
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * CPB;
  const int cnt = (int)min((int64_t)CPB, ncells_total - c0);
  const bool tma = !(cnt & 1) && ((reinterpret_cast<uintptr_t>(u) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  if (tma) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, (uint32_t)(cnt * NP * sizeof(double)));
      bulk_g2s(buf, u + c0 * NP, (uint32_t)(cnt * NP * sizeof(double)), &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
  } else {
    for (int i = tid; i < cnt * NP; i += blockDim.x) buf[i] = u[c0 * NP + i];
    __syncthreads();
  }
  const int c = tid / LPC, p = tid - c * LPC;
  const int a = p / N, b = p - a * N;
  const bool act = c < cnt;
  double v[N], e[NE], o[HO], E[NE], O[HO];
  auto sweep = [&](int base, int stride, double sc) {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = buf[base + q * stride];
    eo_split<N>(v, e, o);
    eo_apply<N, false>(T.Ae, T.Ao, e, o, sc, E, O);
    eo_merge<N>(E, O, v);
#pragma unroll
    for (int q = 0; q < N; ++q) buf[base + q * stride] = v[q];
  };
  // timing experiment (DG_EXP bit 3): 7 sweeps like the Laplace kernel
  const int reps = (g.exp_flags & 8) ? 3 : 1;
  for (int rep = 0; rep < reps; ++rep) {
    if (act) sweep(c * NP + (a * N + b) * N, 1, 1.0);  // x-lines (z=a, y=b)
    __syncthreads();
    if (act) sweep(c * NP + a * N * N + b, N, 1.0);    // y-lines (z=a, x=b)
    __syncthreads();
  }
  if (act) {                                          // z-lines (y=a, x=b) + scale
    const int64_t cell = (c0 + c) % ((int64_t)g.nx * g.ny * g.nz);
    const int ix = (int)(cell % g.nx), iy = (int)((cell / g.nx) % g.ny);
    const int iz = (int)(cell / ((int64_t)g.nx * g.ny));
    double s = 0.125 * g.hx[ix] * g.hy[iy] * g.hz[iz];
    if (inverse) s = 1.0 / s;
    sweep(c * NP + a * N + b, N * N, s);
  }
  // make the generic-proxy smem writes visible to the async proxy (TMA store)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (tma) {
    if (tid == 0) {
      bulk_s2g(out + c0 * NP, buf, (uint32_t)(cnt * NP * sizeof(double)));
      bulk_wait_read();
    }
  } else {
    for (int i = tid; i < cnt * NP; i += blockDim.x) out[c0 * NP + i] = buf[i];
  }
}

}  // namespace dg
