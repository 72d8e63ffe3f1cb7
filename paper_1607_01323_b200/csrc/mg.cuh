// Multigrid transfer kernels (reference multigrid.py:33-73): the tensorial
// polynomial embedding of a coarse cell into its 2^dim children of the
// uniformly refined box (prolongation) and its transpose (restriction).
// One CTA per coarse cell: the parent and its children are staged in shared
// memory, each child gets three (two in 2D) sum-factorised sweeps with the
// 1D embedding matrix of its half along each axis.  Restriction sums the
// children's transposed sweeps in a fixed order (no atomics, deterministic).
#pragma once
#include "common.cuh"

namespace dg {

template <int DIM, int N, class R = double>
constexpr size_t mg_smem() {
  return sizeof(R) * (2 * N * N + (DIM == 3 ? N * N * N : N * N) * (1 + 2 * (1 << DIM)));
}

template <int N>
struct MgTab {
  double E[2][N * N];  // E[c][q*N + j] = l_j(0.5 (xi_q - 1)) (c = 0), l_j(0.5 (xi_q + 1)) (c = 1)
};

// one sweep along axis A on NCH blocks of NP values:
// out[ch][.. r ..] = sum_j M_ch[r][j] in[ch * ics][.. j ..], M_ch = E[bit_A(ch)] (or its
// transpose)
template <int DIM, int N, bool TRANS, class R>
__device__ __forceinline__ void mg_sweep(const R *in, int ics, R *out, const R *E, int A) {
  constexpr int NP = DIM == 3 ? N * N * N : N * N;
  constexpr int NCH = 1 << DIM;
  const int stride = A == 0 ? 1 : (A == 1 ? N : N * N);
  for (int i = threadIdx.x; i < NCH * NP; i += blockDim.x) {
    const int ch = i / NP, o = i - ch * NP;
    const int r = (o / stride) % N;
    const int base = ch * ics + o - r * stride;
    const R *M = E + ((ch >> A) & 1) * N * N;
    R acc = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j)
      acc += (TRANS ? M[j * N + r] : M[r * N + j]) * in[base + j * stride];
    out[i] = acc;
  }
  __syncthreads();
}

// xf[child] (+)= (E_z (x) E_y (x) E_x) xc[parent]
template <int DIM, int N, class R = double>
__global__ void mg_prolong_kernel(const R *__restrict__ xc, R *__restrict__ xf,
                                  const int ncx, const int ncy, const int ncz, const MgTab<N> T,
                                  const int add) {
  constexpr int NP = DIM == 3 ? N * N * N : N * N;
  constexpr int NCH = 1 << DIM;
  extern __shared__ __align__(16) unsigned char mg_raw[];  // E | parent | 2 x children
  R *E = reinterpret_cast<R *>(mg_raw), *par = E + 2 * N * N, *b0 = par + NP, *b1 = b0 + NCH * NP;
  const int64_t pc = blockIdx.x;
  const int px = (int)(pc % ncx), py = (int)((pc / ncx) % ncy), pz = (int)(pc / ((int64_t)ncx * ncy));
  for (int i = threadIdx.x; i < 2 * N * N; i += blockDim.x) E[i] = (R)(&T.E[0][0])[i];
  for (int i = threadIdx.x; i < NP; i += blockDim.x) par[i] = xc[pc * NP + i];
  __syncthreads();
  mg_sweep<DIM, N, false, R>(par, 0, b0, E, 0);
  mg_sweep<DIM, N, false, R>(b0, NP, b1, E, 1);
  const R *res = b1;
  if (DIM == 3) {
    mg_sweep<DIM, N, false, R>(b1, NP, b0, E, 2);
    res = b0;
  }
  const int nfx = 2 * ncx, nfy = 2 * ncy;
  for (int i = threadIdx.x; i < NCH * NP; i += blockDim.x) {
    const int ch = i / NP, o = i - ch * NP;
    const int fx = 2 * px + (ch & 1), fy = 2 * py + ((ch >> 1) & 1);
    const int fz = DIM == 3 ? 2 * pz + ((ch >> 2) & 1) : 0;
    const int64_t fe = fx + (int64_t)nfx * (fy + (int64_t)nfy * fz);
    R *dst = xf + fe * NP + o;
    *dst = add ? *dst + res[i] : res[i];
  }
}

// xc[parent] = sum_children (E_z^T (x) E_y^T (x) E_x^T) xf[child]
template <int DIM, int N, class R = double>
__global__ void mg_restrict_kernel(const R *__restrict__ xf, R *__restrict__ xc,
                                   const int ncx, const int ncy, const int ncz, const MgTab<N> T) {
  constexpr int NP = DIM == 3 ? N * N * N : N * N;
  constexpr int NCH = 1 << DIM;
  extern __shared__ __align__(16) unsigned char mg_raw[];
  R *E = reinterpret_cast<R *>(mg_raw), *b0 = E + 2 * N * N, *b1 = b0 + NCH * NP;
  const int64_t pc = blockIdx.x;
  const int px = (int)(pc % ncx), py = (int)((pc / ncx) % ncy), pz = (int)(pc / ((int64_t)ncx * ncy));
  const int nfx = 2 * ncx, nfy = 2 * ncy;
  for (int i = threadIdx.x; i < 2 * N * N; i += blockDim.x) E[i] = (R)(&T.E[0][0])[i];
  for (int i = threadIdx.x; i < NCH * NP; i += blockDim.x) {
    const int ch = i / NP, o = i - ch * NP;
    const int fx = 2 * px + (ch & 1), fy = 2 * py + ((ch >> 1) & 1);
    const int fz = DIM == 3 ? 2 * pz + ((ch >> 2) & 1) : 0;
    b0[i] = xf[(fx + (int64_t)nfx * (fy + (int64_t)nfy * fz)) * NP + o];
  }
  __syncthreads();
  mg_sweep<DIM, N, true, R>(b0, NP, b1, E, 0);
  mg_sweep<DIM, N, true, R>(b1, NP, b0, E, 1);
  const R *res = b0;
  if (DIM == 3) {
    mg_sweep<DIM, N, true, R>(b0, NP, b1, E, 2);
    res = b1;
  }
  for (int o = threadIdx.x; o < NP; o += blockDim.x) {
    R acc = 0.0;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) acc += res[ch * NP + o];
    xc[pc * NP + o] = acc;
  }
}

}  // namespace dg
