// Multigrid transfer kernels (reference multigrid.py:33-73): the tensorial
// polynomial embedding of a coarse cell into its 2^dim children of the
// uniformly refined box (prolongation) and its transpose (restriction).
// One CTA per coarse cell: the parent and its children are staged in shared
// memory and pass through pairwise tree sweeps with the 1D embedding matrix
// of each half along each axis (mg_tree_sweep); restriction sums the two
// halves of each pair in a fixed order (no atomics, deterministic).
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

// Pairwise tree sweeps along axis A: prolongation doubles the block count
// (out[2 ib + h] = E_h along A applied to in[ib]), restriction halves it
// (out[ob] = sum_h E_h^T along A applied to in[2 ob + h]); with the axes in
// the order z, y, x (prolongation) / x, y, z (restriction) the block index is
// the child index bx + 2 by + 4 bz.  2 + 4 + 8 = 14 blocks of N^4 FMAs per
// coarse cell instead of 3 x 8 = 24 for three sweeps over all children.
template <int DIM, int N, bool TRANS, class R>
__device__ __forceinline__ void mg_tree_sweep(const R *in, int nout, R *out, const R *E, int A) {
  constexpr int NP = DIM == 3 ? N * N * N : N * N;
  const int stride = A == 0 ? 1 : (A == 1 ? N : N * N);
  for (int i = threadIdx.x; i < nout * NP; i += blockDim.x) {
    const int ob = i / NP, o = i - ob * NP;
    const int r = (o / stride) % N;
    const int base = o - r * stride;
    R acc = 0.0;
    if (!TRANS) {  // out block ob = 2 ib + h
      const R *M = E + (ob & 1) * N * N;
      const R *src = in + (ob >> 1) * NP + base;
#pragma unroll
      for (int j = 0; j < N; ++j) acc += M[r * N + j] * src[j * stride];
    } else {  // out block ob = sum_h from in blocks 2 ob + h
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const R *M = E + h * N * N;
        const R *src = in + (2 * ob + h) * NP + base;
#pragma unroll
        for (int j = 0; j < N; ++j) acc += M[j * N + r] * src[j * stride];
      }
    }
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
  const R *res;
  if (DIM == 3) {
    mg_tree_sweep<DIM, N, false, R>(par, 2, b0, E, 2);
    mg_tree_sweep<DIM, N, false, R>(b0, 4, b1, E, 1);
    mg_tree_sweep<DIM, N, false, R>(b1, 8, b0, E, 0);
    res = b0;
  } else {
    mg_tree_sweep<DIM, N, false, R>(par, 2, b0, E, 1);
    mg_tree_sweep<DIM, N, false, R>(b0, 4, b1, E, 0);
    res = b1;
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
  mg_tree_sweep<DIM, N, true, R>(b0, NCH / 2, b1, E, 0);
  mg_tree_sweep<DIM, N, true, R>(b1, NCH / 4, b0, E, 1);
  const R *res = b0;
  if (DIM == 3) {
    mg_tree_sweep<DIM, N, true, R>(b0, 1, b1, E, 2);
    res = b1;
  }
  for (int o = threadIdx.x; o < NP; o += blockDim.x) xc[pc * NP + o] = res[o];
}

}  // namespace dg
