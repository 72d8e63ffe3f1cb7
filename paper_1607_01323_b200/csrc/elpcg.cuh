// Element-local (block-diagonal) PCG for the divergence-penalty projection
// (reference solvers.py:201-256 with op = apply_projection_operator(space, w,
// tau_D, None) and prec = inverse_mass_apply, operators.py:372-412 /
// kernels.py:95-108 -- the V3 projection solve).
//
// One CTA per cell runs the whole per-cell CG in shared memory: the operator
// (tensor mass + tau_D (div u, div v)), the exact inverse-mass
// preconditioner, the two dot products per iteration, the running Lanczos
// lambda_max and the eps floor of the stopping test.  Cells stop
// individually, as in the reference's masked batch.  No global traffic
// beyond reading b once and writing x once.
#pragma once
#include "vector.cuh"

namespace dg {

template <int N>
struct ElTab {
  double S[N * N], D[N * N];      // (q, i) on the n_q = n Gauss rule
  double M[N * N], Minv[N * N];   // 1D reference mass and its inverse
  double w[N];
};

template <int DIM>
struct ElCfg {
  static constexpr int THREADS = 256;
};

// Batched sweep along axis A of DIM component blocks [c][z][y][x] (N^DIM
// each): out[c][..r..] = sum_k T_c[r][k] in[c*ics][..k..], T_c = Tsel if
// c == A (the derivative direction of component c) else T.
template <int DIM, int N>
__device__ __forceinline__ void el_sweep(const double *in, int ics, double *out, const double *T,
                                         const double *Tsel, int A) {
  constexpr int NP = DIM == 3 ? N * N * N : N * N;
  const int stride = A == 0 ? 1 : (A == 1 ? N : N * N);
  for (int i = threadIdx.x; i < DIM * NP; i += blockDim.x) {
    const int c = i / NP, o = i - c * NP;
    const int r = (o / stride) % N;
    const int base = c * ics + o - r * stride;
    const double *Tc = (Tsel != nullptr && c == A) ? Tsel : T;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) acc += Tc[r * N + k] * in[base + k * stride];
    out[i] = acc;
  }
  __syncthreads();
}

template <int DIM, int N>
__global__ void __launch_bounds__(ElCfg<DIM>::THREADS)
el_pcg_kernel(const double *__restrict__ b, double *__restrict__ xout, const Geo g,
              const ElTab<N> tab, const double *__restrict__ tau_d, const double rel_tol,
              const int max_iter, const double floor_factor, int *__restrict__ iters_out,
              int *__restrict__ conv_out, const int64_t ncells) {
  constexpr int NP = DIM == 3 ? N * N * N : N * N;
  constexpr int V = DIM * NP;
  extern __shared__ double el_sm[];   // 7 * V doubles (dynamic: up to 84 KB at k=7)
  double *X = el_sm, *R = X + V, *P = R + V, *Z = P + V, *AP = Z + V, *T0 = AP + V, *T1 = T0 + V;
  __shared__ double S[N * N], D[N * N], ST[N * N], DT[N * N], M[N * N], Mi[N * N], W[N];
  __shared__ double red[32];
  __shared__ double bcast;
  const int tid = threadIdx.x;
  const int64_t e = blockIdx.x;
  const int ix = (int)(e % g.nx), iy = (int)((e / g.nx) % g.ny), iz = (int)(e / ((int64_t)g.nx * g.ny));
  const double h[3] = {g.hx[ix], g.hy[iy], DIM == 3 ? g.hz[iz] : 2.0};
  const double det = DIM == 3 ? 0.125 * h[0] * h[1] * h[2] : 0.25 * h[0] * h[1];
  const double td = tau_d ? tau_d[e] : 0.0;
  for (int i = tid; i < N * N; i += blockDim.x) {
    const int q = i / N, j = i % N;
    S[i] = tab.S[i];
    D[i] = tab.D[i];
    ST[j * N + q] = tab.S[i];
    DT[j * N + q] = tab.D[i];
    M[i] = tab.M[i];
    Mi[i] = tab.Minv[i];
  }
  for (int i = tid; i < N; i += blockDim.x) W[i] = tab.w[i];
  for (int i = tid; i < V; i += blockDim.x) {
    const int c = i / NP, o = i - c * NP;
    R[i] = b[((int64_t)c * ncells + e) * NP + o];
    X[i] = 0.0;
  }
  __syncthreads();

  // deterministic block dot product, broadcast to all threads
  auto dot = [&](const double *a, const double *c) {
    double acc = 0.0;
    for (int i = tid; i < V; i += blockDim.x) acc += a[i] * c[i];
    acc = block_sum(acc, red);
    if (tid == 0) bcast = acc;
    __syncthreads();
    const double v = bcast;
    __syncthreads();
    return v;
  };
  // z = M^-1 r: exact tensor inverse (kernels.py:95-108), one sweep per axis
  auto prec = [&](const double *r, double *z) {
    el_sweep<DIM, N>(r, NP, T0, Mi, nullptr, 0);
    el_sweep<DIM, N>(T0, NP, T1, Mi, nullptr, 1);
    if (DIM == 3) {
      el_sweep<DIM, N>(T1, NP, T0, Mi, nullptr, 2);
      for (int i = tid; i < V; i += blockDim.x) z[i] = T0[i] / det;
    } else {
      for (int i = tid; i < V; i += blockDim.x) z[i] = T1[i] / det;
    }
    __syncthreads();
  };
  // Ap = M p + tau_D (div p, div v) (operators.py:372-412, tau_C = None)
  auto apply = [&](const double *p, double *ap) {
    // tensor mass into ap
    el_sweep<DIM, N>(p, NP, T0, M, nullptr, 0);
    el_sweep<DIM, N>(T0, NP, T1, M, nullptr, 1);
    const double *mp = T1;
    if (DIM == 3) {
      el_sweep<DIM, N>(T1, NP, T0, M, nullptr, 2);
      mp = T0;
    }
    for (int i = tid; i < V; i += blockDim.x) ap[i] = det * mp[i];
    __syncthreads();
    if (td == 0.0) return;
    // d p_c / d xi_c at the Gauss points (D along own axis, S elsewhere)
    el_sweep<DIM, N>(p, NP, T0, S, D, 0);
    el_sweep<DIM, N>(T0, NP, T1, S, D, 1);
    const double *gq = T1;
    if (DIM == 3) {
      el_sweep<DIM, N>(T1, NP, T0, S, D, 2);
      gq = T0;
    }
    // tau div jxw at q points into the other buffer's first block
    double *dv = (gq == T0) ? T1 : T0;
    for (int i = tid; i < NP; i += blockDim.x) {
      double div = 0.0;
#pragma unroll
      for (int c = 0; c < DIM; ++c) div += (2.0 / h[c]) * gq[c * NP + i];
      const int x = i % N, y = (i / N) % N, z = DIM == 3 ? i / (N * N) : 0;
      const double jw = det * W[x] * W[y] * (DIM == 3 ? W[z] : 1.0);
      dv[i] = td * div * jw;
    }
    __syncthreads();
    // test with grad v_c: D^T along c, S^T elsewhere, times 2/h_c
    double *o1 = (dv == T0) ? T1 : T0;
    el_sweep<DIM, N>(dv, 0, o1, ST, DT, 0);      // component stride 0: broadcast
    el_sweep<DIM, N>(o1, NP, dv, ST, DT, 1);
    const double *res = dv;
    if (DIM == 3) {
      el_sweep<DIM, N>(dv, NP, o1, ST, DT, 2);
      res = o1;
    }
    for (int i = tid; i < V; i += blockDim.x) ap[i] += (2.0 / h[i / NP]) * res[i];
    __syncthreads();
  };

  const double eps = 2.220446049250313e-16;
  prec(R, Z);
  double rz = dot(R, Z);
  const double norm0 = sqrt(fmax(rz, 0.0));
  bool active = norm0 > rel_tol * norm0;
  int iters = 0;
  for (int i = tid; i < V; i += blockDim.x) P[i] = Z[i];
  __syncthreads();
  double lan_max = 1.0, alpha_prev = 1.0, beta_prev = 0.0;
  for (int it = 1; it <= max_iter && active; ++it) {
    apply(P, AP);
    const double pAp = dot(P, AP);
    const double alpha = rz / (pAp > 0.0 ? pAp : 1.0);
    lan_max = fmax(lan_max, 1.0 / alpha + beta_prev / alpha_prev);
    for (int i = tid; i < V; i += blockDim.x) {
      X[i] += alpha * P[i];
      R[i] -= alpha * AP[i];
    }
    __syncthreads();
    prec(R, Z);
    const double rz_new = dot(R, Z);
    const double norm = sqrt(fmax(rz_new, 0.0));
    iters = it;
    const double tol = fmax(rel_tol, floor_factor * eps * lan_max) * norm0;
    active = norm > tol;
    const double beta = active ? rz_new / (rz > 0.0 ? rz : 1.0) : 0.0;
    alpha_prev = alpha;
    beta_prev = beta;
    for (int i = tid; i < V; i += blockDim.x) P[i] = Z[i] + beta * P[i];
    __syncthreads();
    rz = rz_new;
  }
  for (int i = tid; i < V; i += blockDim.x) {
    const int c = i / NP, o = i - c * NP;
    xout[((int64_t)c * ncells + e) * NP + o] = X[i];
  }
  if (tid == 0) {
    if (iters_out) iters_out[e] = iters;
    if (conv_out) conv_out[e] = active ? 0 : 1;
  }
}

}  // namespace dg
