// Cartesian fast path of the two vector operators inside the velocity CG
// solves, 3D, fp64, sm_100a:
//   viscous Helmholtz  (gamma0/dt) M u + SIP of -div(2 nu eps(u))
//                      (reference operators.py:418-491)
//   projection         M u + tau_D (div v, div u) + tau_C [u].[v]
//                      (operators.py:372-412)
//
// Same bilinear forms and quadrature (n_q = k+1 Gauss points per axis, face
// integrals on the tensor Gauss points of the face) as the generic
// quadrature-point kernel (vecops.cuh), reorganised for throughput:
//
// * The cell is carried in the Gauss-collocated representation
//   u~ = (S x S x S) u (S: nodes -> Gauss points, square since n_q = N), so
//   values at quadrature points are the data itself, gradients are one
//   N-point collocation derivative (Dg) per axis, and all volume and face
//   test terms accumulate at the Gauss points before one final
//   (S^T x S^T x S^T) back to the nodal basis.
// * Face traces (value and physical normal derivative of every component on
//   every side, at the face Gauss points) are produced once per cell by a
//   trace kernel into a [cell][side][comp][val|dn][face point] buffer; the
//   apply kernel reads its own and its neighbours' traces from it (L2), so
//   no CTA loads a neighbour cell.  Tangential derivatives on a face are
//   taken from the traces (the two cells of a face share the tangential
//   Gauss points of a tensor box mesh).
// * The kernels themselves (one thread per component line) are in
//   vcart2.cuh; this header holds the tables, the shared helpers and the
//   fused CG update of the velocity solves.
//
// Face flux algebra (own frame, outward normal n = nsgn e_d, j = u - u_nbr,
// {.} = average, w = {u_d} (Dirichlet side: u_d, j = u)):
//   V_a   = -(nu nsgn ({d_d u_a} + (a == d ? {d_d u_d} : d_a w)) - tau' j_a) sj
//   Gn_a  = c0 nu nsgn sj (j_a + [a == d] j_d)       normal-gradient test
//   Gt_b  = c0 nu nsgn sj j_b  (b != d, component d) tangential-gradient test
// with tau' = nu max(tau_e, tau_nbr) (Dirichlet: 2 nu tau_e) and c0 = -1/2
// (Dirichlet: -1): the generic kernel's V[a], G[a][b] (vecops.cuh:632-650)
// with the zero entries of G removed.
#pragma once
#include "common.cuh"
#include "vecops.cuh"

namespace dg {

template <int N>
struct VcTab {
  double S[N * N];   // S[q][i] = l_i(x_q), GLL nodal basis at Gauss points
  double Dg[N * N];  // Dg[q][m] = lg_m'(x_q), Lagrange basis on the Gauss points
  double w[N];       // Gauss weights
  double eL[N], eR[N];  // lg_m(-1), lg_m(+1)
  double gL[N], gR[N];  // lg_m'(-1), lg_m'(+1)
};

enum VcOp : int { kVcHelmholtz = 0, kVcProjection = 1 };

template <int N>
struct VcCfg {
  static constexpr int P = N * N * N;  // points per cell
  static constexpr int F = N * N;      // points per face
  static constexpr int CPB = P >= 256 ? 1 : 256 / P;
  static constexpr int THREADS = CPB * P;
  static constexpr int TAB = 2 * N * N + 5 * N;
  // per cell: u~ (3P) + tg / ping-pong (6P) | face scratch (Wf 6F, JV 18F,
  // AN 18F, GT 12F)
  static constexpr int VOL = 9 * P;
  static constexpr int FACE = 54 * F;
  static constexpr int CELL = (VOL > FACE ? VOL : FACE) | 1;
  static constexpr size_t SMEM = sizeof(double) * (TAB + CPB * CELL);
  static constexpr int TRC = 36 * F;  // trace doubles per cell
};

// v[i] for a runtime i without a local-memory copy of v
__device__ __forceinline__ double vc_sel(const double (&v)[3], int i) {
  return i == 0 ? v[0] : (i == 1 ? v[1] : v[2]);
}

// index of the point with coordinate AX replaced by m
template <int N, int AX>
__device__ __forceinline__ int vc_idx(int x, int y, int z, int m) {
  return AX == 0 ? m + N * (y + N * z) : (AX == 1 ? x + N * (m + N * z) : x + N * (y + N * m));
}

// sum_m coef[m * cs] * buf[point with coordinate AX = m]
template <int N, int AX>
__device__ __forceinline__ double vc_dot(const double *coef, int cs, const double *buf, int x, int y,
                                         int z) {
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < N; ++m) acc = fma(coef[m * cs], buf[vc_idx<N, AX>(x, y, z, m)], acc);
  return acc;
}

template <int N>
__device__ __forceinline__ void vc_stage_tab(double *tb, const VcTab<N> &t) {
  constexpr int TAB = VcCfg<N>::TAB;
  const double *src = reinterpret_cast<const double *>(&t);
  for (int i = threadIdx.x; i < TAB; i += blockDim.x) tb[i] = src[i];
}

// One M^-1-preconditioned CG update of the velocity solves (solvers.py:56-67
// with prec = inverse_mass_apply), fused per cell:
//   alpha = rz / pAp;  x += alpha p;  r -= alpha Ap;  z = M^-1 r;  partial r.z
// M^-1 = (Minv x Minv x Minv) / det with the same sweep order (x, y, z) and
// scale as dg_inverse_mass (tensor.cuh).  One thread per node, CPB cells per
// CTA; per-CTA partial sums are added in fixed order by a second kernel.
template <int N>
struct MinvTab {
  double A[N * N];
};

template <int N>
__global__ void __launch_bounds__(((VcCfg<N>::THREADS + 31) / 32) * 32)
vpcg_update_kernel(double *__restrict__ x, double *__restrict__ r, const double *__restrict__ p,
                   const double *__restrict__ Ap, double *__restrict__ z,
                   const double *__restrict__ scal, const __grid_constant__ MinvTab<N> mi,
                   const Geo g, const int64_t ncells, double *__restrict__ partials) {
  using C = VcCfg<N>;
  constexpr int P = C::P;
  __shared__ double buf[2][C::CPB * 3 * P];
  __shared__ double red[32];
  // M^-1 rows in shared memory: indexing the parameter by the lane's node
  // coordinate serialised the constant cache
  __shared__ double sA[N * N];
  if (!(scal[1] > 0.0)) return;  // breakdown: the host stops, x and r stay
  if (threadIdx.x < N * N) sA[threadIdx.x] = mi.A[threadIdx.x];
  const double alpha = __ddiv_rn(scal[0], scal[1]);
  // blockDim = THREADS rounded up to whole warps (full-mask shuffles below);
  // the padding threads own no node
  const bool in = threadIdx.x < C::THREADS;
  const int cs = in ? threadIdx.x / P : 0, q = in ? threadIdx.x % P : 0;
  const int x0 = q % N, y0 = (q / N) % N, z0 = q / (N * N);
  const int64_t e = (int64_t)blockIdx.x * C::CPB + cs;
  const bool valid = in && e < ncells;
  double *b0 = buf[0] + cs * 3 * P, *b1 = buf[1] + cs * 3 * P;
  double rv[3], xv[3], pv[3], av[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {  // all twelve loads first
    const int64_t i = ((int64_t)c * ncells + e) * P + q;
    if (valid) {
      xv[c] = x[i];
      pv[c] = p[i];
      rv[c] = r[i];
      av[c] = Ap[i];
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int64_t i = ((int64_t)c * ncells + e) * P + q;
    double v = 0.0;
    if (valid) {
      x[i] = __dadd_rn(xv[c], __dmul_rn(alpha, pv[c]));
      v = __dsub_rn(rv[c], __dmul_rn(alpha, av[c]));
      r[i] = v;
    }
    rv[c] = v;
    if (in) b0[c * P + q] = v;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double t = vc_dot<N, 0>(sA + x0 * N, 1, b0 + c * P, x0, y0, z0);
    if (in) b1[c * P + q] = t;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double t = vc_dot<N, 1>(sA + y0 * N, 1, b1 + c * P, x0, y0, z0);
    if (in) b0[c * P + q] = t;
  }
  __syncthreads();
  double acc = 0.0;
  if (valid) {
    const unsigned eu = (unsigned)e, nx = (unsigned)g.nx, ny = (unsigned)g.ny;
    const unsigned qq = eu / nx, iz = qq / ny;
    const int ix = (int)(eu - qq * nx), iy = (int)(qq - iz * ny);
    double s = 0.5 * g.hx[ix] * 0.5 * g.hy[iy];
    s *= 0.5 * g.hz[iz];
    s = 1.0 / s;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double zv = s * vc_dot<N, 2>(sA + z0 * N, 1, b0 + c * P, x0, y0, z0);
      z[((int64_t)c * ncells + e) * P + q] = zv;
      acc += rv[c] * zv;
    }
  }
  // deterministic block sum
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = acc;
  __syncthreads();
  if (w == 0) {
    acc = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) partials[blockIdx.x] = acc;
  }
}

}  // namespace dg
