// Quadrature-point DG operators on Cartesian cells, fp64, sm_100a:
//   viscous Helmholtz   (reference operators.py:418-491)
//   projection M + tau_D div-div + tau_C jump   (operators.py:372-412)
//   convective term with local Lax-Friedrichs flux (operators.py:533-604)
//   once-per-step right-hand sides (operators.py:241-366, 494-527, 610-672):
//     divergence a(q,u) (standard / weak / strong), pressure gradient b(v,p)
//     (standard / weak), vorticity (before its inverse mass), consistent
//     pressure Neumann data, pressure-Dirichlet data, viscous boundary data
//
// Per cell: values and reference gradients at the tensor Gauss points by sum
// factorisation, the pointwise physics, then the adjoint contractions; face
// terms are evaluated cell-centrically in the "own cell" frame (own outward
// normal, jump = own - neighbour), which reproduces the reference's
// minus/plus scatter (spaces.py:151-163) with each output DoF written once,
// no atomics.
//
// One CTA per cell.  Neighbour cells are read from global memory (L2) into
// shared memory one face at a time.  NCI input / NCO output components.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace dg {

enum VecOp : int {
  kOpHelmholtz = 0,
  kOpProjection = 1,
  kOpConvective = 2,
  kOpDivergence = 3,
  kOpGradient = 4,
  kOpVorticity = 5,
  kOpPressureNeumann = 6,
  kOpGpDirichlet = 7,
  kOpViscousBc = 8,
};
enum RhsForm : int { kFormStandard = 0, kFormWeak = 1, kFormStrong = 2 };

constexpr int kMaxHist = 4;

struct VecParams {
  int op;
  double gamma0_dt, nu;          // Helmholtz, pressure Neumann, viscous bc
  const double *tau_d;           // projection: per cell (or null)
  const double *tau_c;           // projection: [d*ncell + e] face e|e+d (or null)
  int n_hist;                    // convective, pressure Neumann
  const double *hist[kMaxHist];
  const double *vort[kMaxHist];  // pressure Neumann: vorticity levels
  double beta[kMaxHist];
  double scale;                  // divergence / gradient
  double tau_scale;              // pressure-Dirichlet data
  int form;                      // RhsForm
  int n_vort;                    // vorticity components (1 in 2D, 3 in 3D)
  // boundary face data per side, [tangential cell][component][face point]
  // (face points [slow][fast] over the tangential axes), or null = zero
  const double *bnd[6];
  // convective: Dirichlet data g per history level and side (same layout)
  const double *gh[kMaxHist][6];
  // convective: body force at the volume quadrature points [comp][cell][QP]
  const double *vol_data;
};

template <int N, int NQ>
struct QuadTab {
  double S[NQ * N];   // S[q][i] = l_i(x_q)
  double D[NQ * N];   // D[q][i] = l_i'(x_q)
  double w[NQ];       // Gauss weights
  double dL[N], dR[N];
};

template <int DIM, int N, int NQ, int NCI, int NCO>
struct VecCfg {
  static constexpr int NP = DIM == 3 ? N * N * N : N * N;
  static constexpr int QP = DIM == 3 ? NQ * NQ * NQ : NQ * NQ;
  static constexpr int FQ = DIM == 3 ? NQ * NQ : NQ;  // face points
  static constexpr int FN = DIM == 3 ? N * N : N;     // face nodes
  static constexpr int MX = (N > NQ ? N : NQ);
  static constexpr int BIG = DIM == 3 ? MX * MX * MX : MX * MX;
  static constexpr int THREADS = QP >= 256 ? 256 : (QP > 64 ? 128 : 64);
  static constexpr int NCM = NCI > NCO ? NCI : NCO;
  // shared layout (doubles).  The volume buffers (QV, QG, TG) and the face
  // buffers (NB, FO, FB, FV, FT) are alive in different phases and share one
  // region: fewer doubles per cell, more cells resident per SM.
  static constexpr int U = 0;                       // own cell, NCI * NP
  static constexpr int OUT = U + NCI * NP;          // accumulator, NCO * NP
  static constexpr int T0 = OUT + NCO * NP;         // temporaries, 3 * BIG
  static constexpr int T1 = T0 + BIG;
  static constexpr int T2 = T1 + BIG;
  static constexpr int ACC = T2 + BIG;              // pressure Neumann data, DIM * FQ
  static constexpr int SHARED = ACC + DIM * FQ;     // volume | face region
  static constexpr int QV = SHARED;                 // values at q points, NCM * QP
  static constexpr int QG = QV + NCM * QP;          // phys gradients, NCI * DIM * QP
  static constexpr int TG = QG + NCI * DIM * QP;    // test data, DIM * QP
  static constexpr int VOL_END = TG + DIM * QP;
  static constexpr int NB = SHARED;                 // neighbour cell, NCI * NP
  static constexpr int FO = NB + NCI * NP;          // own face traces NCI*(1+DIM)*FQ
  static constexpr int FB = FO + NCI * (1 + DIM) * FQ;  // neighbour traces
  static constexpr int FV = FB + NCI * (1 + DIM) * FQ;  // face test data NCO*(1+DIM)*FQ
  static constexpr int FT = FV + NCO * (1 + DIM) * FQ;  // face temporaries 2*BIG
  static constexpr int FACE_END = FT + 2 * BIG;
  static constexpr int TAB = VOL_END > FACE_END ? VOL_END : FACE_END;  // tables S, D, ST, DT
  static constexpr int HSM = TAB + 4 * NQ * N + NQ + 2 * N;  // cell sizes: own[3], neighbour[3]
  static constexpr int NDBL = HSM + 6;
  static constexpr size_t SMEM = sizeof(double) * NDBL;
};

// Contraction along axis A of a [E2][E1][E0] array (x = axis 0 fastest):
// out[..r..] = sum_c T[r*Cc + c] in[..c..], T is R x Cc.  All extents are
// compile-time constants (no integer divisions in the index math).
template <int R, int Cc, int A, int E0, int E1, int E2>
__device__ __forceinline__ void contract(const double *in, double *out, const double *T) {
  constexpr int O0 = A == 0 ? R : E0, O1 = A == 1 ? R : E1, O2 = A == 2 ? R : E2;
  constexpr int TOT = O0 * O1 * O2;
  constexpr int STRIDE = A == 0 ? 1 : (A == 1 ? E0 : E0 * E1);
  for (int i = threadIdx.x; i < TOT; i += blockDim.x) {
    const int x = i % O0, y = (i / O0) % O1, z = i / (O0 * O1);
    int r, base;
    if (A == 0) { r = x; base = (z * E1 + y) * E0; }
    else if (A == 1) { r = y; base = z * E1 * E0 + x; }
    else { r = z; base = y * E0 + x; }
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < Cc; ++c) acc += T[r * Cc + c] * in[base + c * STRIDE];
    out[i] = acc;
  }
  __syncthreads();
}

// Shared scratch and tables used by the face helpers.
struct FaceScratch {
  double *t0, *t1, *t2, *ft;
  const double *S, *D, *ST, *DT, *dL, *dR;
  int big;
};

// Index of node (slow sl, fast fa, normal k) of a face normal to d.
template <int DIM, int N>
__device__ __forceinline__ int face_node(int d, int sl, int fa, int k) {
  if (DIM == 3) {
    if (d == 0) return (sl * N + fa) * N + k;       // (z,y) fixed, x=k
    if (d == 1) return (sl * N + k) * N + fa;       // (z,x) fixed, y=k
    return (k * N + sl) * N + fa;                   // (y,x) fixed, z=k
  }
  return d == 0 ? fa * N + k : k * N + fa;
}

// Traces of `ncomp` components of one cell (components NP apart) on side
// (d, s): dst[c][0] value, dst[c][1+b] physical gradient component b, each
// over the FQ face points [slow][fast] (kernels.py:119-156).
template <int DIM, int N, int NQ>
__device__ void face_traces(const double *cell, int ncomp, int d, int s, const double h[3],
                            double *dst, const FaceScratch &F, bool need_grad = true) {
  constexpr int NP = DIM == 3 ? N * N * N : N * N;
  constexpr int FQ = DIM == 3 ? NQ * NQ : NQ;
  constexpr int FN = DIM == 3 ? N * N : N;
  for (int c = 0; c < ncomp; ++c) {
    const double *cc = cell + c * NP;
    for (int i = threadIdx.x; i < FN; i += blockDim.x) {
      const int sl = DIM == 3 ? i / N : 0, fa = DIM == 3 ? i % N : i;
      double vv = 0.0, dd = 0.0;
      for (int k = 0; k < N; ++k) {
        const double x = cc[face_node<DIM, N>(d, sl, fa, k)];
        if (k == (s ? N - 1 : 0)) vv = x;
        dd += (s ? F.dR[k] : F.dL[k]) * x;
      }
      F.ft[i] = vv;
      F.ft[F.big + i] = dd;
    }
    __syncthreads();
    double *dv = dst + (c * (1 + DIM)) * FQ;
    if (!need_grad) {  // values only (convective, projection, divergence, gradient)
      if (DIM == 3) {
        contract<NQ, N, 0, N, N, 1>(F.ft, F.t0, F.S);
        contract<NQ, N, 1, NQ, N, 1>(F.t0, dv, F.S);
      } else {
        contract<NQ, N, 0, N, 1, 1>(F.ft, dv, F.S);
      }
      continue;
    }
    if (DIM == 3) {
      contract<NQ, N, 0, N, N, 1>(F.ft, F.t0, F.S);
      contract<NQ, N, 1, NQ, N, 1>(F.t0, dv, F.S);                          // value
      contract<NQ, N, 0, N, N, 1>(F.ft + F.big, F.t1, F.S);
      contract<NQ, N, 1, NQ, N, 1>(F.t1, dv + (1 + d) * FQ, F.S);           // normal
      const int tfa = d == 0 ? 1 : 0, tsl = d == 2 ? 1 : 2;
      contract<NQ, N, 0, N, N, 1>(F.ft, F.t2, F.D);
      contract<NQ, N, 1, NQ, N, 1>(F.t2, dv + (1 + tfa) * FQ, F.S);         // d/d fast
      contract<NQ, N, 1, NQ, N, 1>(F.t0, dv + (1 + tsl) * FQ, F.D);         // d/d slow
    } else {
      contract<NQ, N, 0, N, 1, 1>(F.ft, dv, F.S);
      contract<NQ, N, 0, N, 1, 1>(F.ft + F.big, dv + (1 + d) * FQ, F.S);
      contract<NQ, N, 0, N, 1, 1>(F.ft, dv + (1 + (1 - d)) * FQ, F.D);
    }
    for (int i = threadIdx.x; i < DIM * FQ; i += blockDim.x) {
      const int b = i / FQ;
      dv[(1 + b) * FQ + (i % FQ)] *= 2.0 / h[b];
    }
    __syncthreads();
  }
}

// Adjoint of face_traces, accumulated into out (components NP apart):
// fv[c][0] value-test data, fv[c][1+b] physical gradient-test data
// (kernels.py:159-186).  Gradient tests only when grad_terms.
template <int DIM, int N, int NQ>
__device__ void face_lift(const double *fv, int ncomp, int d, int s, const double h[3],
                          bool grad_terms, double *out, const FaceScratch &F) {
  constexpr int NP = DIM == 3 ? N * N * N : N * N;
  constexpr int FQ = DIM == 3 ? NQ * NQ : NQ;
  constexpr int FN = DIM == 3 ? N * N : N;
  for (int c = 0; c < ncomp; ++c) {
    const double *dv = fv + (c * (1 + DIM)) * FQ;
    if (DIM == 3) {
      const int tfa = d == 0 ? 1 : 0, tsl = d == 2 ? 1 : 2;
      contract<N, NQ, 0, NQ, NQ, 1>(dv, F.t0, F.ST);
      contract<N, NQ, 1, N, NQ, 1>(F.t0, F.t1, F.ST);           // value part [sl][fa]
      if (grad_terms) {
        contract<N, NQ, 0, NQ, NQ, 1>(dv + (1 + tfa) * FQ, F.t0, F.DT);
        contract<N, NQ, 1, N, NQ, 1>(F.t0, F.t2, F.ST);
        for (int i = threadIdx.x; i < FN; i += blockDim.x) F.t1[i] += (2.0 / h[tfa]) * F.t2[i];
        __syncthreads();
        contract<N, NQ, 0, NQ, NQ, 1>(dv + (1 + tsl) * FQ, F.t0, F.ST);
        contract<N, NQ, 1, N, NQ, 1>(F.t0, F.t2, F.DT);
        for (int i = threadIdx.x; i < FN; i += blockDim.x) F.t1[i] += (2.0 / h[tsl]) * F.t2[i];
        __syncthreads();
        contract<N, NQ, 0, NQ, NQ, 1>(dv + (1 + d) * FQ, F.t0, F.ST);
        contract<N, NQ, 1, N, NQ, 1>(F.t0, F.t2, F.ST);          // normal-gradient part
      }
    } else {
      const int tt = 1 - d;
      contract<N, NQ, 0, NQ, 1, 1>(dv, F.t1, F.ST);
      if (grad_terms) {
        contract<N, NQ, 0, NQ, 1, 1>(dv + (1 + tt) * FQ, F.t2, F.DT);
        for (int i = threadIdx.x; i < FN; i += blockDim.x) F.t1[i] += (2.0 / h[tt]) * F.t2[i];
        __syncthreads();
        contract<N, NQ, 0, NQ, 1, 1>(dv + (1 + d) * FQ, F.t2, F.ST);
      }
    }
    double *oc = out + c * NP;
    const double sn = 2.0 / h[d];
    for (int i = threadIdx.x; i < FN; i += blockDim.x) {
      const int sl = DIM == 3 ? i / N : 0, fa = DIM == 3 ? i % N : i;
      for (int k = 0; k < N; ++k) {
        double add = 0.0;
        if (k == (s ? N - 1 : 0)) add += F.t1[i];
        if (grad_terms) add += sn * (s ? F.dR[k] : F.dL[k]) * F.t2[i];
        oc[face_node<DIM, N>(d, sl, fa, k)] += add;
      }
    }
    __syncthreads();
  }
}

template <int DIM, int N, int NQ, int NCI, int NCO>
__global__ void __launch_bounds__(VecCfg<DIM, N, NQ, NCI, NCO>::THREADS)
vecop_kernel(const double *__restrict__ u, double *__restrict__ out, const Geo g,
             const QuadTab<N, NQ> tab, const VecParams prm, const int64_t ncells) {
  using C = VecCfg<DIM, N, NQ, NCI, NCO>;
  constexpr int NP = C::NP, QP = C::QP, FQ = C::FQ;
  extern __shared__ double sm[];
  double *su = sm + C::U, *snb = sm + C::NB, *sout = sm + C::OUT;
  double *qv = sm + C::QV, *qg = sm + C::QG;
  double *t0 = sm + C::T0, *t1 = sm + C::T1, *t2 = sm + C::T2, *tg = sm + C::TG;
  double *fo = sm + C::FO, *fb = sm + C::FB, *fv = sm + C::FV, *ft = sm + C::FT;
  double *S = sm + C::TAB, *D = S + NQ * N, *ST = D + NQ * N, *DT = ST + NQ * N;
  double *W = DT + NQ * N, *dL = W + NQ, *dR = dL + N;
  double *hs = sm + C::HSM, *hsn = hs + 3;  // cell sizes for the face helpers (shared:
                                            // no local-memory copy of an indexed array)
  // kernel-parameter arrays indexed by runtime level / side, staged in shared
  // memory (a dynamically indexed parameter array would be copied to local)
  __shared__ const double *p_hist[kMaxHist], *p_vort[kMaxHist], *p_bnd[6], *p_gh[kMaxHist][6];
  __shared__ double p_beta[kMaxHist];
  const int tid = threadIdx.x;
  const int64_t e = blockIdx.x;
  const int ix = (int)(e % g.nx), iy = (int)((e / g.nx) % g.ny), iz = (int)(e / ((int64_t)g.nx * g.ny));
  const double h[3] = {g.hx[ix], g.hy[iy], DIM == 3 ? g.hz[iz] : 2.0};
  if (tid < 3) hs[tid] = tid == 0 ? h[0] : (tid == 1 ? h[1] : h[2]);
  double det = 0.125 * h[0] * h[1] * h[2];
  if (DIM == 2) det = 0.25 * h[0] * h[1];
  const FaceScratch F{t0, t1, t2, ft, S, D, ST, DT, dL, dR, C::BIG};

  for (int i = tid; i < NQ * N; i += blockDim.x) {
    S[i] = tab.S[i];
    D[i] = tab.D[i];
    const int q = i / N, j = i % N;
    ST[j * NQ + q] = tab.S[i];
    DT[j * NQ + q] = tab.D[i];
  }
  for (int i = tid; i < NQ; i += blockDim.x) W[i] = tab.w[i];
  for (int i = tid; i < N; i += blockDim.x) {
    dL[i] = tab.dL[i];
    dR[i] = tab.dR[i];
  }
  for (int i = tid; i < NCO * NP; i += blockDim.x) sout[i] = 0.0;
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < kMaxHist; ++j) {
      p_hist[j] = prm.hist[j];
      p_vort[j] = prm.vort[j];
      p_beta[j] = prm.beta[j];
#pragma unroll
      for (int q = 0; q < 6; ++q) p_gh[j][q] = prm.gh[j][q];
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) p_bnd[q] = prm.bnd[q];
  }
  __syncthreads();

  const int op = prm.op;
  constexpr int e0 = N, e1 = N, e2 = DIM == 3 ? N : 1;
  constexpr int q0 = NQ, q1 = NQ, q2 = DIM == 3 ? NQ : 1;
  auto wq = [&](int i) {  // tensor weight * det at q point i
    const int x = i % NQ, y = (i / NQ) % NQ, z = DIM == 3 ? i / (NQ * NQ) : 0;
    return det * W[x] * W[y] * (DIM == 3 ? W[z] : 1.0);
  };
  auto load = [&](const double *src, int ncomp, int64_t cell, double *dst) {
    for (int i = tid; i < ncomp * NP; i += blockDim.x) {
      const int c = i / NP, o = i % NP;
      dst[i] = src[((int64_t)c * ncells + cell) * NP + o];
    }
  };
  // face-weight factor and outward normal sign of side (d, s)
  auto face_det = [&](int d) {
    double f = 1.0;
    for (int b = 0; b < DIM; ++b)
      if (b != d) f *= 0.5 * h[b];
    return f;
  };
  auto face_sj = [&](double fdet, int i) {
    const int fa = DIM == 3 ? i % NQ : i, sl = DIM == 3 ? i / NQ : 0;
    return fdet * W[fa] * (DIM == 3 ? W[sl] : 1.0);
  };
  // boundary kind of side (d, s) of this cell: 0 interior / periodic,
  // kBndNone (velocity-Dirichlet) or kBndNeumann (velocity-Neumann)
  // index of this cell in the boundary-data arrays of a side normal to d
  auto tan_index = [&](int d) -> int64_t {
    if (DIM == 3)
      return d == 0 ? (int64_t)iz * g.ny + iy : (d == 1 ? (int64_t)iz * g.nx + ix : (int64_t)iy * g.nx + ix);
    return d == 0 ? iy : ix;
  };
  auto side_kind = [&](int d, int s) {
    const int nd = d == 0 ? g.nx : (d == 1 ? g.ny : g.nz);
    const int nidx = (d == 0 ? ix : (d == 1 ? iy : iz)) + (s ? 1 : -1);
    if (nidx >= 0 && nidx < nd) return 0;
    const int m = g.mode[2 * d + s];
    return (m == kBndNone || m == kBndNeumann) ? m : 0;
  };

  if (op == kOpPressureNeumann || op == kOpGpDirichlet || op == kOpViscousBc) {
    // ---- boundary-data right-hand sides: face lifts on boundary sides only
    for (int side = 0; side < 2 * DIM; ++side) {
      const int d = side >> 1, s = side & 1;
      const int kind = side_kind(d, s);
      if (kind == 0) continue;
      if (op == kOpPressureNeumann && kind != kBndNone) continue;
      if (op == kOpGpDirichlet && kind != kBndNeumann) continue;
      const int64_t it = tan_index(d);
      const double *bd = p_bnd[side];
      const double fdet = face_det(d);
      const double nsgn = s ? 1.0 : -1.0;
      bool grad_terms = false;
      if (op == kOpPressureNeumann) {
        // h_a = sum_i beta_i (div(u u) + nu curl w)_a (+ dg/dt - f data)
        double *acc = sm + C::ACC;  // DIM * FQ accumulators (the face buffers alias qv)
        for (int i = tid; i < DIM * FQ; i += blockDim.x) acc[i] = 0.0;
        for (int lev = 0; lev < prm.n_hist; ++lev) {
          load(p_hist[lev], DIM, e, su);
          load(p_vort[lev], prm.n_vort, e, snb);
          __syncthreads();
          face_traces<DIM, N, NQ>(su, DIM, d, s, hs, fo, F);
          face_traces<DIM, N, NQ>(snb, prm.n_vort, d, s, hs, fb, F);
          const double beta = p_beta[lev];
          for (int i = tid; i < FQ; i += blockDim.x) {
            double uu[DIM], gr[DIM][DIM], gw[3][DIM];
            for (int c = 0; c < DIM; ++c) {
              uu[c] = fo[(c * (1 + DIM)) * FQ + i];
              for (int b = 0; b < DIM; ++b) gr[c][b] = fo[(c * (1 + DIM) + 1 + b) * FQ + i];
            }
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int b = 0; b < DIM; ++b)
                gw[c][b] = c < prm.n_vort ? fb[(c * (1 + DIM) + 1 + b) * FQ + i] : 0.0;
            double div = 0.0;
            for (int c = 0; c < DIM; ++c) div += gr[c][c];
            double curl[DIM];
            if (DIM == 2) {
              curl[0] = gw[0][1];
              curl[1] = -gw[0][0];
            } else {
              curl[0] = gw[2][1] - gw[1][DIM - 1];
              curl[1] = gw[0][DIM - 1] - gw[2][0];
              curl[DIM - 1] = gw[1][0] - gw[0][1];
            }
            for (int a = 0; a < DIM; ++a) {
              double conv = uu[a] * div;
              for (int c = 0; c < DIM; ++c) conv += uu[c] * gr[a][c];
              acc[a * FQ + i] += beta * (conv + prm.nu * curl[a]);
            }
          }
          __syncthreads();
        }
        for (int i = tid; i < FQ; i += blockDim.x) {
          double hd = acc[d * FQ + i];
          if (bd) hd += bd[(it * DIM + d) * FQ + i];
          fv[i] = -(hd * nsgn) * face_sj(fdet, i);
          for (int b = 0; b < DIM; ++b) fv[(1 + b) * FQ + i] = 0.0;
        }
      } else if (op == kOpGpDirichlet) {
        // 2 tau g_p (q, .) and -g_p (grad q . n) (operators.py:241-259)
        const double taub = prm.tau_scale * g.tau[e];
        grad_terms = true;
        for (int i = tid; i < FQ; i += blockDim.x) {
          const double gp = bd ? bd[it * FQ + i] : 0.0;
          const double sj = face_sj(fdet, i);
          fv[i] = 2.0 * taub * gp * sj;
          for (int b = 0; b < DIM; ++b) fv[(1 + b) * FQ + i] = (b == d) ? -gp * nsgn * sj : 0.0;
        }
      } else {  // viscous boundary data (operators.py:494-527)
        const double taub = g.tau[e] * prm.nu;
        grad_terms = kind == kBndNone;
        for (int i = tid; i < FQ; i += blockDim.x) {
          const double sj = face_sj(fdet, i);
          if (kind == kBndNone) {
            double gu[DIM];
            for (int a = 0; a < DIM; ++a) gu[a] = bd ? bd[(it * DIM + a) * FQ + i] : 0.0;
            for (int a = 0; a < DIM; ++a) {
              fv[(a * (1 + DIM)) * FQ + i] = 2.0 * taub * gu[a] * sj;
              for (int b = 0; b < DIM; ++b) {
                const double na = (a == d) ? nsgn : 0.0, nb = (b == d) ? nsgn : 0.0;
                fv[(a * (1 + DIM) + 1 + b) * FQ + i] = -prm.nu * (gu[a] * nb + gu[b] * na) * sj;
              }
            }
          } else {
            const double gp = bd ? bd[(it * (DIM + 1) + DIM) * FQ + i] : 0.0;
            for (int a = 0; a < DIM; ++a) {
              const double ha = bd ? bd[(it * (DIM + 1) + a) * FQ + i] : 0.0;
              fv[(a * (1 + DIM)) * FQ + i] = (ha + gp * ((a == d) ? nsgn : 0.0)) * sj;
              for (int b = 0; b < DIM; ++b) fv[(a * (1 + DIM) + 1 + b) * FQ + i] = 0.0;
            }
          }
        }
      }
      __syncthreads();
      face_lift<DIM, N, NQ>(fv, NCO, d, s, hs, grad_terms, sout, F);
    }
  } else {
    // ---- volume + face operators ---------------------------------------------
    const bool weak = prm.form == kFormWeak;
    const bool need_qv = op == kOpHelmholtz || op == kOpProjection || op == kOpConvective ||
                         ((op == kOpDivergence || op == kOpGradient) && weak);
    const bool need_qg = op == kOpHelmholtz || op == kOpVorticity ||
                         (op == kOpProjection && prm.tau_d != nullptr) ||
                         ((op == kOpDivergence || op == kOpGradient) && !weak);
    const bool need_val = op == kOpHelmholtz || op == kOpProjection || op == kOpVorticity ||
                          ((op == kOpDivergence || op == kOpGradient) && !weak);
    // gradient tests: all directions, only b == a, or none
    const int grad_mode = (op == kOpHelmholtz || op == kOpConvective ||
                           (op == kOpDivergence && weak)) ? 2
                          : ((op == kOpProjection && prm.tau_d != nullptr) ||
                             (op == kOpGradient && weak)) ? 1 : 0;
    const int nlev = op == kOpConvective ? prm.n_hist : 1;
    for (int lev = 0; lev < nlev; ++lev) {
      const double *src = op == kOpConvective ? p_hist[lev] : u;
      const double beta = op == kOpConvective ? p_beta[lev] : 1.0;
      load(src, NCI, e, su);
      __syncthreads();
      // ---- values and physical gradients at q points ------------------------
      for (int c = 0; c < NCI; ++c) {
        const double *uc = su + c * NP;
        double *val = qv + c * QP;
        if (DIM == 3) {
          contract<NQ, N, 0, e0, e1, e2>(uc, t0, S);                 // [z][y][qx]
          contract<NQ, N, 1, q0, e1, e2>(t0, t1, S);                 // [z][qy][qx]
          if (need_qv) contract<NQ, N, 2, q0, q1, e2>(t1, val, S);   // values
          if (need_qg) {
            contract<NQ, N, 2, q0, q1, e2>(t1, qg + (c * DIM + 2) * QP, D);  // d/dz
            contract<NQ, N, 1, q0, e1, e2>(t0, t2, D);
            contract<NQ, N, 2, q0, q1, e2>(t2, qg + (c * DIM + 1) * QP, S);  // d/dy
            contract<NQ, N, 0, e0, e1, e2>(uc, t0, D);
            contract<NQ, N, 1, q0, e1, e2>(t0, t1, S);
            contract<NQ, N, 2, q0, q1, e2>(t1, qg + (c * DIM + 0) * QP, S);  // d/dx
          }
        } else {
          contract<NQ, N, 0, e0, e1, 1>(uc, t0, S);
          if (need_qv) contract<NQ, N, 1, q0, e1, 1>(t0, val, S);
          if (need_qg) {
            contract<NQ, N, 1, q0, e1, 1>(t0, qg + (c * DIM + 1) * QP, D);
            contract<NQ, N, 0, e0, e1, 1>(uc, t0, D);
            contract<NQ, N, 1, q0, e1, 1>(t0, qg + (c * DIM + 0) * QP, S);
          }
        }
      }
      if (need_qg) {
        for (int i = tid; i < NCI * DIM * QP; i += blockDim.x) {
          const int d = (i / QP) % DIM;
          qg[i] *= 2.0 / hs[d];
        }
        __syncthreads();
      }
      // ---- pointwise physics + adjoint integration per output component -----
      for (int a = 0; a < NCO; ++a) {
        for (int i = tid; i < QP; i += blockDim.x) {
          const double jw = wq(i);
          double vt = 0.0;
          if (op == kOpHelmholtz) {
            vt = prm.gamma0_dt * qv[a * QP + i] * jw;
            for (int b = 0; b < DIM; ++b)
              tg[b * QP + i] = prm.nu * (qg[(a * DIM + b) * QP + i] + qg[(b * DIM + a) * QP + i]) * jw;
          } else if (op == kOpProjection) {
            vt = qv[a * QP + i] * jw;
            if (grad_mode) {
              double div = 0.0;
              for (int b = 0; b < DIM; ++b) div += qg[(b * DIM + b) * QP + i];
              tg[a * QP + i] = prm.tau_d[e] * div * jw;
            }
          } else if (op == kOpConvective) {
            for (int b = 0; b < DIM; ++b) tg[b * QP + i] = beta * qv[a * QP + i] * qv[b * QP + i] * jw;
          } else if (op == kOpDivergence) {
            if (weak) {
              for (int b = 0; b < DIM; ++b) tg[b * QP + i] = prm.scale * qv[b * QP + i] * jw;
            } else {
              double div = 0.0;
              for (int b = 0; b < DIM; ++b) div += qg[(b * DIM + b) * QP + i];
              vt = -prm.scale * div * jw;
            }
          } else if (op == kOpGradient) {
            if (weak) tg[a * QP + i] = prm.scale * qv[i] * jw;
            else vt = -prm.scale * qg[a * QP + i] * jw;
          } else {  // vorticity: curl u, component a (grad[c][b] at qg[(c*DIM+b)])
            double w;
            if (DIM == 2) {
              w = qg[(1 * DIM + 0) * QP + i] - qg[(0 * DIM + 1) * QP + i];
            } else {
              const int b1 = (a + 1) % 3, b2 = (a + 2) % 3;
              w = qg[(b2 * DIM + b1) * QP + i] - qg[(b1 * DIM + b2) * QP + i];
            }
            vt = w * jw;
          }
          t2[i] = vt;
        }
        __syncthreads();
        double *oa = sout + a * NP;
        if (need_val) {
          if (DIM == 3) {
            contract<N, NQ, 0, q0, q1, q2>(t2, t0, ST);
            contract<N, NQ, 1, e0, q1, q2>(t0, t1, ST);
            contract<N, NQ, 2, e0, e1, q2>(t1, t0, ST);
          } else {
            contract<N, NQ, 0, q0, q1, 1>(t2, t1, ST);
            contract<N, NQ, 1, e0, q1, 1>(t1, t0, ST);
          }
          for (int i = tid; i < NP; i += blockDim.x) oa[i] += t0[i];
          __syncthreads();
        }
        for (int b = 0; b < DIM; ++b) {
          if (grad_mode == 0 || (grad_mode == 1 && b != a)) continue;
          // phys test: (2/h_b) * reference gradient test along b
          const double sc = 2.0 / h[b];
          const double *gb = tg + b * QP;
          if (DIM == 3) {
            contract<N, NQ, 0, q0, q1, q2>(gb, t0, b == 0 ? DT : ST);
            contract<N, NQ, 1, e0, q1, q2>(t0, t1, b == 1 ? DT : ST);
            contract<N, NQ, 2, e0, e1, q2>(t1, t0, b == 2 ? DT : ST);
          } else {
            contract<N, NQ, 0, q0, q1, 1>(gb, t1, b == 0 ? DT : ST);
            contract<N, NQ, 1, e0, q1, 1>(t1, t0, b == 1 ? DT : ST);
          }
          for (int i = tid; i < NP; i += blockDim.x) oa[i] += sc * t0[i];
          __syncthreads();
        }
      }
      // ---- faces ------------------------------------------------------------
      const bool faces = (op == kOpHelmholtz && prm.nu != 0.0) ||
                         (op == kOpProjection && prm.tau_c != nullptr) || op == kOpConvective ||
                         ((op == kOpDivergence || op == kOpGradient) && prm.form != kFormStandard);
      if (!faces) continue;
      // the face physics indexes gradients by the face direction: make it a
      // compile-time constant (no local-memory arrays)
      auto do_side = [&](auto dconst, const int s) {
        constexpr int d = decltype(dconst)::value;
        const int side = 2 * d + s;
        const int kind = side_kind(d, s);
        // projection / strong divergence: interior faces only; Helmholtz:
        // nothing on velocity-Neumann faces; others: all faces
        if ((op == kOpProjection || (op == kOpDivergence && prm.form == kFormStrong)) && kind != 0)
          return;
        if (op == kOpHelmholtz && kind == kBndNeumann) return;
        int64_t en = e;
        double hn = h[d];
        if (kind == 0) {
          const int nd = d == 0 ? g.nx : (d == 1 ? g.ny : g.nz);
          int nidx = (d == 0 ? ix : (d == 1 ? iy : iz)) + (s ? 1 : -1);
          if (nidx < 0 || nidx >= nd) nidx = s ? 0 : nd - 1;  // periodic wrap
          const int cx = d == 0 ? nidx : ix, cy = d == 1 ? nidx : iy, cz = d == 2 ? nidx : iz;
          en = cx + (int64_t)g.nx * (cy + (int64_t)g.ny * cz);
          hn = d == 0 ? g.hx[nidx] : (d == 1 ? g.hy[nidx] : g.hz[nidx]);
          load(src, NCI, en, snb);
        }
        __syncthreads();
        const bool tgrad = op == kOpHelmholtz;  // only the viscous flux needs face gradients
        if (tid < 3) hsn[tid] = tid == d ? hn : hs[tid];  // the neighbour differs along d only
        __syncthreads();
        face_traces<DIM, N, NQ>(su, NCI, d, s, hs, fo, F, tgrad);
        if (kind == 0) face_traces<DIM, N, NQ>(snb, NCI, d, 1 - s, hsn, fb, F, tgrad);
        const double fdet = face_det(d);
        const double nsgn = s ? 1.0 : -1.0;  // own outward normal = nsgn e_d
        double tau = 0.0;
        if (op == kOpHelmholtz) {
          const double te = g.tau[e];
          tau = (kind == 0 ? fmax(te, g.tau[en]) : te) * prm.nu;
        } else if (op == kOpProjection) {
          // tau_c of the face between the lower cell and its +d neighbour
          tau = prm.tau_c[(int64_t)d * ncells + (s ? e : en)];
        }
        for (int i = tid; i < FQ; i += blockDim.x) {
          const double sj = face_sj(fdet, i);
          double uo[NCI], un[NCI], go[NCI][DIM], gn[NCI][DIM];
          for (int c = 0; c < NCI; ++c) {
            uo[c] = fo[(c * (1 + DIM)) * FQ + i];
            un[c] = kind == 0 ? fb[(c * (1 + DIM)) * FQ + i] : 0.0;
            for (int b = 0; b < DIM; ++b) {
              go[c][b] = fo[(c * (1 + DIM) + 1 + b) * FQ + i];
              gn[c][b] = kind == 0 ? fb[(c * (1 + DIM) + 1 + b) * FQ + i] : 0.0;
            }
          }
          double V[NCO], G[NCO][DIM];
          for (int c = 0; c < NCO; ++c) {
            V[c] = 0.0;
            for (int b = 0; b < DIM; ++b) G[c][b] = 0.0;
          }
          if (op == kOpHelmholtz) {
            // (2 nu eps(u) n)_a with the own outward normal n = nsgn e_d
            for (int a = 0; a < NCO; ++a) {
              const double vo = prm.nu * (go[a][d] + go[d][a]) * nsgn;
              if (kind == 0) {
                const double vn = prm.nu * (gn[a][d] + gn[d][a]) * nsgn;
                const double avg = 0.5 * (vo + vn);
                V[a] = -(avg - tau * (uo[a] - un[a])) * sj;
              } else {  // velocity-Dirichlet face (operators.py:473-483)
                V[a] = -(vo - 2.0 * tau * uo[a]) * sj;
              }
            }
            for (int a = 0; a < NCO; ++a)
              for (int b = 0; b < DIM; ++b) {
                const double ja = kind == 0 ? uo[a] - un[a] : uo[a];
                const double jb = kind == 0 ? uo[b] - un[b] : uo[b];
                const double na = (a == d) ? nsgn : 0.0, nb = (b == d) ? nsgn : 0.0;
                G[a][b] = (kind == 0 ? -0.5 : -1.0) * prm.nu * (ja * nb + jb * na) * sj;
              }
          } else if (op == kOpProjection) {
            for (int a = 0; a < NCO; ++a) V[a] = tau * (uo[a] - un[a]) * sj;
          } else if (op == kOpConvective) {
            // local Lax-Friedrichs, own frame (operators.py:597-604)
            double up[NCI];
            if (kind == 0) {
              for (int c = 0; c < NCI; ++c) up[c] = un[c];
            } else {  // mirror state 2 g - u with the level's Dirichlet data
              const double *gd = p_gh[lev][side];
              for (int c = 0; c < NCI; ++c)
                up[c] = (gd ? 2.0 * gd[(tan_index(d) * NCI + c) * FQ + i] : 0.0) - uo[c];
            }
            const double unm = uo[d] * nsgn, unp = up[d] * nsgn;
            if (kind == kBndNeumann) {
              for (int a = 0; a < NCO; ++a) V[a] = -beta * uo[a] * unm * sj;
            } else {
              const double lam = 2.0 * fmax(fabs(unm), fabs(unp));
              for (int a = 0; a < NCO; ++a) {
                const double Fl = 0.5 * (uo[a] * unm + up[a] * unp) + 0.5 * lam * (uo[a] - up[a]);
                V[a] = -beta * Fl * sj;
              }
            }
          } else if (op == kOpDivergence) {
            // own-frame u.n: weak -scale {u}.n (boundary: own trace),
            // strong +scale [u].n / 2 (operators.py:289-316)
            if (prm.form == kFormWeak)
              V[0] = -prm.scale * (kind == 0 ? 0.5 * (uo[d] + un[d]) : uo[d]) * nsgn * sj;
            else
              V[0] = prm.scale * 0.5 * (uo[d] - un[d]) * nsgn * sj;
          } else {  // weak pressure gradient: -scale {p} n_a (operators.py:346-366)
            const double pav = kind == 0 ? 0.5 * (uo[0] + un[0]) : uo[0];
            for (int a = 0; a < NCO; ++a) V[a] = (a == d) ? -prm.scale * pav * nsgn * sj : 0.0;
          }
          for (int c = 0; c < NCO; ++c) {
            fv[(c * (1 + DIM)) * FQ + i] = V[c];
            for (int b = 0; b < DIM; ++b) fv[(c * (1 + DIM) + 1 + b) * FQ + i] = G[c][b];
          }
        }
        __syncthreads();
        face_lift<DIM, N, NQ>(fv, NCO, d, s, hs, op == kOpHelmholtz, sout, F);
      };
      for (int side = 0; side < 2 * DIM; ++side) {
        const int sd = side & 1;
        switch (side >> 1) {
          case 0: do_side(std::integral_constant<int, 0>(), sd); break;
          case 1: do_side(std::integral_constant<int, 1>(), sd); break;
          default:
            if (DIM == 3) do_side(std::integral_constant<int, DIM - 1>(), sd);
            break;
        }
      }
    }
    if (op == kOpConvective && prm.vol_data != nullptr) {
      // (v, f) with the body force sampled at the quadrature points
      for (int a = 0; a < NCO; ++a) {
        for (int i = tid; i < QP; i += blockDim.x)
          t2[i] = prm.vol_data[((int64_t)a * ncells + e) * QP + i] * wq(i);
        __syncthreads();
        if (DIM == 3) {
          contract<N, NQ, 0, q0, q1, q2>(t2, t0, ST);
          contract<N, NQ, 1, e0, q1, q2>(t0, t1, ST);
          contract<N, NQ, 2, e0, e1, q2>(t1, t0, ST);
        } else {
          contract<N, NQ, 0, q0, q1, 1>(t2, t1, ST);
          contract<N, NQ, 1, e0, q1, 1>(t1, t0, ST);
        }
        for (int i = tid; i < NP; i += blockDim.x) sout[a * NP + i] += t0[i];
        __syncthreads();
      }
    }
  }
  for (int i = tid; i < NCO * NP; i += blockDim.x) {
    const int c = i / NP, o = i % NP;
    out[((int64_t)c * ncells + e) * NP + o] = sout[i];
  }
}

}  // namespace dg
