// General-geometry 2D operators (quadrilaterals with iso-parametric, possibly
// curved mappings and arbitrary conforming connectivity, face orientation
// flips), fp64, sm_100a: the reference's 2D code path exactly as it is
// written (operators.py, kernels.py, geometry.py, spaces.py), with per
// quadrature-point geometry data instead of the Cartesian closed forms:
//
//   volume  JxW (q) and J^-T (q), kernel layout [cell][qy][qx]
//   faces   own J^-T, outward unit normal and surface JxW per (cell, slot,
//           face point); on interior faces both cells use the minus side's
//           normal (negated on the plus side) and sJxW, as the reference's
//           gather/scatter does (spaces.py:140-163)
//   links   neighbour cell / slot / flip per (cell, slot); boundary kind per
//           (cell, slot) from the boundary conditions
//
// Cells are evaluated cell-centrically in their own frame (own outward
// normal, jump = own - neighbour): every output node is written by exactly
// one thread, no atomics.  2D cells are small (n^2 <= 64 nodes), so values
// and gradients at a point are direct n^2 sums over the cell (no sum
// factorisation): per-cell work is a few thousand FMAs and the path is
// bound by the geometry data it streams (5 doubles per volume point, 7 per
// face point), like the reference's own layout.
//
// Operators (one kernel, NCI input / NCO output components, runtime op):
//   mass, exact inverse mass, SIP pressure Laplacian (+ its block-diagonal
//   part for the Jacobi diagonal), viscous Helmholtz, projection, convective
//   term (over-integration geometry, history levels, Dirichlet data, body
//   force), divergence (standard / weak / strong), pressure gradient
//   (standard / weak), vorticity (before its inverse mass), and the
//   boundary-data right-hand sides (pressure-Dirichlet data, viscous
//   boundary data, consistent pressure Neumann data) whose data callables
//   the host samples at the face points.
#pragma once
#include "common.cuh"

namespace dg {

constexpr int kG2MaxN = 8, kG2MaxQ = 11, kG2MaxHist = 4;

enum G2Op : int {
  kG2Mass = 0,
  kG2InvMass = 1,
  kG2Laplace = 2,
  kG2Helmholtz = 3,
  kG2Projection = 4,
  kG2Convective = 5,
  kG2Divergence = 6,
  kG2Gradient = 7,
  kG2Vorticity = 8,
  kG2LaplaceLocal = 9,  // neighbour traces zeroed (block-diagonal part)
  kG2GpDirichlet = 10,  // pressure-Dirichlet data (operators.py:241-259)
  kG2ViscousBc = 11,    // viscous boundary data (operators.py:494-527)
  kG2PressureNeumann = 12,  // consistent pressure Neumann data (operators.py:621-672)
};

struct G2Tab {  // 1D tables of the rule (S, D: n_q x n, row-major)
  double S[kG2MaxQ * kG2MaxN], D[kG2MaxQ * kG2MaxN];
  double Si[kG2MaxN * kG2MaxN];  // S^-1 (n_q = n only)
  double ld[kG2MaxN], rd[kG2MaxN];
};

struct G2Geo {
  int n, nq;
  int64_t ncells;
  const double *jxw;      // [e][q][q]
  const double *jit;      // [e][4][q][q]  (00 01 10 11)
  const double *fsj;      // [e][4][q]
  const double *fnrm;     // [e][4][2][q]
  const double *fjit;     // [e][4][4][q]
  const int64_t *nbr;     // [e][4] neighbour cell or -1
  const int *nslot;       // [e][4]
  const int *nflip;       // [e][4]
  const double *tau;      // [e]
};

struct G2Params {
  int op;
  double tau_scale;       // Laplace
  const int *kind;        // [e][4]: 0 interior, DG_BC_VELOCITY_DIRICHLET / _NEUMANN
  int local_node;         // kG2LaplaceLocal: unit vector at this node (-1: use src)
  double gamma0_dt, nu;   // Helmholtz
  const double *tau_d;    // projection: [e] or null
  const double *tau_c;    // projection: [e][4] or null
  double scale;           // divergence / gradient
  int form;               // 0 standard, 1 weak, 2 strong
  int n_hist;             // convective: levels, their beta and Dirichlet data
  const double *hist[kG2MaxHist];
  double beta[kG2MaxHist];
  const double *gdata[kG2MaxHist];  // [e][4][2][q] or null (homogeneous)
  const double *body;     // [2][e][q][q] body force at the points, or null
  const double *vort[kG2MaxHist];   // pressure Neumann: vorticity levels (scalar)
  const double *fdata;    // boundary-data ops: host-sampled data per (cell, slot, point):
                          //   gp Dirichlet [e][4][q]; viscous bc [e][4][3][q]
                          //   (g0 g1 - | h0 h1 g_p); pressure Neumann [e][4][2][q]
                          //   (dg/dt - f), or null
};

// value and reference gradient of a cell field at face point q of slot s
// (kernels.py:119-156)
__device__ __forceinline__ void g2_trace(const double *u, int N, const G2Tab &T, int s, int q,
                                         double &v, double &gx, double &gy) {
  v = gx = gy = 0.0;
  if (s < 2) {  // x = -1 / +1: points along y
    const int i0 = s == 0 ? 0 : N - 1;
    const double *dd = s == 0 ? T.ld : T.rd;
    for (int j = 0; j < N; ++j) {
      const double sq = T.S[q * N + j];
      double dxl = 0.0;
      for (int i = 0; i < N; ++i) dxl = fma(u[j * N + i], dd[i], dxl);
      v = fma(sq, u[j * N + i0], v);
      gx = fma(sq, dxl, gx);
      gy = fma(T.D[q * N + j], u[j * N + i0], gy);
    }
  } else {      // y = -1 / +1: points along x
    const int j0 = s == 2 ? 0 : N - 1;
    const double *dd = s == 2 ? T.ld : T.rd;
    for (int i = 0; i < N; ++i) {
      const double sq = T.S[q * N + i];
      double dyl = 0.0;
      for (int j = 0; j < N; ++j) dyl = fma(dd[j], u[j * N + i], dyl);
      v = fma(sq, u[j0 * N + i], v);
      gx = fma(T.D[q * N + i], u[j0 * N + i], gx);
      gy = fma(sq, dyl, gy);
    }
  }
}

__device__ __forceinline__ int g2_nci(int op) {
  if (op == kG2GpDirichlet || op == kG2ViscousBc) return 0;
  if (op == kG2PressureNeumann) return 3;  // u (2) + vorticity (1)
  return (op == kG2Helmholtz || op == kG2Projection || op == kG2Convective ||
          op == kG2Divergence || op == kG2Vorticity) ? 2 : 1;
}
__device__ __forceinline__ int g2_nco(int op) {
  return (op == kG2Helmholtz || op == kG2Projection || op == kG2Convective ||
          op == kG2Gradient || op == kG2ViscousBc) ? 2 : 1;
}

// Lax-Friedrichs F*(u) . n with the own outward normal (operators.py:597-604)
__device__ __forceinline__ void g2_lf(double a0, double a1, double b0, double b1, double nx,
                                      double ny, double &F0, double &F1) {
  const double unm = a0 * nx + a1 * ny, unp = b0 * nx + b1 * ny;
  const double lam = 2.0 * fmax(fabs(unm), fabs(unp));
  F0 = 0.5 * (a0 * unm + b0 * unp) + 0.5 * lam * (a0 - b0);
  F1 = 0.5 * (a1 * unm + b1 * unp) + 0.5 * lam * (a1 - b1);
}

// threads per cell: one per quadrature point (at least one per node and per
// face point), several cells per CTA; shared arrays sized for (N, NQ)
template <int N, int NQ>
struct G2Cfg {
  static constexpr int NP = N * N, QP = NQ * NQ;
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  static constexpr int TPC = mx(mx(QP, NP), 4 * NQ);
  static constexpr int CPB = TPC >= 128 ? 1 : 128 / TPC;
  static constexpr int THREADS = CPB * TPC;
};

template <int N, int NQ>
__global__ void __launch_bounds__(G2Cfg<N, NQ>::THREADS)
g2_kernel(const double *__restrict__ src, double *__restrict__ dst, const G2Geo g,
          const __grid_constant__ G2Tab T, const __grid_constant__ G2Params prm) {
  using C = G2Cfg<N, NQ>;
  constexpr int TPC = C::TPC, CPB = C::CPB, NP = C::NP, QP = C::QP;
  const int op = prm.op;
  const int nci = g2_nci(op), nco = g2_nco(op);
  const int64_t nc = g.ncells;
  __shared__ double su[CPB][3][NP];
  __shared__ double sq[CPB][2][3][QP];         // [comp][value | ref-x | ref-y test]
  __shared__ double sf[CPB][4][2][3][NQ];      // [slot][comp][value | ref-x | ref-y]
  const int cs = threadIdx.x / TPC, t = threadIdx.x % TPC;
  const int64_t e = (int64_t)blockIdx.x * CPB + cs;
  const bool valid = e < nc;
  const bool bdata = op == kG2GpDirichlet || op == kG2ViscousBc || op == kG2PressureNeumann;
  const int nlev = (op == kG2Convective || op == kG2PressureNeumann) ? prm.n_hist : 1;
  const bool faces = bdata || op == kG2Laplace || op == kG2LaplaceLocal ||
                     (op == kG2Helmholtz && prm.nu != 0.0) ||
                     (op == kG2Projection && prm.tau_c != nullptr) || op == kG2Convective ||
                     ((op == kG2Divergence || op == kG2Gradient) && prm.form != 0);

  for (int i = t; i < 2 * 3 * QP; i += TPC) (&sq[cs][0][0][0])[i] = 0.0;
  for (int i = t; i < 4 * 2 * 3 * NQ; i += TPC) (&sf[cs][0][0][0][0])[i] = 0.0;

  for (int lev = 0; lev < nlev; ++lev) {
    const bool hist = op == kG2Convective || op == kG2PressureNeumann;
    const double *in = hist ? prm.hist[lev] : src;
    const double beta = hist ? prm.beta[lev] : 1.0;
    __syncthreads();
    for (int i = t; i < nci * NP; i += TPC) {
      const int c = i / NP, o = i % NP;
      double v = 0.0;
      if (valid) {
        if (op == kG2LaplaceLocal && prm.local_node >= 0) v = (o == prm.local_node) ? 1.0 : 0.0;
        else if (c == 2) v = prm.vort[lev][e * NP + o];  // pressure Neumann: vorticity
        else v = in[((int64_t)c * nc + e) * NP + o];
      }
      su[cs][c][o] = v;
    }
    __syncthreads();

    if (op == kG2InvMass) {
      // S^-1 diag(1/JxW) S^-T (kernels.py:95-107): Q = (Si^T x Si^T) R / JxW
      const double *u = su[cs][0];
      for (int i = t; i < QP; i += TPC) {
        const int qx = i % NQ, qy = i / NQ;
        double a = 0.0;
        for (int j = 0; j < N; ++j) {
          double b = 0.0;
          for (int l = 0; l < N; ++l) b = fma(u[j * N + l], T.Si[l * N + qx], b);
          a = fma(T.Si[j * N + qy], b, a);
        }
        sq[cs][0][0][i] = valid ? a / g.jxw[e * QP + i] : 0.0;
      }
      __syncthreads();
      for (int i = t; i < NP; i += TPC) {
        const int x = i % N, y = i / N;
        double a = 0.0;
        for (int qy = 0; qy < NQ; ++qy) {
          double b = 0.0;
          for (int qx = 0; qx < NQ; ++qx) b = fma(sq[cs][0][0][qy * NQ + qx], T.Si[x * N + qx], b);
          a = fma(T.Si[y * N + qy], b, a);
        }
        if (valid) dst[e * NP + i] = a;
      }
      return;
    }

    // ---- volume: test data at the quadrature points ---------------------------
    for (int i = t; i < (bdata ? 0 : QP); i += TPC) {
      const int qx = i % NQ, qy = i / NQ;
      double v[3] = {0.0, 0.0, 0.0}, px[3] = {0.0, 0.0, 0.0}, py[3] = {0.0, 0.0, 0.0};
      double jw = 0.0, j00 = 0.0, j01 = 0.0, j10 = 0.0, j11 = 0.0;
      if (valid) {
        jw = g.jxw[e * QP + i];
        const double *J = g.jit + e * 4 * QP + i;
        j00 = J[0];
        j01 = J[QP];
        j10 = J[2 * QP];
        j11 = J[3 * QP];
      }
      for (int c = 0; c < nci; ++c) {
        const double *u = su[cs][c];
        double vv = 0.0, gx = 0.0, gy = 0.0;
        for (int j = 0; j < N; ++j) {
          double sv = 0.0, dv = 0.0;
          for (int l = 0; l < N; ++l) {
            sv = fma(T.S[qx * N + l], u[j * N + l], sv);
            dv = fma(T.D[qx * N + l], u[j * N + l], dv);
          }
          vv = fma(T.S[qy * N + j], sv, vv);
          gx = fma(T.S[qy * N + j], dv, gx);
          gy = fma(T.D[qy * N + j], sv, gy);
        }
        v[c] = vv;
        px[c] = j00 * gx + j01 * gy;  // _phys_grad_vol (operators.py:137-140)
        py[c] = j10 * gx + j11 * gy;
      }
      // value test VT[a] and physical gradient test (dx[a], dy[a])
      double VT[2] = {0.0, 0.0}, dx[2] = {0.0, 0.0}, dy[2] = {0.0, 0.0};
      switch (op) {
        case kG2Mass:
          VT[0] = v[0] * jw;
          break;
        case kG2Laplace:
        case kG2LaplaceLocal:
          dx[0] = px[0] * jw;
          dy[0] = py[0] * jw;
          break;
        case kG2Helmholtz: {  // operators.py:423-437
          const double e01 = prm.nu * (py[0] + px[1]);
          const double t00 = (2.0 * prm.nu * px[0]) * jw, t01 = e01 * jw;
          const double t11 = (2.0 * prm.nu * py[1]) * jw;
          dx[0] = t00;
          dy[0] = t01;
          dx[1] = t01;
          dy[1] = t11;
          VT[0] = prm.gamma0_dt * v[0] * jw;
          VT[1] = prm.gamma0_dt * v[1] * jw;
          break;
        }
        case kG2Projection:  // operators.py:381-395
          VT[0] = v[0] * jw;
          VT[1] = v[1] * jw;
          if (prm.tau_d) {
            const double s = valid ? (prm.tau_d[e] * (px[0] + py[1])) * jw : 0.0;
            dx[0] = s;
            dy[1] = s;
          }
          break;
        case kG2Convective: {  // operators.py:545-552, 588-591
          const double t00 = v[0] * v[0] * jw, t01 = v[0] * v[1] * jw, t11 = v[1] * v[1] * jw;
          dx[0] = beta * t00;
          dy[0] = beta * t01;
          dx[1] = beta * t01;
          dy[1] = beta * t11;
          if (lev == 0 && prm.body && valid) {
            VT[0] = prm.body[e * QP + i] * jw;
            VT[1] = prm.body[(nc + e) * QP + i] * jw;
          }
          break;
        }
        case kG2Divergence:  // operators.py:270-316
          if (prm.form == 1) {
            dx[0] = prm.scale * v[0] * jw;
            dy[0] = prm.scale * v[1] * jw;
          } else {
            VT[0] = -prm.scale * (px[0] + py[1]) * jw;
          }
          break;
        case kG2Gradient:  // operators.py:326-345
          if (prm.form == 1) {
            const double s = prm.scale * v[0] * jw;
            dx[0] = s;
            dy[1] = s;
          } else {
            VT[0] = -prm.scale * px[0] * jw;
            VT[1] = -prm.scale * py[0] * jw;
          }
          break;
        default:  // vorticity (operators.py:610-618)
          VT[0] = (px[1] - py[0]) * jw;
          break;
      }
      for (int a = 0; a < nco; ++a) {  // _ref_test_vol (operators.py:143-147)
        sq[cs][a][0][i] += VT[a];
        sq[cs][a][1][i] += j00 * dx[a] + j10 * dy[a];
        sq[cs][a][2][i] += j01 * dx[a] + j11 * dy[a];
      }
    }

    // ---- faces: own-frame fluxes ------------------------------------------------
    if (faces) {
      for (int i = t; i < 4 * NQ; i += TPC) {
        const int s = i / NQ, q = i % NQ;
        const int kind = valid ? prm.kind[e * 4 + s] : DG_BC_VELOCITY_DIRICHLET;
        bool active = valid;
        if (op == kG2Laplace || op == kG2LaplaceLocal) active &= kind != DG_BC_VELOCITY_DIRICHLET;
        if (op == kG2Helmholtz) active &= kind != DG_BC_VELOCITY_NEUMANN;
        if (op == kG2Projection || (op == kG2Divergence && prm.form == 2)) active &= kind == 0;
        if (op == kG2GpDirichlet) active &= kind == DG_BC_VELOCITY_NEUMANN;
        if (op == kG2ViscousBc) active &= kind != 0;
        if (op == kG2PressureNeumann) active &= kind == DG_BC_VELOCITY_DIRICHLET;
        if (!active) continue;
        const int64_t fi = (e * 4 + s) * NQ + q;
        const double sj = g.fsj[fi];
        const double nx = g.fnrm[(e * 4 + s) * 2 * NQ + q];
        const double ny = g.fnrm[(e * 4 + s) * 2 * NQ + NQ + q];
        const double *J = g.fjit + (e * 4 + s) * 4 * NQ + q;
        const double j00 = J[0], j01 = J[NQ], j10 = J[2 * NQ], j11 = J[3 * NQ];
        // own traces (value, physical gradient) of the input components
        double vo[3] = {0.0, 0.0, 0.0}, xo[3] = {0.0, 0.0, 0.0}, yo[3] = {0.0, 0.0, 0.0};
        double vn[3] = {0.0, 0.0, 0.0}, xn[3] = {0.0, 0.0, 0.0}, yn[3] = {0.0, 0.0, 0.0};
        for (int c = 0; c < nci; ++c) {
          double gx, gy;
          g2_trace(su[cs][c], N, T, s, q, vo[c], gx, gy);
          xo[c] = j00 * gx + j01 * gy;  // _phys_grad_face (operators.py:150-153)
          yo[c] = j10 * gx + j11 * gy;
        }
        int64_t en = -1;
        if (kind == 0 && !bdata) {
          en = g.nbr[e * 4 + s];
          if (en < 0) continue;  // kinds must mark boundary slots; never read outside
          if (op != kG2LaplaceLocal) {
            const int sn = g.nslot[e * 4 + s];
            const int qn = g.nflip[e * 4 + s] ? NQ - 1 - q : q;
            const double *Jn = g.fjit + (en * 4 + sn) * 4 * NQ + qn;
            for (int c = 0; c < nci; ++c) {
              double gx, gy;
              g2_trace(in + ((int64_t)c * nc + en) * NP, N, T, sn, qn, vn[c], gx, gy);
              xn[c] = Jn[0] * gx + Jn[NQ] * gy;
              yn[c] = Jn[2 * NQ] * gx + Jn[3 * NQ] * gy;
            }
          }
        }
        // value test V[a] and physical gradient test (Gx[a], Gy[a])
        double V[2] = {0.0, 0.0}, Gx[2] = {0.0, 0.0}, Gy[2] = {0.0, 0.0};
        if (op == kG2PressureNeumann) {
          // beta (div(u x u) + nu curl w), accumulated over the levels in the
          // gradient slots of side (s, q); finalised after the level loop
          const double div = xo[0] + yo[1];
          const double c0 = vo[0] * div + vo[0] * xo[0] + vo[1] * yo[0];
          const double c1 = vo[1] * div + vo[0] * xo[1] + vo[1] * yo[1];
          sf[cs][s][0][1][q] += beta * (c0 + prm.nu * yo[2]);
          sf[cs][s][0][2][q] += beta * (c1 - prm.nu * xo[2]);
          continue;
        }
        if (op == kG2GpDirichlet) {
          const double gp = prm.fdata ? prm.fdata[(e * 4 + s) * NQ + q] : 0.0;
          V[0] = 2.0 * prm.tau_scale * g.tau[e] * gp * sj;
          Gx[0] = -gp * nx * sj;
          Gy[0] = -gp * ny * sj;
        } else if (op == kG2ViscousBc) {
          const double *fd = prm.fdata ? prm.fdata + (e * 4 + s) * 3 * NQ + q : nullptr;
          const double d0 = fd ? fd[0] : 0.0, d1 = fd ? fd[NQ] : 0.0, d2 = fd ? fd[2 * NQ] : 0.0;
          if (kind == DG_BC_VELOCITY_DIRICHLET) {
            const double taub = g.tau[e] * prm.nu;
            V[0] = 2.0 * taub * d0 * sj;
            V[1] = 2.0 * taub * d1 * sj;
            const double D01 = -prm.nu * (d0 * ny + d1 * nx) * sj;
            Gx[0] = -2.0 * prm.nu * d0 * nx * sj;
            Gy[0] = D01;
            Gx[1] = D01;
            Gy[1] = -2.0 * prm.nu * d1 * ny * sj;
          } else {
            V[0] = (d0 + d2 * nx) * sj;
            V[1] = (d1 + d2 * ny) * sj;
          }
        } else if (op == kG2Laplace || op == kG2LaplaceLocal) {  // operators.py:203-233
          const double gno = nx * xo[0] + ny * yo[0];
          if (kind == 0) {
            const double gnn = nx * xn[0] + ny * yn[0];
            const double tau = prm.tau_scale * fmax(g.tau[e], g.tau[en]);
            const double jump = vo[0] - vn[0];
            V[0] = -(0.5 * (gno + gnn) - tau * jump) * sj;
            Gx[0] = -0.5 * jump * nx * sj;
            Gy[0] = -0.5 * jump * ny * sj;
          } else {
            const double taub = prm.tau_scale * g.tau[e];
            V[0] = -(gno - 2.0 * taub * vo[0]) * sj;
            Gx[0] = -vo[0] * nx * sj;
            Gy[0] = -vo[0] * ny * sj;
          }
        } else if (op == kG2Helmholtz) {  // operators.py:440-483
          const double nu = prm.nu;
          const double vo0 = nu * (2.0 * xo[0] * nx + (yo[0] + xo[1]) * ny);
          const double vo1 = nu * ((yo[0] + xo[1]) * nx + 2.0 * yo[1] * ny);
          if (kind == 0) {
            const double vn0 = nu * (2.0 * xn[0] * nx + (yn[0] + xn[1]) * ny);
            const double vn1 = nu * ((yn[0] + xn[1]) * nx + 2.0 * yn[1] * ny);
            const double tau = fmax(g.tau[e], g.tau[en]) * nu;
            const double j0 = vo[0] - vn[0], j1 = vo[1] - vn[1];
            V[0] = -(0.5 * (vo0 + vn0) - tau * j0) * sj;
            V[1] = -(0.5 * (vo1 + vn1) - tau * j1) * sj;
            const double G01 = -0.5 * nu * (j0 * ny + j1 * nx) * sj;
            Gx[0] = -nu * j0 * nx * sj;
            Gy[0] = G01;
            Gx[1] = G01;
            Gy[1] = -nu * j1 * ny * sj;
          } else {  // velocity-Dirichlet side
            const double taub = g.tau[e] * nu;
            V[0] = -(vo0 - 2.0 * taub * vo[0]) * sj;
            V[1] = -(vo1 - 2.0 * taub * vo[1]) * sj;
            const double D01 = -nu * (vo[0] * ny + vo[1] * nx) * sj;
            Gx[0] = -2.0 * nu * vo[0] * nx * sj;
            Gy[0] = D01;
            Gx[1] = D01;
            Gy[1] = -2.0 * nu * vo[1] * ny * sj;
          }
        } else if (op == kG2Projection) {  // operators.py:396-411
          const double tc = prm.tau_c[e * 4 + s];
          V[0] = tc * (vo[0] - vn[0]) * sj;
          V[1] = tc * (vo[1] - vn[1]) * sj;
        } else if (op == kG2Convective) {  // operators.py:554-586
          double F0, F1;
          if (kind == 0) {
            g2_lf(vo[0], vo[1], vn[0], vn[1], nx, ny, F0, F1);
          } else if (kind == DG_BC_VELOCITY_DIRICHLET) {
            const double *gd = prm.gdata[lev];
            const double g0 = gd ? gd[((e * 4 + s) * 2 + 0) * NQ + q] : 0.0;
            const double g1 = gd ? gd[((e * 4 + s) * 2 + 1) * NQ + q] : 0.0;
            g2_lf(vo[0], vo[1], 2 * g0 - vo[0], 2 * g1 - vo[1], nx, ny, F0, F1);
          } else {
            const double un = vo[0] * nx + vo[1] * ny;
            F0 = vo[0] * un;
            F1 = vo[1] * un;
          }
          V[0] = -beta * F0 * sj;
          V[1] = -beta * F1 * sj;
        } else if (op == kG2Divergence) {
          const double uno = vo[0] * nx + vo[1] * ny;
          const double unn = vn[0] * nx + vn[1] * ny;
          if (prm.form == 1)  // weak: -scale {u}.n (boundary: own trace)
            V[0] = -prm.scale * (kind == 0 ? 0.5 * (uno + unn) : uno) * sj;
          else                // strong: +scale [u].n / 2, interior only
            V[0] = prm.scale * 0.5 * (uno - unn) * sj;
        } else {  // weak pressure gradient: -scale {p} n (boundary: own trace)
          const double pav = kind == 0 ? 0.5 * (vo[0] + vn[0]) : vo[0];
          V[0] = -prm.scale * pav * nx * sj;
          V[1] = -prm.scale * pav * ny * sj;
        }
        for (int a = 0; a < nco; ++a) {  // _ref_test_face (operators.py:156-159)
          sf[cs][s][a][0][q] += V[a];
          sf[cs][s][a][1][q] += j00 * Gx[a] + j10 * Gy[a];
          sf[cs][s][a][2][q] += j01 * Gx[a] + j11 * Gy[a];
        }
      }
    }
  }
  __syncthreads();
  if (op == kG2PressureNeumann) {  // V = -((dg/dt - f + hp) . n) sJxW (operators.py:657-669)
    for (int i = t; i < 4 * NQ; i += TPC) {
      const int s = i / NQ, q = i % NQ;
      double V = 0.0;
      if (valid && prm.kind[e * 4 + s] == DG_BC_VELOCITY_DIRICHLET) {
        const int64_t fi = (e * 4 + s) * NQ + q;
        const double nx = g.fnrm[(e * 4 + s) * 2 * NQ + q];
        const double ny = g.fnrm[(e * 4 + s) * 2 * NQ + NQ + q];
        double h0 = sf[cs][s][0][1][q], h1 = sf[cs][s][0][2][q];
        if (prm.fdata) {
          h0 = prm.fdata[((e * 4 + s) * 2 + 0) * NQ + q] + h0;
          h1 = prm.fdata[((e * 4 + s) * 2 + 1) * NQ + q] + h1;
        }
        V = -(h0 * nx + h1 * ny) * g.fsj[fi];
      }
      sf[cs][s][0][0][q] = V;
      sf[cs][s][0][1][q] = 0.0;
      sf[cs][s][0][2][q] = 0.0;
    }
    __syncthreads();
  }

  // ---- tests: volume integrate + face lifts (kernels.py:86-92, 159-186) -------
  for (int i = t; i < nco * NP; i += TPC) {
    const int a = i / NP, o = i % NP;
    const int x = o % N, y = o / N;
    double acc = 0.0;
    for (int qy = 0; qy < NQ; ++qy) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (int qx = 0; qx < NQ; ++qx) {
        const int k = qy * NQ + qx;
        a0 = fma(T.S[qx * N + x], sq[cs][a][0][k], a0);
        a1 = fma(T.D[qx * N + x], sq[cs][a][1][k], a1);
        a2 = fma(T.S[qx * N + x], sq[cs][a][2][k], a2);
      }
      acc = fma(T.S[qy * N + y], a0 + a1, acc);
      acc = fma(T.D[qy * N + y], a2, acc);
    }
    if (faces) {
      for (int q = 0; q < NQ; ++q) {
        // slot 0 / 1 (x = -1 / +1): values at x = 0 / N-1, d/dxi via ld / rd
        const double sy = T.S[q * N + y], dyv = T.D[q * N + y];
        double v = T.ld[x] * sy * sf[cs][0][a][1][q] + T.rd[x] * sy * sf[cs][1][a][1][q];
        if (x == 0) v += sy * sf[cs][0][a][0][q] + dyv * sf[cs][0][a][2][q];
        if (x == N - 1) v += sy * sf[cs][1][a][0][q] + dyv * sf[cs][1][a][2][q];
        // slot 2 / 3 (y = -1 / +1)
        const double sx = T.S[q * N + x], dxv = T.D[q * N + x];
        v += T.ld[y] * sx * sf[cs][2][a][2][q] + T.rd[y] * sx * sf[cs][3][a][2][q];
        if (y == 0) v += sx * sf[cs][2][a][0][q] + dxv * sf[cs][2][a][1][q];
        if (y == N - 1) v += sx * sf[cs][3][a][0][q] + dxv * sf[cs][3][a][1][q];
        acc += v;
      }
    }
    if (valid && (op != kG2LaplaceLocal || prm.local_node < 0 || o == prm.local_node))
      dst[((int64_t)a * nc + e) * NP + o] = acc;
  }
}

// Multigrid transfers on a refined general mesh (reference multigrid.py:
// 33-73): child (quadrant qd = 2 dy + dx) of parent p carries the tensor
// embedding (E_dy x E_dx) of p's polynomial; restriction is its transpose,
// summed parent-centrically over the four children (fixed order, no atomics).
struct G2Emb {
  double E[2][kG2MaxN * kG2MaxN];  // E[c][q][i] = l_i(0.5 (x_q -/+ 1))
};

__global__ void g2_prolong_kernel(const double *__restrict__ xc, double *__restrict__ xf, int N,
                                  int64_t nfine, const int64_t *__restrict__ parent,
                                  const int *__restrict__ quadrant,
                                  const __grid_constant__ G2Emb T, int add) {
  const int NP = N * N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nfine * NP; i += stride) {
    const int64_t f = i / NP;
    const int o = (int)(i % NP), x = o % N, y = o / N;
    const int qd = quadrant[f], dx = qd & 1, dy = qd >> 1;
    const double *pc = xc + parent[f] * NP;
    double a = 0.0;
    for (int j = 0; j < N; ++j) {
      double b = 0.0;
      for (int l = 0; l < N; ++l) b = fma(T.E[dx][x * N + l], pc[j * N + l], b);
      a = fma(T.E[dy][y * N + j], b, a);
    }
    xf[i] = add ? xf[i] + a : a;
  }
}

__global__ void g2_restrict_kernel(const double *__restrict__ xf, double *__restrict__ xc, int N,
                                   int64_t ncoarse, const int64_t *__restrict__ children,
                                   const __grid_constant__ G2Emb T) {
  const int NP = N * N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ncoarse * NP;
       i += stride) {
    const int64_t p = i / NP;
    const int o = (int)(i % NP), il = o % N, jl = o / N;
    double acc = 0.0;
    for (int qd = 0; qd < 4; ++qd) {
      const int64_t f = children[p * 4 + qd];
      if (f < 0) continue;
      const int dx = qd & 1, dy = qd >> 1;
      const double *cf = xf + f * NP;
      double a = 0.0;
      for (int y = 0; y < N; ++y) {
        double b = 0.0;
        for (int x = 0; x < N; ++x) b = fma(T.E[dx][x * N + il], cf[y * N + x], b);
        a = fma(T.E[dy][y * N + jl], b, a);
      }
      acc += a;
    }
    xc[i] = acc;
  }
}

}  // namespace dg

