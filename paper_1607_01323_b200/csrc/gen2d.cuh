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
#pragma once
#include "common.cuh"

namespace dg {

constexpr int kG2MaxN = 8, kG2MaxQ = 11;

enum G2Op : int {
  kG2Mass = 0,
  kG2InvMass = 1,
  kG2Laplace = 2,
  kG2LaplaceLocal = 3,  // neighbour traces zeroed (block-diagonal part)
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
  double tau_scale;
  const int *kind;        // [e][4]: 0 interior, DG_BC_VELOCITY_DIRICHLET / _NEUMANN
  int local_node;         // kG2LaplaceLocal: unit vector at this node (-1: use src)
};

// value and reference gradient of a cell field at face point q of slot s
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

template <int CPB>
__global__ void __launch_bounds__(64 * CPB)
g2_kernel(const double *__restrict__ src, double *__restrict__ dst, const G2Geo g,
          const __grid_constant__ G2Tab T, const G2Params prm) {
  constexpr int TPC = 64;
  const int N = g.n, NQ = g.nq, NP = N * N, QP = NQ * NQ;
  __shared__ double su[CPB][kG2MaxN * kG2MaxN];
  __shared__ double sq[CPB][3][kG2MaxQ * kG2MaxQ];
  __shared__ double sf[CPB][4][3][kG2MaxQ];
  const int cs = threadIdx.x / TPC, t = threadIdx.x % TPC;
  const int64_t e = (int64_t)blockIdx.x * CPB + cs;
  const bool valid = e < g.ncells;
  const int op = prm.op;
  for (int i = t; i < NP; i += TPC) {
    double v = 0.0;
    if (valid) {
      if (op == kG2LaplaceLocal && prm.local_node >= 0) v = (i == prm.local_node) ? 1.0 : 0.0;
      else v = src[e * NP + i];
    }
    su[cs][i] = v;
  }
  __syncthreads();
  const double *u = su[cs];

  if (op == kG2InvMass) {
    // S^-1 diag(1/JxW) S^-T (kernels.py:95-107): Q = (Si^T x Si^T) R / JxW
    for (int i = t; i < QP; i += TPC) {
      const int qx = i % NQ, qy = i / NQ;
      double a = 0.0;
      for (int j = 0; j < N; ++j) {
        double b = 0.0;
        for (int l = 0; l < N; ++l) b = fma(u[j * N + l], T.Si[l * N + qx], b);
        a = fma(T.Si[j * N + qy], b, a);
      }
      sq[cs][0][i] = valid ? a / g.jxw[e * QP + i] : 0.0;
    }
    __syncthreads();
    for (int i = t; i < NP; i += TPC) {
      const int x = i % N, y = i / N;
      double a = 0.0;
      for (int qy = 0; qy < NQ; ++qy) {
        double b = 0.0;
        for (int qx = 0; qx < NQ; ++qx) b = fma(sq[cs][0][qy * NQ + qx], T.Si[x * N + qx], b);
        a = fma(T.Si[y * N + qy], b, a);
      }
      if (valid) dst[e * NP + i] = a;
    }
    return;
  }

  // ---- volume: data at the quadrature points --------------------------------
  for (int i = t; i < QP; i += TPC) {
    const int qx = i % NQ, qy = i / NQ;
    double v = 0.0, gx = 0.0, gy = 0.0;
    for (int j = 0; j < N; ++j) {
      double sv = 0.0, dv = 0.0;
      for (int l = 0; l < N; ++l) {
        sv = fma(T.S[qx * N + l], u[j * N + l], sv);
        dv = fma(T.D[qx * N + l], u[j * N + l], dv);
      }
      v = fma(T.S[qy * N + j], sv, v);
      gx = fma(T.S[qy * N + j], dv, gx);
      gy = fma(T.D[qy * N + j], sv, gy);
    }
    double r0 = 0.0, r1 = 0.0, vt = 0.0;
    if (valid) {
      const double jw = g.jxw[e * QP + i];
      if (op == kG2Mass) {
        vt = v * jw;
      } else {  // Laplace: (grad q, grad p) (operators.py:199-201)
        const double *J = g.jit + e * 4 * QP + i;
        const double j00 = J[0], j01 = J[QP], j10 = J[2 * QP], j11 = J[3 * QP];
        const double px = j00 * gx + j01 * gy, py = j10 * gx + j11 * gy;
        const double dx = px * jw, dy = py * jw;
        r0 = j00 * dx + j10 * dy;
        r1 = j01 * dx + j11 * dy;
      }
    }
    sq[cs][0][i] = vt;
    sq[cs][1][i] = r0;
    sq[cs][2][i] = r1;
  }

  // ---- faces (Laplace): own-frame SIP fluxes (operators.py:203-236) ----------
  const bool faces = op == kG2Laplace || op == kG2LaplaceLocal;
  if (faces) {
    for (int i = t; i < 4 * NQ; i += TPC) {
      const int s = i / NQ, q = i % NQ;
      double V = 0.0, R0 = 0.0, R1 = 0.0;
      // velocity-Dirichlet sides carry no pressure term (operators.py:189-193)
      const int kind = valid ? prm.kind[e * 4 + s] : DG_BC_VELOCITY_DIRICHLET;
      if (valid && kind != DG_BC_VELOCITY_DIRICHLET) {
        const int64_t fi = (e * 4 + s) * NQ + q;
        const double sj = g.fsj[fi];
        const double nx = g.fnrm[(e * 4 + s) * 2 * NQ + q], ny = g.fnrm[(e * 4 + s) * 2 * NQ + NQ + q];
        const double *J = g.fjit + (e * 4 + s) * 4 * NQ + q;
        const double j00 = J[0], j01 = J[NQ], j10 = J[2 * NQ], j11 = J[3 * NQ];
        double vo, gxo, gyo;
        g2_trace(u, N, T, s, q, vo, gxo, gyo);
        const double gno = nx * (j00 * gxo + j01 * gyo) + ny * (j10 * gxo + j11 * gyo);
        double Gx, Gy;
        if (kind == 0) {
          const int64_t en = g.nbr[e * 4 + s];
          const int sn = g.nslot[e * 4 + s];
          const int qn = g.nflip[e * 4 + s] ? NQ - 1 - q : q;
          double vn = 0.0, gxn = 0.0, gyn = 0.0, gnn = 0.0;
          if (op == kG2Laplace) {
            g2_trace(src + en * NP, N, T, sn, qn, vn, gxn, gyn);
            const double *Jn = g.fjit + (en * 4 + sn) * 4 * NQ + qn;
            // neighbour gradient in the own outward normal direction
            gnn = nx * (Jn[0] * gxn + Jn[NQ] * gyn) + ny * (Jn[2 * NQ] * gxn + Jn[3 * NQ] * gyn);
          }
          const double tau = prm.tau_scale * fmax(g.tau[e], g.tau[en]);
          const double jump = vo - vn;
          V = -(0.5 * (gno + gnn) - tau * jump) * sj;
          Gx = -0.5 * jump * nx * sj;
          Gy = -0.5 * jump * ny * sj;
        } else {  // velocity-Neumann = pressure-Dirichlet side (operators.py:227-233)
          const double taub = prm.tau_scale * g.tau[e];
          V = -(gno - 2.0 * taub * vo) * sj;
          Gx = -vo * nx * sj;
          Gy = -vo * ny * sj;
        }
        R0 = j00 * Gx + j10 * Gy;
        R1 = j01 * Gx + j11 * Gy;
      }
      sf[cs][s][0][q] = V;
      sf[cs][s][1][q] = R0;
      sf[cs][s][2][q] = R1;
    }
  }
  __syncthreads();

  // ---- tests: volume integrate + face lifts (kernels.py:86-92, 159-186) -------
  for (int i = t; i < NP; i += TPC) {
    const int x = i % N, y = i / N;
    double acc = 0.0;
    for (int qy = 0; qy < NQ; ++qy) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (int qx = 0; qx < NQ; ++qx) {
        const int k = qy * NQ + qx;
        a0 = fma(T.S[qx * N + x], sq[cs][0][k], a0);
        a1 = fma(T.D[qx * N + x], sq[cs][1][k], a1);
        a2 = fma(T.S[qx * N + x], sq[cs][2][k], a2);
      }
      acc = fma(T.S[qy * N + y], a0 + a1, acc);
      acc = fma(T.D[qy * N + y], a2, acc);
    }
    if (faces) {
      for (int q = 0; q < NQ; ++q) {
        // slot 0 / 1 (x = -1 / +1): values at x = 0 / N-1, d/dxi via ld / rd
        const double sy = T.S[q * N + y], dy = T.D[q * N + y];
        double a = T.ld[x] * sy * sf[cs][0][1][q] + T.rd[x] * sy * sf[cs][1][1][q];
        if (x == 0) a += sy * sf[cs][0][0][q] + dy * sf[cs][0][2][q];
        if (x == N - 1) a += sy * sf[cs][1][0][q] + dy * sf[cs][1][2][q];
        // slot 2 / 3 (y = -1 / +1)
        const double sx = T.S[q * N + x], dx = T.D[q * N + x];
        a += T.ld[y] * sx * sf[cs][2][2][q] + T.rd[y] * sx * sf[cs][3][2][q];
        if (y == 0) a += sx * sf[cs][2][0][q] + dx * sf[cs][2][1][q];
        if (y == N - 1) a += sx * sf[cs][3][0][q] + dx * sf[cs][3][1][q];
        acc += a;
      }
    }
    if (valid && (op != kG2LaplaceLocal || prm.local_node < 0 || i == prm.local_node))
      dst[e * NP + i] = acc;
  }
}

}  // namespace dg
