// Vector-valued DG operators on Cartesian cells, fp64, sm_100a:
//   viscous Helmholtz   (reference operators.py:418-491)
//   projection M + tau_D div-div + tau_C jump   (operators.py:372-412)
//   convective term with local Lax-Friedrichs flux (operators.py:533-604)
//
// Quadrature-point formulation mirroring the reference: per cell, values and
// reference gradients at the tensor Gauss points by sum factorisation, the
// pointwise physics, then the adjoint contractions; face terms are evaluated
// cell-centrically in the "own cell" frame (own outward normal, jump =
// own - neighbour), which reproduces the reference's minus/plus scatter
// (spaces.py:151-163) with each output DoF written once, no atomics.
//
// One CTA per cell.  Neighbour cells are read from global memory (L2) into
// shared memory one face at a time.
#pragma once
#include "common.cuh"

namespace dg {

enum VecOp : int { kOpHelmholtz = 0, kOpProjection = 1, kOpConvective = 2 };

constexpr int kMaxHist = 4;

struct VecParams {
  int op;
  double gamma0_dt, nu;          // Helmholtz
  const double *tau_d;           // projection: per cell (or null)
  const double *tau_c;           // projection: [d*ncell + e] face e|e+d (or null)
  int n_hist;                    // convective
  const double *hist[kMaxHist];
  double beta[kMaxHist];
};

template <int N, int NQ>
struct QuadTab {
  double S[NQ * N];   // S[q][i] = l_i(x_q)
  double D[NQ * N];   // D[q][i] = l_i'(x_q)
  double w[NQ];       // Gauss weights
  double dL[N], dR[N];
};

template <int DIM, int N, int NQ, int NC>
struct VecCfg {
  static constexpr int NP = DIM == 3 ? N * N * N : N * N;
  static constexpr int QP = DIM == 3 ? NQ * NQ * NQ : NQ * NQ;
  static constexpr int FQ = DIM == 3 ? NQ * NQ : NQ;  // face points
  static constexpr int FN = DIM == 3 ? N * N : N;     // face nodes
  static constexpr int MX = (N > NQ ? N : NQ);
  static constexpr int BIG = DIM == 3 ? MX * MX * MX : MX * MX;
  static constexpr int THREADS = QP >= 256 ? 256 : 128;
  // shared layout (doubles)
  static constexpr int U = 0;                       // own cell, NC * NP
  static constexpr int NB = U + NC * NP;            // neighbour cell, NC * NP
  static constexpr int OUT = NB + NC * NP;          // accumulator, NC * NP
  static constexpr int QV = OUT + NC * NP;          // values at q points, NC * QP
  static constexpr int QG = QV + NC * QP;           // phys gradients, NC * DIM * QP
  static constexpr int T0 = QG + NC * DIM * QP;     // temporaries, 3 * BIG
  static constexpr int T1 = T0 + BIG;
  static constexpr int T2 = T1 + BIG;
  static constexpr int TG = T2 + BIG;               // test data, DIM * QP
  static constexpr int FO = TG + DIM * QP;          // own face traces NC*(1+DIM)*FQ
  static constexpr int FB = FO + NC * (1 + DIM) * FQ;  // neighbour traces
  static constexpr int FV = FB + NC * (1 + DIM) * FQ;  // face test data NC*(1+DIM)*FQ
  static constexpr int FT = FV + NC * (1 + DIM) * FQ;  // face temporaries 2*BIG
  static constexpr int TAB = FT + 2 * BIG;             // tables S, D, ST(N x NQ), DT
  static constexpr int NDBL = TAB + 4 * NQ * N + NQ + 2 * N;
  static constexpr size_t SMEM = sizeof(double) * NDBL;
};

// Generic contraction along axis A of a [e2][e1][e0] array (x = axis 0
// fastest): out[..r..] = sum_c T[r*ldc + c] in[..c..].  T is R x Cc.
__device__ __forceinline__ void contract(const double *in, double *out, const double *T, int R,
                                         int Cc, int A, int e0, int e1, int e2) {
  int o0 = e0, o1 = e1, o2 = e2;
  if (A == 0) o0 = R; else if (A == 1) o1 = R; else o2 = R;
  const int tot = o0 * o1 * o2;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) {
    const int x = i % o0, y = (i / o0) % o1, z = i / (o0 * o1);
    int r, base, stride;
    if (A == 0) { r = x; base = (z * e1 + y) * e0; stride = 1; }
    else if (A == 1) { r = y; base = z * e1 * e0 + x; stride = e0; }
    else { r = z; base = y * e0 + x; stride = e0 * e1; }
    double acc = 0.0;
    for (int c = 0; c < Cc; ++c) acc += T[r * Cc + c] * in[base + c * stride];
    out[i] = acc;
  }
  __syncthreads();
}

template <int DIM, int N, int NQ, int NC>
__global__ void __launch_bounds__(VecCfg<DIM, N, NQ, NC>::THREADS)
vecop_kernel(const double *__restrict__ u, double *__restrict__ out, const Geo g,
             const QuadTab<N, NQ> tab, const VecParams prm, const int64_t ncells) {
  using C = VecCfg<DIM, N, NQ, NC>;
  constexpr int NP = C::NP, QP = C::QP, FQ = C::FQ;
  extern __shared__ double sm[];
  double *su = sm + C::U, *snb = sm + C::NB, *sout = sm + C::OUT;
  double *qv = sm + C::QV, *qg = sm + C::QG;
  double *t0 = sm + C::T0, *t1 = sm + C::T1, *t2 = sm + C::T2, *tg = sm + C::TG;
  double *fo = sm + C::FO, *fb = sm + C::FB, *fv = sm + C::FV, *ft = sm + C::FT;
  double *S = sm + C::TAB, *D = S + NQ * N, *ST = D + NQ * N, *DT = ST + NQ * N;
  double *W = DT + NQ * N, *dL = W + NQ, *dR = dL + N;
  const int tid = threadIdx.x;
  const int64_t e = blockIdx.x;
  const int ix = (int)(e % g.nx), iy = (int)((e / g.nx) % g.ny), iz = (int)(e / ((int64_t)g.nx * g.ny));
  double h[3] = {g.hx[ix], g.hy[iy], DIM == 3 ? g.hz[iz] : 2.0};
  double det = 0.125 * h[0] * h[1] * h[2];
  if (DIM == 2) det = 0.25 * h[0] * h[1];

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
  for (int i = tid; i < NC * NP; i += blockDim.x) sout[i] = 0.0;
  __syncthreads();

  const int nlev = prm.op == kOpConvective ? prm.n_hist : 1;
  const int e0 = N, e1 = N, e2 = DIM == 3 ? N : 1;
  const int q0 = NQ, q1 = NQ, q2 = DIM == 3 ? NQ : 1;
  auto wq = [&](int i) {  // tensor weight * det at q point i
    const int x = i % NQ, y = (i / NQ) % NQ, z = DIM == 3 ? i / (NQ * NQ) : 0;
    return det * W[x] * W[y] * (DIM == 3 ? W[z] : 1.0);
  };

  for (int lev = 0; lev < nlev; ++lev) {
    const double *src = prm.op == kOpConvective ? prm.hist[lev] : u;
    const double beta = prm.op == kOpConvective ? prm.beta[lev] : 1.0;
    for (int i = tid; i < NC * NP; i += blockDim.x) {
      const int c = i / NP, o = i % NP;
      su[i] = src[((int64_t)c * ncells + e) * NP + o];
    }
    __syncthreads();
    // ---- volume: values and physical gradients at q points ---------------
    for (int c = 0; c < NC; ++c) {
      const double *uc = su + c * NP;
      double *val = qv + c * QP;
      // values: S along x, y, z ; gradients as in kernels.py:66-79
      contract(uc, t0, S, NQ, N, 0, e0, e1, e2);                 // [z][y][qx]
      if (DIM == 3) {
        contract(t0, t1, S, NQ, N, 1, q0, e1, e2);               // [z][qy][qx]
        contract(t1, val, S, NQ, N, 2, q0, q1, e2);              // values
        contract(t1, qg + (c * DIM + 2) * QP, D, NQ, N, 2, q0, q1, e2);  // d/dz
        contract(t0, t2, D, NQ, N, 1, q0, e1, e2);
        contract(t2, qg + (c * DIM + 1) * QP, S, NQ, N, 2, q0, q1, e2);  // d/dy
        contract(uc, t0, D, NQ, N, 0, e0, e1, e2);
        contract(t0, t1, S, NQ, N, 1, q0, e1, e2);
        contract(t1, qg + (c * DIM + 0) * QP, S, NQ, N, 2, q0, q1, e2);  // d/dx
      } else {
        contract(t0, val, S, NQ, N, 1, q0, e1, 1);
        contract(t0, qg + (c * DIM + 1) * QP, D, NQ, N, 1, q0, e1, 1);
        contract(uc, t0, D, NQ, N, 0, e0, e1, 1);
        contract(t0, qg + (c * DIM + 0) * QP, S, NQ, N, 1, q0, e1, 1);
      }
    }
    // reference -> physical gradients
    for (int i = tid; i < NC * DIM * QP; i += blockDim.x) {
      const int d = (i / QP) % DIM;
      qg[i] *= 2.0 / h[d];
    }
    __syncthreads();
    // ---- volume physics + adjoint integration per output component ---------
    for (int a = 0; a < NC; ++a) {
      // gradient-test data tg[b] (physical) and value-test data (in t2)
      for (int i = tid; i < QP; i += blockDim.x) {
        const double jw = wq(i);
        double vt = 0.0;
        if (prm.op == kOpHelmholtz) {
          vt = prm.gamma0_dt * qv[a * QP + i] * jw;
          for (int b = 0; b < DIM; ++b)
            tg[b * QP + i] = prm.nu * (qg[(a * DIM + b) * QP + i] + qg[(b * DIM + a) * QP + i]) * jw;
        } else if (prm.op == kOpProjection) {
          vt = qv[a * QP + i] * jw;
          double div = 0.0;
          for (int b = 0; b < DIM; ++b) div += qg[(b * DIM + b) * QP + i];
          const double td = prm.tau_d ? prm.tau_d[e] : 0.0;
          for (int b = 0; b < DIM; ++b) tg[b * QP + i] = (b == a) ? td * div * jw : 0.0;
        } else {
          for (int b = 0; b < DIM; ++b) tg[b * QP + i] = beta * qv[a * QP + i] * qv[b * QP + i] * jw;
        }
        t2[i] = vt;
      }
      __syncthreads();
      // integrate: value test (S^T along all axes) + gradient tests
      double *oa = sout + a * NP;
      auto accumulate = [&](const double *res) {
        for (int i = tid; i < NP; i += blockDim.x) oa[i] += res[i];
        __syncthreads();
      };
      if (prm.op != kOpConvective) {
        if (DIM == 3) {
          contract(t2, t0, ST, N, NQ, 0, q0, q1, q2);
          contract(t0, t1, ST, N, NQ, 1, e0, q1, q2);
          contract(t1, t0, ST, N, NQ, 2, e0, e1, q2);
        } else {
          contract(t2, t1, ST, N, NQ, 0, q0, q1, 1);
          contract(t1, t0, ST, N, NQ, 1, e0, q1, 1);
        }
        accumulate(t0);
      }
      for (int b = 0; b < DIM; ++b) {
        // phys test: (2/h_b) * reference gradient test along b
        const double sc = 2.0 / h[b];
        const double *gb = tg + b * QP;
        if (DIM == 3) {
          contract(gb, t0, b == 0 ? DT : ST, N, NQ, 0, q0, q1, q2);
          contract(t0, t1, b == 1 ? DT : ST, N, NQ, 1, e0, q1, q2);
          contract(t1, t0, b == 2 ? DT : ST, N, NQ, 2, e0, e1, q2);
        } else {
          contract(gb, t1, b == 0 ? DT : ST, N, NQ, 0, q0, q1, 1);
          contract(t1, t0, b == 1 ? DT : ST, N, NQ, 1, e0, q1, 1);
        }
        for (int i = tid; i < NP; i += blockDim.x) oa[i] += sc * t0[i];
        __syncthreads();
      }
    }
    // ---- faces ------------------------------------------------------------
    const bool faces = (prm.op == kOpHelmholtz && prm.nu != 0.0) ||
                       (prm.op == kOpProjection && prm.tau_c != nullptr) ||
                       prm.op == kOpConvective;
    if (!faces) continue;
    for (int side = 0; side < 2 * DIM; ++side) {
      const int d = side >> 1, s = side & 1;
      // neighbour resolution (no x-slab ghosts for vector operators)
      const int nd = d == 0 ? g.nx : (d == 1 ? g.ny : g.nz);
      const int cd = d == 0 ? ix : (d == 1 ? iy : iz);
      int nidx = cd + (s ? 1 : -1);
      int kind = 0;  // 0 interior, 2 velocity-Dirichlet, 3 velocity-Neumann
      if (nidx < 0 || nidx >= nd) {
        const int m = g.mode[side];
        if (m == kWrap) nidx = s ? 0 : nd - 1;
        else kind = m;  // kBndNone (velocity-Dirichlet) / kBndNeumann
      }
      int64_t en = e;
      double hn = h[d];
      if (kind == 0) {
        const int cx = d == 0 ? nidx : ix, cy = d == 1 ? nidx : iy, cz = d == 2 ? nidx : iz;
        en = cx + (int64_t)g.nx * (cy + (int64_t)g.ny * cz);
        hn = d == 0 ? g.hx[nidx] : (d == 1 ? g.hy[nidx] : g.hz[nidx]);
      }
      // projection: jump penalty only on interior faces; Helmholtz: nothing on
      // velocity-Neumann faces; convective: all faces
      if (prm.op == kOpProjection && kind != 0) continue;
      if (prm.op == kOpHelmholtz && kind == kBndNeumann) continue;
      if (kind == 0)
        for (int i = tid; i < NC * NP; i += blockDim.x) {
          const int c = i / NP, o = i % NP;
          snb[i] = src[((int64_t)c * ncells + en) * NP + o];
        }
      __syncthreads();
      // traces: [c][0] value, [c][1+b] physical gradient component b
      auto traces = [&](const double *cell, int send, double *dst) {
        // end layer / derivative layer along d -> face nodes (FN), then S/D on
        // tangential axes.  Layers are stored [slow][fast] over the
        // tangential node indices in increasing axis order (z,y,x minus d).
        for (int c = 0; c < NC; ++c) {
          const double *cc = cell + c * NP;
          // layer buffers in ft: val layer (FN) at ft, deriv layer at ft+C::BIG
          for (int i = tid; i < C::FN; i += blockDim.x) {
            const int sl = DIM == 3 ? i / N : 0, fa = DIM == 3 ? i % N : i;
            double vv = 0.0, dd = 0.0;
            for (int k = 0; k < N; ++k) {
              int idx;
              if (DIM == 3) {
                if (d == 0) idx = (sl * N + fa) * N + k;         // (z,y) fixed, x=k
                else if (d == 1) idx = (sl * N + k) * N + fa;    // (z,x) fixed, y=k
                else idx = (k * N + sl) * N + fa;                // (y,x) fixed, z=k
              } else {
                idx = d == 0 ? fa * N + k : k * N + fa;
              }
              const double x = cc[idx];
              if (k == (send ? N - 1 : 0)) vv = x;
              dd += (send ? dR[k] : dL[k]) * x;
            }
            ft[i] = vv;
            ft[C::BIG + i] = dd;
          }
          __syncthreads();
          // tangential contractions: value (S,S), normal deriv (S,S),
          // tangential derivs (D on one axis)
          double *dv = dst + (c * (1 + DIM)) * FQ;
          if (DIM == 3) {
            // fast axis first then slow axis; face arrays [slow][fast]
            contract(ft, t0, S, NQ, N, 0, N, N, 1);
            contract(t0, dv, S, NQ, N, 1, NQ, N, 1);                       // value
            contract(ft + C::BIG, t1, S, NQ, N, 0, N, N, 1);
            contract(t1, dv + (1 + d) * FQ, S, NQ, N, 1, NQ, N, 1);       // normal
            // tangential directions: fast axis dir tfa, slow axis dir tsl
            const int tfa = d == 0 ? 1 : 0, tsl = d == 2 ? 1 : 2;
            contract(ft, t2, D, NQ, N, 0, N, N, 1);
            contract(t2, dv + (1 + tfa) * FQ, S, NQ, N, 1, NQ, N, 1);     // d/d fast
            contract(t0, dv + (1 + tsl) * FQ, D, NQ, N, 1, NQ, N, 1);     // d/d slow
          } else {
            contract(ft, dv, S, NQ, N, 0, N, 1, 1);
            contract(ft + C::BIG, dv + (1 + d) * FQ, S, NQ, N, 0, N, 1, 1);
            contract(ft, dv + (1 + (1 - d)) * FQ, D, NQ, N, 0, N, 1, 1);
          }
          for (int i = tid; i < DIM * FQ; i += blockDim.x) {
            const int b = i / FQ;
            dv[(1 + b) * FQ + (i % FQ)] *= 2.0 / h[b];
          }
          __syncthreads();
        }
      };
      traces(su, s, fo);
      if (kind == 0) {
        // traces() scales by 2/h[b]; the neighbour differs only along d
        const double hsave = h[d];
        h[d] = hn;
        traces(snb, 1 - s, fb);
        h[d] = hsave;
      }
      // face weights: prod tangential (h/2) * w w
      double fdet = 1.0;
      for (int b = 0; b < DIM; ++b)
        if (b != d) fdet *= 0.5 * h[b];
      const double nsgn = s ? 1.0 : -1.0;  // own outward normal = nsgn e_d
      double tau = 0.0;
      if (prm.op == kOpHelmholtz) {
        const double te = g.tau[e];
        tau = (kind == 0 ? fmax(te, g.tau[en]) : te) * prm.nu;
      } else if (prm.op == kOpProjection) {
        // tau_c of the face between the lower cell and its +d neighbour
        tau = prm.tau_c[(int64_t)d * ncells + (s ? e : en)];
      }
      for (int i = tid; i < FQ; i += blockDim.x) {
        const int fa = DIM == 3 ? i % NQ : i, sl = DIM == 3 ? i / NQ : 0;
        const double sj = fdet * W[fa] * (DIM == 3 ? W[sl] : 1.0);
        double uo[NC], un[NC], go[NC][DIM], gn[NC][DIM];
        for (int c = 0; c < NC; ++c) {
          uo[c] = fo[(c * (1 + DIM)) * FQ + i];
          un[c] = kind == 0 ? fb[(c * (1 + DIM)) * FQ + i] : 0.0;
          for (int b = 0; b < DIM; ++b) {
            go[c][b] = fo[(c * (1 + DIM) + 1 + b) * FQ + i];
            gn[c][b] = kind == 0 ? fb[(c * (1 + DIM) + 1 + b) * FQ + i] : 0.0;
          }
        }
        double V[NC], G[NC][DIM];
        for (int c = 0; c < NC; ++c) {
          V[c] = 0.0;
          for (int b = 0; b < DIM; ++b) G[c][b] = 0.0;
        }
        if (prm.op == kOpHelmholtz) {
          // (2 nu eps(u) n)_a with the own outward normal n = nsgn e_d
          for (int a = 0; a < NC; ++a) {
            const double vo = prm.nu * (go[a][d] + go[d][a]) * nsgn;
            if (kind == 0) {
              const double vn = prm.nu * (gn[a][d] + gn[d][a]) * nsgn;
              const double avg = 0.5 * (vo + vn);
              V[a] = -(avg - tau * (uo[a] - un[a])) * sj;
            } else {  // velocity-Dirichlet face (operators.py:473-483)
              V[a] = -(vo - 2.0 * tau * uo[a]) * sj;
            }
          }
          for (int a = 0; a < NC; ++a)
            for (int b = 0; b < DIM; ++b) {
              const double ja = kind == 0 ? uo[a] - un[a] : uo[a];
              const double jb = kind == 0 ? uo[b] - un[b] : uo[b];
              const double na = (a == d) ? nsgn : 0.0, nb = (b == d) ? nsgn : 0.0;
              G[a][b] = (kind == 0 ? -0.5 : -1.0) * prm.nu * (ja * nb + jb * na) * sj;
            }
        } else if (prm.op == kOpProjection) {
          for (int a = 0; a < NC; ++a) V[a] = tau * (uo[a] - un[a]) * sj;
        } else {
          // local Lax-Friedrichs, own frame (operators.py:597-604)
          double up[NC];
          if (kind == 0) for (int c = 0; c < NC; ++c) up[c] = un[c];
          else for (int c = 0; c < NC; ++c) up[c] = -uo[c];  // mirror 2g - u, g = 0
          const double unm = uo[d] * nsgn, unp = up[d] * nsgn;
          if (kind == kBndNeumann) {
            for (int a = 0; a < NC; ++a) V[a] = -beta * uo[a] * unm * sj;
          } else {
            const double lam = 2.0 * fmax(fabs(unm), fabs(unp));
            for (int a = 0; a < NC; ++a) {
              const double F = 0.5 * (uo[a] * unm + up[a] * unp) + 0.5 * lam * (uo[a] - up[a]);
              V[a] = -beta * F * sj;
            }
          }
        }
        for (int c = 0; c < NC; ++c) {
          fv[(c * (1 + DIM)) * FQ + i] = V[c];
          for (int b = 0; b < DIM; ++b) fv[(c * (1 + DIM) + 1 + b) * FQ + i] = G[c][b];
        }
      }
      __syncthreads();
      // lift: adjoint of the traces into sout
      const bool grad_terms = prm.op == kOpHelmholtz;
      for (int c = 0; c < NC; ++c) {
        const double *dv = fv + (c * (1 + DIM)) * FQ;
        // ft[0..FN) <- value-row lift data, ft[BIG..] <- derivative-row data
        if (DIM == 3) {
          const int tfa = d == 0 ? 1 : 0, tsl = d == 2 ? 1 : 2;
          // value test + tangential gradient tests land on the end layer
          contract(dv, t0, ST, N, NQ, 0, NQ, NQ, 1);
          contract(t0, t1, ST, N, NQ, 1, N, NQ, 1);          // value part [sl][fa]
          if (grad_terms) {
            contract(dv + (1 + tfa) * FQ, t0, DT, N, NQ, 0, NQ, NQ, 1);
            contract(t0, t2, ST, N, NQ, 1, N, NQ, 1);
            for (int i = tid; i < C::FN; i += blockDim.x) t1[i] += (2.0 / h[tfa]) * t2[i];
            __syncthreads();
            contract(dv + (1 + tsl) * FQ, t0, ST, N, NQ, 0, NQ, NQ, 1);
            contract(t0, t2, DT, N, NQ, 1, N, NQ, 1);
            for (int i = tid; i < C::FN; i += blockDim.x) t1[i] += (2.0 / h[tsl]) * t2[i];
            __syncthreads();
            contract(dv + (1 + d) * FQ, t0, ST, N, NQ, 0, NQ, NQ, 1);
            contract(t0, t2, ST, N, NQ, 1, N, NQ, 1);          // normal-gradient part
          }
        } else {
          const int tt = 1 - d;
          contract(dv, t1, ST, N, NQ, 0, NQ, 1, 1);
          if (grad_terms) {
            contract(dv + (1 + tt) * FQ, t2, DT, N, NQ, 0, NQ, 1, 1);
            for (int i = tid; i < C::FN; i += blockDim.x) t1[i] += (2.0 / h[tt]) * t2[i];
            __syncthreads();
            contract(dv + (1 + d) * FQ, t2, ST, N, NQ, 0, NQ, 1, 1);
          }
        }
        double *oc = sout + c * NP;
        const double sn = 2.0 / h[d];
        for (int i = tid; i < C::FN; i += blockDim.x) {
          const int sl = DIM == 3 ? i / N : 0, fa = DIM == 3 ? i % N : i;
          for (int k = 0; k < N; ++k) {
            int idx;
            if (DIM == 3) {
              if (d == 0) idx = (sl * N + fa) * N + k;
              else if (d == 1) idx = (sl * N + k) * N + fa;
              else idx = (k * N + sl) * N + fa;
            } else {
              idx = d == 0 ? fa * N + k : k * N + fa;
            }
            double add = 0.0;
            if (k == (s ? N - 1 : 0)) add += t1[i];
            if (grad_terms) add += sn * (s ? dR[k] : dL[k]) * t2[i];
            oc[idx] += add;
          }
        }
        __syncthreads();
      }
    }
  }
  for (int i = tid; i < NC * NP; i += blockDim.x) {
    const int c = i / NP, o = i % NP;
    out[((int64_t)c * ncells + e) * NP + o] = sout[i];
  }
}

}  // namespace dg
