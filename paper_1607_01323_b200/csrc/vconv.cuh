// Cartesian fast path of the convective term, 3D, fp64, sm_100a:
//   sum_i beta_i [(grad v, u_i (x) u_i) - (v, F*(u_i) . n)] + (v, f)
// with the local Lax-Friedrichs flux on the over-integration rule
// (reference operators.py:533-604, n_q = floor(3k/2)+1 or the literal
// 3(k+1)/2).  Same algebra and rule as the generic quadrature-point kernel
// (vecops.cuh, kOpConvective), reorganised so every phase works on all
// components (and all six sides) at once:
//
//   volume, per history level: nodal u -> Gauss points (three sweeps),
//   G_ab = beta u_a u_b JxW (symmetric, 6 arrays), then the gradient test
//   sum_b s_b (d_b v, G_ab) as   z: S^T / D^T,  y: combine into
//   A_a = S^T_y D^T_z G_a2 + D^T_y S^T_z G_a1 and B_a = S^T_y S^T_z G_a0,
//   x: out_a += S^T_x A_a + D^T_x B_a   (8 sweeps per component);
//   faces: GLL nodes include the cell ends, so a side's trace is the end
//   layer of nodes (own: shared memory, neighbour: read straight from global
//   memory / L2) interpolated tangentially (two sweeps); the LF flux at the
//   face Gauss points; the adjoint two sweeps; a gather adds the six lifted
//   sides to the nodes on them (no two threads write one node).
//
// One CTA per cell, T threads.  Every phase is "one thread per line": a
// thread loads one line of its input (Cc values) into registers and writes
// the R outputs of that line, with the 1D matrix entries as compile-time
// offsets into the __grid_constant__ parameter table (constant-bank operands,
// no shared-memory table loads): one shared load per Cc FMAs instead of two
// per FMA.
#pragma once
#include "common.cuh"
#include "vecops.cuh"

namespace dg {

// TV / MB: threads per CTA and the CTAs per SM the register budget must
// allow (0: the defaults below; other values are A/B experiments)
template <int N, int NQ, int TV = 0, int MB = 0>
struct CvCfg {
  static constexpr int NP = N * N * N, QP = NQ * NQ * NQ, FQ = NQ * NQ, FN = N * N;
  static constexpr int T = TV ? TV : (QP <= 64 ? 64 : 128);
  static constexpr int MINB = MB ? MB : (N >= 5 ? 3 : 4);
  static constexpr int TAB = NQ;  // Gauss weights (runtime-indexed)
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  // regions (doubles)
  static constexpr int U = TAB;                  // own nodal cell, 3 NP
  static constexpr int OUT = U + 3 * NP;         // accumulator, 3 NP
  static constexpr int NB = OUT + 3 * NP;        // neighbour end layers, 18 FN
  static constexpr int RA = NB + 18 * FN;
  // RA: u (3 QP) | A, B (6 N N NQ) | face fast sweep (36 N NQ) | lift 1 (18 NQ N) |
  //     body force (3 N N NQ)
  static constexpr int SZA = mx(mx(3 * QP, 6 * N * N * NQ), 36 * N * NQ);
  static constexpr int RB = RA + SZA;
  // RB: X1 + X2 (3 N N NQ + 3 N NQ NQ) | Z (9 N NQ NQ) | traces (36 FQ) + V (18 FQ) |
  //     lift 2 (18 N N) | body force (3 N NQ NQ)
  static constexpr int SZB = mx(mx(3 * N * N * NQ + 3 * N * NQ * NQ, 9 * N * NQ * NQ), 54 * FQ);
  static constexpr int NDBL = RB + SZB;
  static constexpr size_t SMEM = sizeof(double) * NDBL;
};

// v[i] for a runtime i without a local-memory copy of v
__device__ __forceinline__ double cv_sel3(const double (&v)[3], int i) {
  return i == 0 ? v[0] : (i == 1 ? v[1] : v[2]);
}

// node index of the end layer of side (d, s) at tangential nodes (sl, fa)
template <int N>
__device__ __forceinline__ int cv_end_node(int d, int s, int sl, int fa) {
  const int m = s ? N - 1 : 0;
  if (d == 0) return m + N * (fa + N * sl);
  if (d == 1) return fa + N * (m + N * sl);
  return fa + N * (sl + N * m);
}

// y = A x for one line, A(r, c) = TR ? tab[c * LD + r] : tab[r * LD + c]
template <int R, int Cc, int LD, bool TR>
__device__ __forceinline__ void cv_line(const double *tab, const double (&x)[Cc], double (&y)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double a = 0.0;
#pragma unroll
    for (int c = 0; c < Cc; ++c) a = fma(TR ? tab[c * LD + r] : tab[r * LD + c], x[c], a);
    y[r] = a;
  }
}
// Even-odd (flip-symmetric) form of an R x C matrix A with
// A[R-1-r][C-1-c] = SIG A[r][c] (SIG = +1: the GLL -> Gauss interpolation S
// and S^T; -1: the derivative D and D^T): with xs = x[c] + x[C-1-c],
// xd = x[c] - x[C-1-c] (c < C/2), E = (A[r][c] + A[r][C-1-c]) / 2 and
// O = (A[r][c] - A[r][C-1-c]) / 2, the rows r and R-1-r are ye +- yo with
// ye = E xs (+ A[r][C/2] x[C/2]), yo = O xd: about half the FMAs of y = A x.
template <int R, int C>
struct EoTab {
  static constexpr int RH = R / 2, CH = C / 2;
  double E[RH > 0 ? RH : 1][CH > 0 ? CH : 1];
  double O[RH > 0 ? RH : 1][CH > 0 ? CH : 1];
  double Mc[RH > 0 ? RH : 1];  // A[r][C/2], odd C
  double Mr[CH > 0 ? CH : 1];  // A[R/2][c], odd R
  double MM;                   // A[R/2][C/2], odd R and C
};

template <int R, int C>
static EoTab<R, C> eo_tab(const double *A) {  // A row-major R x C
  EoTab<R, C> t{};
  constexpr int RH = R / 2, CH = C / 2;
  for (int r = 0; r < RH; ++r) {
    for (int c = 0; c < CH; ++c) {
      t.E[r][c] = 0.5 * (A[r * C + c] + A[r * C + C - 1 - c]);
      t.O[r][c] = 0.5 * (A[r * C + c] - A[r * C + C - 1 - c]);
    }
    if (C & 1) t.Mc[r] = A[r * C + CH];
  }
  if (R & 1) {
    for (int c = 0; c < CH; ++c) t.Mr[c] = A[RH * C + c];
    if (C & 1) t.MM = A[RH * C + CH];
  }
  return t;
}

template <int R, int C, int SIG>
__device__ __forceinline__ void eo_line(const EoTab<R, C> &t, const double (&x)[C], double (&y)[R]) {
  constexpr int RH = R / 2, CH = C / 2;
  double xs[CH > 0 ? CH : 1], xd[CH > 0 ? CH : 1];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    xs[c] = x[c] + x[C - 1 - c];
    xd[c] = x[c] - x[C - 1 - c];
  }
#pragma unroll
  for (int r = 0; r < RH; ++r) {
    double ye = (C & 1) ? t.Mc[r] * x[CH] : 0.0, yo = 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      ye = fma(t.E[r][c], xs[c], ye);
      yo = fma(t.O[r][c], xd[c], yo);
    }
    y[r] = ye + yo;
    y[R - 1 - r] = SIG > 0 ? ye - yo : yo - ye;
  }
  if (R & 1) {
    double ym = (SIG > 0 && (C & 1)) ? t.MM * x[CH] : 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) ym = fma(t.Mr[c], SIG > 0 ? xs[c] : xd[c], ym);
    y[RH] = ym;
  }
}

// the four 1D operators of the convective kernel in even-odd form
template <int N, int NQ>
struct CvEo {
  EoTab<NQ, N> S, D;    // nodes -> Gauss points: values, derivatives
  EoTab<N, NQ> St, Dt;  // their transposes (the tests)
};

template <int Cc>
__device__ __forceinline__ void cv_load(const double *p, int stride, double (&x)[Cc]) {
#pragma unroll
  for (int c = 0; c < Cc; ++c) x[c] = p[c * stride];
}
template <int R>
__device__ __forceinline__ void cv_store(double *p, int stride, const double (&y)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r) p[r * stride] = y[r];
}

template <int N, int NQ, int TV = 0, int MB = 0>
__global__ void __launch_bounds__(CvCfg<N, NQ, TV, MB>::T, CvCfg<N, NQ, TV, MB>::MINB)
vconv_kernel(double *__restrict__ out, const Geo g, const __grid_constant__ QuadTab<N, NQ> tab,
             const __grid_constant__ CvEo<N, NQ> eo, const VecParams prm, const int64_t ncells) {
  using C = CvCfg<N, NQ, TV, MB>;
  constexpr int NP = C::NP, QP = C::QP, FQ = C::FQ, FN = C::FN, T = C::T;
  constexpr int NQ2 = NQ * NQ;
  extern __shared__ double sm[];
  __shared__ const double *p_hist[kMaxHist], *p_gh[kMaxHist][6];
  __shared__ double p_beta[kMaxHist];
  __shared__ int kind[6];
  __shared__ int64_t nbr[6];
  double *W = sm;
  double *su = sm + C::U, *so = sm + C::OUT, *snb = sm + C::NB, *ra = sm + C::RA, *rb = sm + C::RB;
  const int tid = threadIdx.x;
  const int64_t e = blockIdx.x;
  const int ix = (int)(e % g.nx), iy = (int)((e / g.nx) % g.ny), iz = (int)(e / ((int64_t)g.nx * g.ny));
  const double h[3] = {g.hx[ix], g.hy[iy], g.hz[iz]};
  const double sc[3] = {2.0 * g.hxi[ix], 2.0 * g.hyi[iy], 2.0 * g.hzi[iz]};
  const double det = 0.125 * h[0] * h[1] * h[2];
  for (int i = tid; i < NQ; i += T) W[i] = tab.w[i];
  for (int i = tid; i < 3 * NP; i += T) so[i] = 0.0;
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < kMaxHist; ++j) {
      p_hist[j] = prm.hist[j];
      p_beta[j] = prm.beta[j];
#pragma unroll
      for (int q = 0; q < 6; ++q) p_gh[j][q] = prm.gh[j][q];
    }
  }
  // side kinds and neighbours (shared: indexed by runtime side below)
  if (tid < 6) {
    const int side = tid;
    const int d = side >> 1, s = side & 1;
    const int nd = d == 0 ? g.nx : (d == 1 ? g.ny : g.nz);
    int nidx = (d == 0 ? ix : (d == 1 ? iy : iz)) + (s ? 1 : -1);
    int k = 0;
    if (nidx < 0 || nidx >= nd) {
      const int m = g.mode[side];
      k = (m == kBndNone || m == kBndNeumann) ? m : 0;
      nidx = s ? 0 : nd - 1;  // periodic wrap
    }
    kind[side] = k;
    const int cx = d == 0 ? nidx : ix, cy = d == 1 ? nidx : iy, cz = d == 2 ? nidx : iz;
    nbr[side] = cx + (int64_t)g.nx * (cy + (int64_t)g.ny * cz);
  }
  __syncthreads();

  for (int lev = 0; lev < prm.n_hist; ++lev) {
    const double *src = p_hist[lev];
    const double beta = p_beta[lev];
    // ---- loads: own cell and the neighbours' end layers ----------------------
    for (int i = tid; i < 3 * NP; i += T) {
      const int c = i / NP, o = i % NP;
      su[i] = src[((int64_t)c * ncells + e) * NP + o];
    }
    for (int i = tid; i < 18 * FN; i += T) {
      const int side = i / (3 * FN), c = (i / FN) % 3, f = i % FN;
      double v = 0.0;
      if (kind[side] == 0)
        v = src[((int64_t)c * ncells + nbr[side]) * NP + cv_end_node<N>(side >> 1, (side & 1) ^ 1, f / N, f % N)];
      snb[i] = v;
    }
    __syncthreads();
    // ---- volume: nodes -> Gauss points --------------------------------------
    double *x1 = rb, *x2 = rb + 3 * N * N * NQ;
    for (int l = tid; l < 3 * N * N; l += T) {  // x lines: x1[c][z][y][qx]
      double xi[N], yo[NQ];
      cv_load<N>(su + l * N, 1, xi);
      eo_line<NQ, N, 1>(eo.S, xi, yo);
      cv_store<NQ>(x1 + l * NQ, 1, yo);
    }
    __syncthreads();
    for (int l = tid; l < 3 * N * NQ; l += T) {  // y lines: x2[c][z][qy][qx]
      const int cz = l / NQ, qx = l % NQ;
      double xi[N], yo[NQ];
      cv_load<N>(x1 + cz * N * NQ + qx, NQ, xi);
      eo_line<NQ, N, 1>(eo.S, xi, yo);
      cv_store<NQ>(x2 + cz * NQ2 + qx, NQ, yo);
    }
    __syncthreads();
    // z lines: u at the Gauss points -> ra[c][qz][qy][qx]
    for (int l = tid; l < 3 * NQ2; l += T) {
      const int c = l / NQ2, qxy = l % NQ2;
      double xi[N], yo[NQ];
      cv_load<N>(x2 + c * N * NQ2 + qxy, NQ2, xi);
      eo_line<NQ, N, 1>(eo.S, xi, yo);
      cv_store<NQ>(ra + c * QP + qxy, NQ2, yo);
    }
    __syncthreads();
    // G_ab = beta u_a u_b JxW on z lines and its z test contraction
    // Z_ab[z][qy][qx] = s_b (b == 2 ? D : S)^T G_ab -> rb[ab][z][qy][qx]; the 8
    // distinct contractions (G symmetric) are separate work items
    for (int l = tid; l < 8 * NQ2; l += T) {
      const int job = l / NQ2, qxy = l % NQ2;
      // job: 0 G00 S | 1 G11 S | 2 G22 D | 3 G01 S (-> Z01, Z10) | 4 G02 D | 5 G02 S | 6 G12 D | 7 G12 S
      const int a = job == 1 ? 1 : (job == 2 ? 2 : (job >= 6 ? 1 : 0));
      const int b = job == 0 ? 0 : (job == 1 || job == 3 ? 1 : 2);
      const bool dz = job == 2 || job == 4 || job == 6;
      const double wxy = beta * det * W[qxy % NQ] * W[qxy / NQ];
      double ua[NQ], ub[NQ], gz[NQ], zo[N];
      cv_load<NQ>(ra + a * QP + qxy, NQ2, ua);
      cv_load<NQ>(ra + b * QP + qxy, NQ2, ub);
#pragma unroll
      for (int q = 0; q < NQ; ++q) gz[q] = ua[q] * ub[q] * (wxy * tab.w[q]);
      if (dz) eo_line<N, NQ, -1>(eo.Dt, gz, zo);
      else eo_line<N, NQ, 1>(eo.St, gz, zo);
      // destination (r, t) = test direction t for component r: dz -> (a, 2);
      // S jobs: 0 (0,0) 1 (1,1) 3 (0,1)+(1,0) 5 (2,0) 7 (2,1)
      const int r = dz ? a : (job == 5 || job == 7 ? 2 : a);
      const int t = dz ? 2 : (job == 5 ? 0 : (job == 7 ? 1 : b));
      const double st = cv_sel3(sc, t);
      double *zd = rb + (r * 3 + t) * N * NQ2 + qxy;
#pragma unroll
      for (int z = 0; z < N; ++z) zd[z * NQ2] = st * zo[z];
      if (job == 3) {
        double *z2 = rb + (1 * 3 + 0) * N * NQ2 + qxy;
#pragma unroll
        for (int z = 0; z < N; ++z) z2[z * NQ2] = sc[0] * zo[z];
      }
    }
    __syncthreads();
    // y lines: A_a = S^T Z_a2 + D^T Z_a1, B_a = S^T Z_a0   -> rb[a][A|B][z][y][qx]
    for (int l = tid; l < 3 * N * NQ; l += T) {
      const int a = l / (N * NQ), z = (l / NQ) % N, qx = l % NQ;
      double z0[NQ], z1[NQ], z2[NQ], ya[N], yb[N], yd[N];
      const double *zb = rb + (a * 3 * N + z) * NQ2 + qx;
      cv_load<NQ>(zb, NQ, z0);
      cv_load<NQ>(zb + N * NQ2, NQ, z1);
      cv_load<NQ>(zb + 2 * N * NQ2, NQ, z2);
      eo_line<N, NQ, 1>(eo.St, z2, ya);
      eo_line<N, NQ, -1>(eo.Dt, z1, yd);
      eo_line<N, NQ, 1>(eo.St, z0, yb);
#pragma unroll
      for (int y = 0; y < N; ++y) ya[y] += yd[y];
      cv_store<N>(ra + ((a * 2 + 0) * N + z) * N * NQ + qx, NQ, ya);
      cv_store<N>(ra + ((a * 2 + 1) * N + z) * N * NQ + qx, NQ, yb);
    }
    __syncthreads();
    // x lines: out_a += S^T A_a + D^T B_a
    for (int l = tid; l < 3 * N * N; l += T) {
      const int a = l / (N * N), zy = l % (N * N);
      double xa[NQ], xb[NQ], oa[N], ob[N];
      cv_load<NQ>(ra + ((a * 2 + 0) * N * N + zy) * NQ, 1, xa);
      cv_load<NQ>(ra + ((a * 2 + 1) * N * N + zy) * NQ, 1, xb);
      eo_line<N, NQ, 1>(eo.St, xa, oa);
      eo_line<N, NQ, -1>(eo.Dt, xb, ob);
      double *o = so + a * NP + zy * N;
#pragma unroll
      for (int x = 0; x < N; ++x) o[x] += oa[x] + ob[x];
    }
    __syncthreads();
    // ---- faces ----------------------------------------------------------------
    // fast tangential sweep of own / neighbour end layers: ra[o][side][c][sl][qfa]
    for (int l = tid; l < 36 * N; l += T) {
      const int o = l / (18 * N), side = (l / (3 * N)) % 6, c = (l / N) % 3, sl = l % N;
      const int d = side >> 1;
      double xi[N], yo[NQ];
      if (o == 0) cv_load<N>(su + c * NP + cv_end_node<N>(d, side & 1, sl, 0), d == 0 ? N : 1, xi);
      else cv_load<N>(snb + (side * 3 + c) * FN + sl * N, 1, xi);
      eo_line<NQ, N, 1>(eo.S, xi, yo);
      cv_store<NQ>(ra + l * NQ, 1, yo);
    }
    __syncthreads();
    // slow sweep: traces rb[o][side][c][qsl][qfa]
    for (int l = tid; l < 36 * NQ; l += T) {
      const int osc = l / NQ, qfa = l % NQ;
      double xi[N], yo[NQ];
      cv_load<N>(ra + osc * N * NQ + qfa, NQ, xi);
      eo_line<NQ, N, 1>(eo.S, xi, yo);
      cv_store<NQ>(rb + osc * FQ + qfa, NQ, yo);
    }
    __syncthreads();
    // Lax-Friedrichs flux at the face Gauss points -> vf[side][a][f] (rb + 36 FQ)
    double *vf = rb + 36 * FQ;
    for (int i = tid; i < 6 * FQ; i += T) {
      const int side = i / FQ, f = i % FQ, d = side >> 1, s = side & 1;
      const int k = kind[side];
      const double nsgn = s ? 1.0 : -1.0;
      const double fdet = d == 0 ? 0.25 * h[1] * h[2] : (d == 1 ? 0.25 * h[0] * h[2] : 0.25 * h[0] * h[1]);
      const double sj = fdet * W[f % NQ] * W[f / NQ];
      double uo[3], up[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        uo[c] = rb[(side * 3 + c) * FQ + f];
        up[c] = rb[(18 + side * 3 + c) * FQ + f];
      }
      if (k != 0) {  // mirror state 2 g - u with the level's Dirichlet data
        const double *gd = p_gh[lev][side];
        const int64_t it = d == 0 ? (int64_t)iz * g.ny + iy
                                  : (d == 1 ? (int64_t)iz * g.nx + ix : (int64_t)iy * g.nx + ix);
#pragma unroll
        for (int c = 0; c < 3; ++c) up[c] = (gd ? 2.0 * gd[(it * 3 + c) * FQ + f] : 0.0) - uo[c];
      }
      const double unm = cv_sel3(uo, d) * nsgn, unp = cv_sel3(up, d) * nsgn;
      if (k == kBndNeumann) {
#pragma unroll
        for (int a = 0; a < 3; ++a) vf[(side * 3 + a) * FQ + f] = -beta * uo[a] * unm * sj;
      } else {
        const double lam = 2.0 * fmax(fabs(unm), fabs(unp));
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double Fl = 0.5 * (uo[a] * unm + up[a] * unp) + 0.5 * lam * (uo[a] - up[a]);
          vf[(side * 3 + a) * FQ + f] = -beta * Fl * sj;
        }
      }
    }
    __syncthreads();
    // lift, fast: ra[side][a][qsl][fa] = S^T along the fast face axis
    for (int l = tid; l < 18 * NQ; l += T) {
      double xi[NQ], yo[N];
      cv_load<NQ>(vf + l * NQ, 1, xi);
      eo_line<N, NQ, 1>(eo.St, xi, yo);
      cv_store<N>(ra + l * N, 1, yo);
    }
    __syncthreads();
    // lift, slow: rb[side][a][sl][fa]
    for (int l = tid; l < 18 * N; l += T) {
      const int sa = l / N, fa = l % N;
      double xi[NQ], yo[N];
      cv_load<NQ>(ra + sa * NQ * N + fa, N, xi);
      eo_line<N, NQ, 1>(eo.St, xi, yo);
      cv_store<N>(rb + sa * FN + fa, N, yo);
    }
    __syncthreads();
    // gather the lifted sides onto the end nodes
    for (int i = tid; i < 3 * NP; i += T) {
      const int a = i / NP, r = i % NP;
      const int x = r % N, y = (r / N) % N, z = r / (N * N);
      double add = 0.0;
      if (x == 0) add += rb[(0 * 3 + a) * FN + z * N + y];
      if (x == N - 1) add += rb[(1 * 3 + a) * FN + z * N + y];
      if (y == 0) add += rb[(2 * 3 + a) * FN + z * N + x];
      if (y == N - 1) add += rb[(3 * 3 + a) * FN + z * N + x];
      if (z == 0) add += rb[(4 * 3 + a) * FN + y * N + x];
      if (z == N - 1) add += rb[(5 * 3 + a) * FN + y * N + x];
      so[i] += add;
    }
    __syncthreads();
  }

  if (prm.vol_data != nullptr) {
    // (v, f) with the body force sampled at the quadrature points:
    // (S^T x S^T x S^T)(f JxW), z then y then x
    for (int l = tid; l < 3 * NQ2; l += T) {  // rb[a][z][qy][qx]
      const int a = l / NQ2, qxy = l % NQ2;
      const double wxy = det * W[qxy % NQ] * W[qxy / NQ];
      const double *fd = prm.vol_data + ((int64_t)a * ncells + e) * QP + qxy;
      double xi[NQ], yo[N];
#pragma unroll
      for (int q = 0; q < NQ; ++q) xi[q] = fd[q * NQ2] * (wxy * tab.w[q]);
      eo_line<N, NQ, 1>(eo.St, xi, yo);
      cv_store<N>(rb + a * N * NQ2 + qxy, NQ2, yo);
    }
    __syncthreads();
    for (int l = tid; l < 3 * N * NQ; l += T) {  // ra[a][z][y][qx]
      const int az = l / NQ, qx = l % NQ;
      double xi[NQ], yo[N];
      cv_load<NQ>(rb + az * NQ2 + qx, NQ, xi);
      eo_line<N, NQ, 1>(eo.St, xi, yo);
      cv_store<N>(ra + az * N * NQ + qx, NQ, yo);
    }
    __syncthreads();
    for (int l = tid; l < 3 * N * N; l += T) {
      double xi[NQ], yo[N];
      cv_load<NQ>(ra + l * NQ, 1, xi);
      eo_line<N, NQ, 1>(eo.St, xi, yo);
      double *o = so + l * N;
#pragma unroll
      for (int x = 0; x < N; ++x) o[x] += yo[x];
    }
    __syncthreads();
  }
  for (int i = tid; i < 3 * NP; i += T) {
    const int c = i / NP, o = i % NP;
    out[((int64_t)c * ncells + e) * NP + o] = so[i];
  }
}

}  // namespace dg
