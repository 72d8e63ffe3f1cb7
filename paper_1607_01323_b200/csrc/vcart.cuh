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
//   every side, at the face Gauss points) are produced once per cell by
//   vc_trace_kernel into a [cell][side][comp][val|dn][face point] buffer;
//   vc_apply_kernel reads its own and its neighbours' traces from it (L2),
//   so no CTA loads a neighbour cell.  Tangential derivatives on a face are
//   taken from the traces (the two cells of a face share the tangential
//   Gauss points of a tensor box mesh).
// * One thread per Gauss point, CPB cells per CTA; every contraction is an
//   N-term dot over a line of a shared-memory array (conflict-free: the
//   threads of a half-warp read distinct 8-byte words or broadcast).
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

// cell e's nodal components -> u~ (Gauss-collocated) in ug[c * P + p];
// uses r[0 .. 3P) as scratch.  Ends with a barrier.
template <int N>
__device__ __forceinline__ void vc_to_gauss(const double *__restrict__ u, int64_t e, int64_t ncells,
                                            bool valid, const double *S, double *ug, double *r, int p,
                                            int x, int y, int z) {
  constexpr int P = VcCfg<N>::P;
#pragma unroll
  for (int c = 0; c < 3; ++c) r[c * P + p] = valid ? u[((int64_t)c * ncells + e) * P + p] : 0.0;
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 3; ++c) ug[c * P + p] = vc_dot<N, 0>(S + x * N, 1, r + c * P, x, y, z);
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 3; ++c) r[c * P + p] = vc_dot<N, 1>(S + y * N, 1, ug + c * P, x, y, z);
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 3; ++c) ug[c * P + p] = vc_dot<N, 2>(S + z * N, 1, r + c * P, x, y, z);
  __syncthreads();
}

// volume point of side d at face point f and normal coordinate m
template <int N>
__device__ __forceinline__ int vc_face_pt(int d, int f, int m) {
  const int fa = f % N, sl = f / N;
  if (d == 0) return m + N * (fa + N * sl);
  if (d == 1) return fa + N * (m + N * sl);
  return fa + N * (sl + N * m);
}

// Traces of all three components on all six sides at the face Gauss points:
// trc[cell][side][comp][0] values, [1] physical d/dx_d (NEED_DN).
template <int N, bool NEED_DN>
__global__ void __launch_bounds__(VcCfg<N>::THREADS)
vc_trace_kernel(const double *__restrict__ u, double *__restrict__ trc, const Geo g,
                const VcTab<N> tab, const int64_t ncells) {
  using C = VcCfg<N>;
  constexpr int P = C::P, F = C::F;
  extern __shared__ double sm[];
  double *tb = sm;
  const double *S = tb, *EL = tb + 2 * N * N + N, *ER = EL + N, *GL = ER + N, *GR = GL + N;
  const int cs = threadIdx.x / P, p = threadIdx.x % P;
  const int x = p % N, y = (p / N) % N, z = p / (N * N);
  const int64_t e = (int64_t)blockIdx.x * C::CPB + cs;
  const bool valid = e < ncells;
  double *base = sm + C::TAB + cs * C::CELL;
  double *ug = base, *r = base + 3 * P;
  vc_stage_tab<N>(tb, tab);
  vc_to_gauss<N>(u, e, ncells, valid, S, ug, r, p, x, y, z);
  if (!valid) return;
  const int ix = (int)(e % g.nx), iy = (int)((e / g.nx) % g.ny), iz = (int)(e / ((int64_t)g.nx * g.ny));
  const double sx = 2.0 * g.hxi[ix], sy = 2.0 * g.hyi[iy], sz = 2.0 * g.hzi[iz];
  double *dst = trc + e * C::TRC;
  for (int i = p; i < 6 * F; i += P) {
    const int side = i / F, f = i % F, d = side >> 1, s = side & 1;
    const double *ev = s ? ER : EL, *gv = s ? GR : GL;
    const double sd = d == 0 ? sx : (d == 1 ? sy : sz);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double v = 0.0, dn = 0.0;
#pragma unroll
      for (int m = 0; m < N; ++m) {
        const double um = ug[c * P + vc_face_pt<N>(d, f, m)];
        v = fma(ev[m], um, v);
        if (NEED_DN) dn = fma(gv[m], um, dn);
      }
      double *o = dst + ((side * 3 + c) * 2) * F;
      o[f] = v;
      if (NEED_DN) o[F + f] = sd * dn;
    }
  }
}

template <int N, int OP>
__global__ void __launch_bounds__(VcCfg<N>::THREADS)
vc_apply_kernel(const double *__restrict__ u, const double *__restrict__ trc,
                double *__restrict__ out, const Geo g, const VcTab<N> tab, const double gamma0_dt,
                const double nu, const double *__restrict__ tau_d, const double *__restrict__ tau_c,
                const int64_t ncells) {
  using C = VcCfg<N>;
  constexpr int P = C::P, F = C::F;
  extern __shared__ double sm[];
  double *tb = sm;
  const double *S = tb, *Dg = tb + N * N, *W = tb + 2 * N * N;
  const double *EL = W + N, *ER = EL + N, *GL = ER + N, *GR = GL + N;
  const int cs = threadIdx.x / P, p = threadIdx.x % P;
  const int x = p % N, y = (p / N) % N, z = p / (N * N);
  const int64_t e = (int64_t)blockIdx.x * C::CPB + cs;
  const bool valid = e < ncells;
  const int64_t ec = valid ? e : 0;  // geometry of a clamped cell for idle slots
  double *base = sm + C::TAB + cs * C::CELL;
  double *ug = base, *r = base + 3 * P;
  vc_stage_tab<N>(tb, tab);
  vc_to_gauss<N>(u, e, ncells, valid, S, ug, r, p, x, y, z);

  const int ix = (int)(ec % g.nx), iy = (int)((ec / g.nx) % g.ny), iz = (int)(ec / ((int64_t)g.nx * g.ny));
  const double hx = g.hx[ix], hy = g.hy[iy], hz = g.hz[iz];
  const double sc[3] = {2.0 * g.hxi[ix], 2.0 * g.hyi[iy], 2.0 * g.hzi[iz]};
  const double det = 0.125 * hx * hy * hz;
  const double jw = det * W[x] * W[y] * W[z];

  double acc[3];
  const double ut[3] = {ug[p], ug[P + p], ug[2 * P + p]};
  // ---- volume ---------------------------------------------------------------
  if (OP == kVcHelmholtz) {
    double gr[3][3];  // gr[c][b] = d u_c / d x_b
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      gr[c][0] = sc[0] * vc_dot<N, 0>(Dg + x * N, 1, ug + c * P, x, y, z);
      gr[c][1] = sc[1] * vc_dot<N, 1>(Dg + y * N, 1, ug + c * P, x, y, z);
      gr[c][2] = sc[2] * vc_dot<N, 2>(Dg + z * N, 1, ug + c * P, x, y, z);
      acc[c] = gamma0_dt * ut[c] * jw;
    }
    // symmetric test data T_ab = nu (d_b u_a + d_a u_b) jw at r[6][P]:
    // slots 00 11 22 01 02 12 (r is free: the last sweep read it before the
    // barrier that ended vc_to_gauss)
    const double nj = nu * jw;
    r[0 * P + p] = nj * (gr[0][0] + gr[0][0]);
    r[1 * P + p] = nj * (gr[1][1] + gr[1][1]);
    r[2 * P + p] = nj * (gr[2][2] + gr[2][2]);
    r[3 * P + p] = nj * (gr[0][1] + gr[1][0]);
    r[4 * P + p] = nj * (gr[0][2] + gr[2][0]);
    r[5 * P + p] = nj * (gr[1][2] + gr[2][1]);
    __syncthreads();
    // acc_a += sum_b s_b Dg^T_b T_ab
    constexpr int slot[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      acc[a] += sc[0] * vc_dot<N, 0>(Dg + x, N, r + slot[a][0] * P, x, y, z);
      acc[a] += sc[1] * vc_dot<N, 1>(Dg + y, N, r + slot[a][1] * P, x, y, z);
      acc[a] += sc[2] * vc_dot<N, 2>(Dg + z, N, r + slot[a][2] * P, x, y, z);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] = ut[c] * jw;
    if (tau_d != nullptr) {
      const double div = sc[0] * vc_dot<N, 0>(Dg + x * N, 1, ug, x, y, z) +
                         sc[1] * vc_dot<N, 1>(Dg + y * N, 1, ug + P, x, y, z) +
                         sc[2] * vc_dot<N, 2>(Dg + z * N, 1, ug + 2 * P, x, y, z);
      r[p] = tau_d[ec] * div * jw;
      __syncthreads();
      acc[0] += sc[0] * vc_dot<N, 0>(Dg + x, N, r, x, y, z);
      acc[1] += sc[1] * vc_dot<N, 1>(Dg + y, N, r, x, y, z);
      acc[2] += sc[2] * vc_dot<N, 2>(Dg + z, N, r, x, y, z);
    }
  }
  __syncthreads();  // ug / r are reused as face scratch below

  // ---- faces ------------------------------------------------------------------
  const bool faces = OP == kVcHelmholtz ? nu != 0.0 : tau_c != nullptr;
  if (faces) {
    double *Wf = base, *JV = Wf + 6 * F, *AN = JV + 18 * F, *GT = AN + 18 * F;
    const double te = g.tau[ec];
    auto kind_of = [&](int d, int s) {
      const int nd = d == 0 ? g.nx : (d == 1 ? g.ny : g.nz);
      const int nidx = (d == 0 ? ix : (d == 1 ? iy : iz)) + (s ? 1 : -1);
      if (nidx >= 0 && nidx < nd) return 0;
      const int m = g.mode[2 * d + s];
      return (m == kBndNone || m == kBndNeumann) ? m : 0;
    };
    auto nbr_of = [&](int d, int s) -> int64_t {
      const int nd = d == 0 ? g.nx : (d == 1 ? g.ny : g.nz);
      int nidx = (d == 0 ? ix : (d == 1 ? iy : iz)) + (s ? 1 : -1);
      if (nidx < 0 || nidx >= nd) nidx = s ? 0 : nd - 1;  // periodic wrap
      const int cx = d == 0 ? nidx : ix, cy = d == 1 ? nidx : iy, cz = d == 2 ? nidx : iz;
      return cx + (int64_t)g.nx * (cy + (int64_t)g.ny * cz);
    };
    auto face_sj = [&](int d, int f) {
      const double fdet = d == 0 ? 0.25 * hy * hz : (d == 1 ? 0.25 * hx * hz : 0.25 * hx * hy);
      return fdet * W[f % N] * W[f / N];
    };
    // FA: jumps, averaged normal derivatives, w; projection: final value test
    for (int i = p; i < 6 * F; i += P) {
      const int side = i / F, f = i % F, d = side >> 1, s = side & 1;
      const int kind = kind_of(d, s);
      const bool skip = !valid || (OP == kVcHelmholtz ? kind == kBndNeumann : kind != 0);
      double jv[3] = {0.0, 0.0, 0.0}, an[3] = {0.0, 0.0, 0.0}, w = 0.0;
      if (!skip) {
        const double *to = trc + ec * C::TRC + (side * 6) * F + f;
        double uo[3], un[3] = {0.0, 0.0, 0.0}, dno[3], dnn[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          uo[c] = to[(2 * c) * F];
          if (OP == kVcHelmholtz) dno[c] = to[(2 * c + 1) * F];
        }
        int64_t en = ec;
        if (kind == 0) {
          en = nbr_of(d, s);
          const double *tn = trc + en * C::TRC + ((side ^ 1) * 6) * F + f;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            un[c] = tn[(2 * c) * F];
            if (OP == kVcHelmholtz) dnn[c] = tn[(2 * c + 1) * F];
          }
        }
        if (OP == kVcHelmholtz) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            jv[c] = kind == 0 ? uo[c] - un[c] : uo[c];
            an[c] = kind == 0 ? 0.5 * (dno[c] + dnn[c]) : dno[c];
          }
          w = kind == 0 ? 0.5 * (vc_sel(uo, d) + vc_sel(un, d)) : vc_sel(uo, d);
        } else {
          const double tau = tau_c[(int64_t)d * ncells + (s ? ec : en)];
          const double sj = face_sj(d, f);
#pragma unroll
          for (int c = 0; c < 3; ++c) jv[c] = tau * (uo[c] - un[c]) * sj;
        }
      }
      Wf[i] = w;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        JV[(side * 3 + c) * F + f] = jv[c];
        AN[(side * 3 + c) * F + f] = an[c];
      }
    }
    __syncthreads();
    if (OP == kVcHelmholtz) {
      // FB: fluxes and test coefficients
      for (int i = p; i < 6 * F; i += P) {
        const int side = i / F, f = i % F, d = side >> 1, s = side & 1;
        const int kind = kind_of(d, s);
        const int tf = d == 0 ? 1 : 0, ts = d == 2 ? 1 : 2;
        const int fa = f % N, sl = f / N;
        double gt0 = 0.0, gt1 = 0.0;
        if (valid && kind != kBndNeumann) {
          const double *wf = Wf + side * F;
          double dwf = 0.0, dws = 0.0;
#pragma unroll
          for (int m = 0; m < N; ++m) {
            dwf = fma(Dg[fa * N + m], wf[sl * N + m], dwf);
            dws = fma(Dg[sl * N + m], wf[m * N + fa], dws);
          }
          const double stf = vc_sel(sc, tf), sts = vc_sel(sc, ts), sdn = vc_sel(sc, d);
          dwf *= stf;
          dws *= sts;
          const double nsgn = s ? 1.0 : -1.0;
          const double sj = face_sj(d, f);
          double tau, c0;
          if (kind == 0) {
            tau = fmax(te, g.tau[nbr_of(d, s)]) * nu;
            c0 = -0.5;
          } else {
            tau = 2.0 * te * nu;
            c0 = -1.0;
          }
          double j[3], a_[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            j[c] = JV[(side * 3 + c) * F + f];
            a_[c] = AN[(side * 3 + c) * F + f];
          }
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const double da_w = a == d ? vc_sel(a_, d) : (a == tf ? dwf : dws);
            const double A = nu * (a_[a] + da_w) * nsgn;
            JV[(side * 3 + a) * F + f] = -(A - tau * j[a]) * sj;
            const double gn = c0 * nu * nsgn * sj * (j[a] + (a == d ? vc_sel(j, d) : 0.0));
            AN[(side * 3 + a) * F + f] = sdn * gn;
          }
          gt0 = stf * c0 * nu * nsgn * sj * vc_sel(j, tf);
          gt1 = sts * c0 * nu * nsgn * sj * vc_sel(j, ts);
        }
        GT[(side * 2 + 0) * F + f] = gt0;
        GT[(side * 2 + 1) * F + f] = gt1;
      }
      __syncthreads();
      // FC: tangential-gradient tests of component d, transposed onto the face
      for (int i = p; i < 6 * F; i += P) {
        const int side = i / F, f = i % F, d = side >> 1;
        const int fa = f % N, sl = f / N;
        const double *g0 = GT + (side * 2 + 0) * F, *g1 = GT + (side * 2 + 1) * F;
        double add = 0.0;
#pragma unroll
        for (int m = 0; m < N; ++m) {
          add = fma(Dg[m * N + fa], g0[sl * N + m], add);
          add = fma(Dg[m * N + sl], g1[m * N + fa], add);
        }
        JV[(side * 3 + d) * F + f] += add;
      }
      __syncthreads();
    }
    // lift: gather the six sides' test data at this Gauss point
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int f = d == 0 ? z * N + y : (d == 1 ? z * N + x : y * N + x);
      const int m = d == 0 ? x : (d == 1 ? y : z);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int side = 2 * d + s;
        const double ev = s ? ER[m] : EL[m];
        const double gv = s ? GR[m] : GL[m];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          acc[a] = fma(ev, JV[(side * 3 + a) * F + f], acc[a]);
          if (OP == kVcHelmholtz) acc[a] = fma(gv, AN[(side * 3 + a) * F + f], acc[a]);
        }
      }
    }
    __syncthreads();
  }

  // ---- back to the nodal basis: (S^T x S^T x S^T) acc --------------------------
#pragma unroll
  for (int c = 0; c < 3; ++c) ug[c * P + p] = acc[c];
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 3; ++c) r[c * P + p] = vc_dot<N, 0>(S + x, N, ug + c * P, x, y, z);
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 3; ++c) ug[c * P + p] = vc_dot<N, 1>(S + y, N, r + c * P, x, y, z);
  __syncthreads();
  if (valid) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      out[((int64_t)c * ncells + e) * P + p] = vc_dot<N, 2>(S + z, N, ug + c * P, x, y, z);
  }
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
  if (!(scal[1] > 0.0)) return;  // breakdown: the host stops, x and r stay
  const double alpha = __ddiv_rn(scal[0], scal[1]);
  // blockDim = THREADS rounded up to whole warps (full-mask shuffles below);
  // the padding threads own no node
  const bool in = threadIdx.x < C::THREADS;
  const int cs = in ? threadIdx.x / P : 0, q = in ? threadIdx.x % P : 0;
  const int x0 = q % N, y0 = (q / N) % N, z0 = q / (N * N);
  const int64_t e = (int64_t)blockIdx.x * C::CPB + cs;
  const bool valid = in && e < ncells;
  double *b0 = buf[0] + cs * 3 * P, *b1 = buf[1] + cs * 3 * P;
  double rv[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int64_t i = ((int64_t)c * ncells + e) * P + q;
    double v = 0.0;
    if (valid) {
      x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
      v = __dsub_rn(r[i], __dmul_rn(alpha, Ap[i]));
      r[i] = v;
    }
    rv[c] = v;
    if (in) b0[c * P + q] = v;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double t = vc_dot<N, 0>(mi.A + x0 * N, 1, b0 + c * P, x0, y0, z0);
    if (in) b1[c * P + q] = t;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double t = vc_dot<N, 1>(mi.A + y0 * N, 1, b1 + c * P, x0, y0, z0);
    if (in) b0[c * P + q] = t;
  }
  __syncthreads();
  double acc = 0.0;
  if (valid) {
    const int ix = (int)(e % g.nx), iy = (int)((e / g.nx) % g.ny), iz = (int)(e / ((int64_t)g.nx * g.ny));
    double s = 0.5 * g.hx[ix] * 0.5 * g.hy[iy];
    s *= 0.5 * g.hz[iz];
    s = 1.0 / s;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double zv = s * vc_dot<N, 2>(mi.A + z0 * N, 1, b0 + c * P, x0, y0, z0);
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
