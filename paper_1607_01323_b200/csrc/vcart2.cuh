// Line-per-thread kernels of the Cartesian Helmholtz / projection fast path
// (algebra and Gauss-collocated representation described in vcart.cuh):
// every volume phase gives one thread one line of one component (N values
// in registers) and applies a 1D matrix whose entries are compile-time
// offsets into the __grid_constant__ parameter table, so a line costs N
// shared loads and N stores for N*N FMAs (a point-per-thread version paid
// two shared loads per FMA and was bound by shared-memory bandwidth).  One
// thread per component line (3 N^2 threads per cell): the cells resident per
// SM are set by shared memory, so more threads per cell is more latency
// hiding (1.5x over one thread per line looping over components).
//
//   trace:  x: S, y: S, z: S (u~) + z-side traces, y / x: side traces
//   apply:  faces (point-wise: fluxes, tangential terms; vcart.cuh algebra)
//           x: S  y: S  z: S -> u~, d/dz -> T  y: d/dy -> T  x: d/dx -> T
//           x: mass + Dg^T T_a0 + x-side lifts   y: + Dg^T T_a1 + lifts
//           z: + Dg^T T_a2 + lifts, S^T   x: S^T   y: S^T -> global
//
// Shared arrays per cell use a padded layout x + LS y + PS z (LS odd) so the
// x-line, y-line and z-line access patterns of a half-warp hit distinct
// banks.
#pragma once
#include "vcart.cuh"

namespace dg {

template <int N, int CB = 0>
struct VlCfg {
  static constexpr int P = N * N * N, F = N * N;
  static constexpr int LS = (N & 1) ? N : N + 1;  // padded line stride
  static constexpr int PS = LS * N;               // plane stride
  static constexpr int CS = PS * N;               // one component of one cell
  // cells per CTA (Q3: 2 -- C4 projection apply 248 -> 227 us, Helmholtz
  // 348 -> 343 us against 4; 1 and 8 slower; profiles/r02/vec_time.py)
  static constexpr int CPB = CB ? CB : (N <= 2 ? 32 : (N == 3 ? 16 : (N == 4 ? 2 : (N <= 6 ? 4 : 2))));
  static constexpr int LINES = CPB * N * N;       // lines of one component
  static constexpr int THREADS = ((3 * LINES + 31) / 32) * 32;  // one thread per component line
  static constexpr int TAB = 2 * N * N + 5 * N;   // VcTab staged for the face phases
  // per cell: UG (3 CS: u~, then the accumulator), TT (6 CS: ping-pong, T,
  // face transients Wf / GT), JA (36 F: face value / normal-gradient tests)
  static constexpr int UG = 0, TT = 3 * CS, JA = 9 * CS;
  static constexpr int CELL = 9 * CS + 36 * F;
  static constexpr size_t SMEM = sizeof(double) * (TAB + CPB * CELL);
};

template <int N>
__device__ __forceinline__ int vl_idx(int x, int y, int z) {
  return x + VlCfg<N>::LS * y + VlCfg<N>::PS * z;
}

// y = A x, A(r, c) = TR ? tab[c * N + r] : tab[r * N + c]
template <int N, bool TR>
__device__ __forceinline__ void vl_mat(const double *tab, const double (&x)[N], double (&y)[N]) {
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double a = 0.0;
#pragma unroll
    for (int c = 0; c < N; ++c) a = fma(TR ? tab[c * N + r] : tab[r * N + c], x[c], a);
    y[r] = a;
  }
}

// line `ax` (0 x, 1 y, 2 z) through (i, j) = the other two coordinates in
// increasing axis order: first element index and stride
template <int N>
__device__ __forceinline__ void vl_line(int ax, int i, int j, int &first, int &stride) {
  using C = VlCfg<N>;
  if (ax == 0) { first = C::LS * i + C::PS * j; stride = 1; }
  else if (ax == 1) { first = i + C::PS * j; stride = C::LS; }
  else { first = i + C::LS * j; stride = C::PS; }
}

template <int N>
__device__ __forceinline__ void vl_ld(const double *p, int stride, double (&v)[N]) {
#pragma unroll
  for (int m = 0; m < N; ++m) v[m] = p[m * stride];
}
template <int N>
__device__ __forceinline__ void vl_st(double *p, int stride, const double (&v)[N]) {
#pragma unroll
  for (int m = 0; m < N; ++m) p[m * stride] = v[m];
}

// cell geometry
struct VlGeo {
  int ix, iy, iz;
  double h[3], sc[3], det;
};
// cell coordinates by 32-bit division (cell counts < 2^31)
__device__ __forceinline__ void vl_cell_xyz(const Geo &g, int64_t e, int &ix, int &iy, int &iz) {
  const unsigned ei = (unsigned)e, nx = (unsigned)g.nx, ny = (unsigned)g.ny;
  const unsigned q = ei / nx;
  ix = (int)(ei - q * nx);
  iz = (int)(q / ny);
  iy = (int)(q - (unsigned)iz * ny);
}
__device__ __forceinline__ VlGeo vl_geo(const Geo &g, int64_t e) {
  VlGeo v;
  vl_cell_xyz(g, e, v.ix, v.iy, v.iz);
  v.h[0] = g.hx[v.ix];
  v.h[1] = g.hy[v.iy];
  v.h[2] = g.hz[v.iz];
  v.sc[0] = 2.0 * g.hxi[v.ix];
  v.sc[1] = 2.0 * g.hyi[v.iy];
  v.sc[2] = 2.0 * g.hzi[v.iz];
  v.det = 0.125 * v.h[0] * v.h[1] * v.h[2];
  return v;
}

// nodal -> Gauss-collocated u~ of all CPB cells: x (global -> TT), y (TT ->
// UG), z (UG -> UG).  The z phase hands each z line of u~ to `zline`
// (cs, c, x, y, u~ line) while it is in registers.  Ends with a barrier.
// pz != null: the input is first updated in place, u = pz + beta u (the CG
// direction update p = z + beta p of the velocity PCG, rounded like
// vpcg_p_kernel), so u may not be __restrict__
template <int N, int CB, class ZL>
__device__ __forceinline__ void vl_to_gauss(const double *u, int64_t e0,
                                            int64_t ncells, const double *S, double *sm_cells,
                                            ZL &&zline, const double *pz = nullptr,
                                            double beta = 0.0) {
  using C = VlCfg<N, CB>;
  constexpr int NN = N * N;
  #pragma unroll
  for (int it = threadIdx.x; it < 3 * C::LINES; it += C::THREADS) {  // x lines
    const int cs = it / (3 * NN), c = (it / NN) % 3, l = it % NN, y = l % N, z = l / N;
    const int64_t e = e0 + cs;
    double v[N], w[N];
    if (e < ncells) {
      const int64_t off = ((int64_t)c * ncells + e) * C::P + (z * N + y) * N;
      vl_ld<N>(u + off, 1, v);
      if (pz) {
        double zz[N];
        vl_ld<N>(pz + off, 1, zz);
#pragma unroll
        for (int m = 0; m < N; ++m) v[m] = __dadd_rn(zz[m], __dmul_rn(beta, v[m]));
        vl_st<N>(const_cast<double *>(u) + off, 1, v);
      }
    } else {
#pragma unroll
      for (int m = 0; m < N; ++m) v[m] = 0.0;
    }
    vl_mat<N, false>(S, v, w);
    vl_st<N>(sm_cells + cs * C::CELL + C::TT + c * C::CS + vl_idx<N>(0, y, z), 1, w);
  }
  __syncthreads();
  #pragma unroll
  for (int it = threadIdx.x; it < 3 * C::LINES; it += C::THREADS) {  // y lines
    const int cs = it / (3 * NN), c = (it / NN) % 3, l = it % NN, x = l % N, z = l / N;
    double *cell = sm_cells + cs * C::CELL;
    double v[N], w[N];
    vl_ld<N>(cell + C::TT + c * C::CS + vl_idx<N>(x, 0, z), C::LS, v);
    vl_mat<N, false>(S, v, w);
    vl_st<N>(cell + C::UG + c * C::CS + vl_idx<N>(x, 0, z), C::LS, w);
  }
  __syncthreads();
  #pragma unroll
  for (int it = threadIdx.x; it < 3 * C::LINES; it += C::THREADS) {  // z lines
    const int cs = it / (3 * NN), c = (it / NN) % 3, l = it % NN, x = l % N, y = l / N;
    double *p = sm_cells + cs * C::CELL + C::UG + c * C::CS + vl_idx<N>(x, y, 0);
    double v[N], w[N];
    vl_ld<N>(p, C::PS, v);
    vl_mat<N, false>(S, v, w);
    vl_st<N>(p, C::PS, w);
    zline(cs, c, x, y, w);
  }
  __syncthreads();
}

// Traces of all three components on all six sides at the face Gauss points
// trc[cell][side][comp][val | dn][f].
// pz != null: p = pz + beta p in place first (u = p), and scal[0] = rz_new
template <int N, bool NEED_DN, int CB = 0>
__global__ void __launch_bounds__(VlCfg<N, CB>::THREADS)
vl_trace_kernel(const double *u, double *__restrict__ trc, const Geo g,
                const __grid_constant__ VcTab<N> tab, const int64_t ncells,
                const double *__restrict__ pz = nullptr, double beta = 0.0,
                double *__restrict__ scal = nullptr, double rz_new = 0.0) {
  if (pz && scal && blockIdx.x == 0 && threadIdx.x == 0) scal[0] = rz_new;
  using C = VlCfg<N, CB>;
  constexpr int F = C::F, NN = N * N;
  extern __shared__ double sm[];
  double *cells = sm + C::TAB;
  const int64_t e0 = (int64_t)blockIdx.x * C::CPB;
  __shared__ double ssc[C::CPB][3];
  if (threadIdx.x < 3 * C::CPB) {  // one thread per (cell, axis)
    const int cs = threadIdx.x / 3, d = threadIdx.x - 3 * cs;
    int ix, iy, iz;
    vl_cell_xyz(g, e0 + cs < ncells ? e0 + cs : 0, ix, iy, iz);
    ssc[cs][d] = 2.0 * (d == 0 ? g.hxi[ix] : (d == 1 ? g.hyi[iy] : g.hzi[iz]));
  }
  __syncthreads();
  auto emit = [&](int64_t e, int side, int c, int f, const double (&w)[N], double sd) {
    double v0 = 0.0, d0 = 0.0;
    const bool hi = side & 1;
#pragma unroll
    for (int m = 0; m < N; ++m) {
      v0 = fma(hi ? tab.eR[m] : tab.eL[m], w[m], v0);
      if (NEED_DN) d0 = fma(hi ? tab.gR[m] : tab.gL[m], w[m], d0);
    }
    double *o = trc + e * (36 * F) + ((side * 3 + c) * 2) * F + f;
    o[0] = v0;
    if (NEED_DN) o[F] = sd * d0;
  };
  auto zl = [&](int cs, int c, int x, int y, const double (&w)[N]) {
    const int64_t e = e0 + cs;
    if (e >= ncells) return;
    const double sz = ssc[cs][2];
    emit(e, 4, c, y * N + x, w, sz);
    emit(e, 5, c, y * N + x, w, sz);
  };
  vl_to_gauss<N, CB>(u, e0, ncells, tab.S, cells, zl, pz, beta);
  #pragma unroll
  for (int it = threadIdx.x; it < 6 * C::LINES; it += C::THREADS) {  // y and x lines of u~
    const int ax = it < 3 * C::LINES ? 1 : 0;
    const int jt = ax == 1 ? it : it - 3 * C::LINES;
    const int cs = jt / (3 * NN), c = (jt / NN) % 3, l = jt % NN, i = l % N, j = l / N;
    const int64_t e = e0 + cs;
    if (e >= ncells) continue;
    int first, stride;
    vl_line<N>(ax, i, j, first, stride);
    double w[N];
    vl_ld<N>(cells + cs * C::CELL + C::UG + c * C::CS + first, stride, w);
    const double sd = ssc[cs][ax];
    // y line (i, j) = (x, z): f = z N + x; x line (i, j) = (y, z): f = z N + y
    emit(e, 2 * ax + 0, c, j * N + i, w, sd);
    emit(e, 2 * ax + 1, c, j * N + i, w, sd);
  }
}

template <int N, int OP, int CB = 0>
__global__ void __launch_bounds__(VlCfg<N, CB>::THREADS)
vl_apply_kernel(const double *__restrict__ u, const double *__restrict__ trc,
                double *__restrict__ out, const Geo g, const __grid_constant__ VcTab<N> tab,
                const double gamma0_dt, const double nu, const double *__restrict__ tau_d,
                const double *__restrict__ tau_c, const int64_t ncells,
                double *__restrict__ pdot = nullptr) {
  using C = VlCfg<N, CB>;
  constexpr int F = C::F, NN = N * N;
  extern __shared__ double sm[];
  double *tb = sm;
  const double *Dg = tb + N * N, *W = tb + 2 * N * N;
  double *cells = sm + C::TAB;
  const int64_t e0 = (int64_t)blockIdx.x * C::CPB;
  // per-cell geometry, side kinds and neighbours, computed once
  __shared__ VlGeo sgeo[C::CPB];
  __shared__ int skind[C::CPB][6];
  __shared__ int64_t snbr[C::CPB][6];
  vc_stage_tab<N>(tb, tab);
  // one thread per (cell, side) for the side kinds / neighbours, one per cell
  // for the geometry (all in the first warps, in parallel)
  static_assert(7 * C::CPB <= C::THREADS, "setup: one pass");
  if (threadIdx.x < 7 * C::CPB) {
    const int cs = threadIdx.x / 7, side = threadIdx.x - 7 * cs;
    const int64_t e = e0 + cs < ncells ? e0 + cs : 0;
    if (side == 6) {
      sgeo[cs] = vl_geo(g, e);
    } else {
      int ix, iy, iz;
      vl_cell_xyz(g, e, ix, iy, iz);
      const int d = side >> 1, s = side & 1;
      const int nd = d == 0 ? g.nx : (d == 1 ? g.ny : g.nz);
      int nidx = (d == 0 ? ix : (d == 1 ? iy : iz)) + (s ? 1 : -1);
      int k = 0;
      if (nidx < 0 || nidx >= nd) {
        const int m = g.mode[side];
        k = (m == kBndNone || m == kBndNeumann) ? m : 0;
        nidx = s ? 0 : nd - 1;  // periodic wrap
      }
      const int cx = d == 0 ? nidx : ix, cy = d == 1 ? nidx : iy, cz = d == 2 ? nidx : iz;
      skind[cs][side] = k;
      snbr[cs][side] = cx + (int64_t)g.nx * (cy + (int64_t)g.ny * cz);
    }
  }
  __syncthreads();
  const bool faces = OP == kVcHelmholtz ? nu != 0.0 : tau_c != nullptr;
  const bool divdiv = OP == kVcHelmholtz || tau_d != nullptr;

  // ---- faces (point-wise, vcart.cuh algebra) ---------------------------------
  if (faces) {
    auto face_sj = [&](const VlGeo &v, int d, int f) {
      const double fdet = d == 0 ? 0.25 * v.h[1] * v.h[2]
                                 : (d == 1 ? 0.25 * v.h[0] * v.h[2] : 0.25 * v.h[0] * v.h[1]);
      return fdet * W[f % N] * W[f / N];
    };
    // FA: jumps, averaged normal derivatives, w; projection: final value test
    #pragma unroll
    for (int it = threadIdx.x; it < C::CPB * 6 * F; it += C::THREADS) {
      const int cs = it / (6 * F), i = it % (6 * F);
      const int side = i / F, f = i % F, d = side >> 1, s = side & 1;
      const int64_t e = e0 + cs;
      const bool valid = e < ncells;
      const int64_t ec = valid ? e : 0;
      const VlGeo &v = sgeo[cs];
      double *cell = cells + cs * C::CELL;
      double *Wf = cell + C::TT, *JV = cell + C::JA, *AN = JV + 18 * F;
      const int kind = skind[cs][side];
      const bool skip = !valid || (OP == kVcHelmholtz ? kind == kBndNeumann : kind != 0);
      double jv[3] = {0.0, 0.0, 0.0}, an[3] = {0.0, 0.0, 0.0}, w = 0.0;
      if (!skip) {
        const double *to = trc + ec * (36 * F) + (side * 6) * F + f;
        double uo[3], un[3] = {0.0, 0.0, 0.0}, dno[3], dnn[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          uo[c] = to[(2 * c) * F];
          if (OP == kVcHelmholtz) dno[c] = to[(2 * c + 1) * F];
        }
        int64_t en = ec;
        if (kind == 0) {
          en = snbr[cs][side];
          const double *tn = trc + en * (36 * F) + ((side ^ 1) * 6) * F + f;
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
          const double sj = face_sj(v, d, f);
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
      #pragma unroll
    for (int it = threadIdx.x; it < C::CPB * 6 * F; it += C::THREADS) {
        const int cs = it / (6 * F), i = it % (6 * F);
        const int side = i / F, f = i % F, d = side >> 1, s = side & 1;
        const int64_t e = e0 + cs;
        const bool valid = e < ncells;
        const VlGeo &v = sgeo[cs];
        double *cell = cells + cs * C::CELL;
        double *Wf = cell + C::TT, *GT = Wf + 6 * F, *JV = cell + C::JA, *AN = JV + 18 * F;
        const int kind = skind[cs][side];
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
          const double stf = vc_sel(v.sc, tf), sts = vc_sel(v.sc, ts), sdn = vc_sel(v.sc, d);
          dwf *= stf;
          dws *= sts;
          const double nsgn = s ? 1.0 : -1.0;
          const double sj = face_sj(v, d, f);
          double tau, c0;
          if (kind == 0) {
            tau = fmax(g.tau[e], g.tau[snbr[cs][side]]) * nu;
            c0 = -0.5;
          } else {
            tau = 2.0 * g.tau[e] * nu;
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
      #pragma unroll
    for (int it = threadIdx.x; it < C::CPB * 6 * F; it += C::THREADS) {
        const int cs = it / (6 * F), i = it % (6 * F);
        const int side = i / F, f = i % F, d = side >> 1;
        const int fa = f % N, sl = f / N;
        double *cell = cells + cs * C::CELL;
        const double *GT = cell + C::TT + 6 * F;
        double *JV = cell + C::JA;
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
  }

  // ---- volume: u~ and the test data T ----------------------------------------
  // T slots (TT + k CS): 0 T00, 1 T11, 2 T22, 3 T01, 4 T02, 5 T12 (Helmholtz,
  // symmetric nu (d_b u_a + d_a u_b) JxW); projection: slot 0 = tau_D div JxW
  auto zl = [&](int cs, int c, int x, int y, const double (&w)[N]) {
    if (!divdiv) return;
    if (OP == kVcProjection && c != 2) return;
    const VlGeo &v = sgeo[cs];
    double gz[N];
    vl_mat<N, false>(tab.Dg, w, gz);
    double *cell = cells + cs * C::CELL;
    const int first = vl_idx<N>(x, y, 0);
    if (OP == kVcHelmholtz) {
      if (c == 2) {  // T22 final
        const double wxy = nu * v.det * W[x] * W[y];
#pragma unroll
        for (int m = 0; m < N; ++m) gz[m] = (v.sc[2] * gz[m] + v.sc[2] * gz[m]) * (wxy * tab.w[m]);
      } else {
#pragma unroll
        for (int m = 0; m < N; ++m) gz[m] *= v.sc[2];
      }
      vl_st<N>(cell + C::TT + (c == 0 ? 4 : (c == 1 ? 5 : 2)) * C::CS + first, C::PS, gz);
    } else {
#pragma unroll
      for (int m = 0; m < N; ++m) gz[m] *= v.sc[2];
      vl_st<N>(cell + C::TT + first, C::PS, gz);  // div accumulator
    }
  };
  vl_to_gauss<N, CB>(u, e0, ncells, tab.S, cells, zl);
  if (divdiv) {
    // y lines: d/dy
    #pragma unroll
    for (int it = threadIdx.x; it < 3 * C::LINES; it += C::THREADS) {
      const int cs = it / (3 * NN), c = (it / NN) % 3, l = it % NN, x = l % N, z = l / N;
      if (OP == kVcProjection && c != 1) continue;
      const VlGeo &v = sgeo[cs];
      double *cell = cells + cs * C::CELL;
      const int first = vl_idx<N>(x, 0, z);
      double w[N], gy[N];
      vl_ld<N>(cell + C::UG + c * C::CS + first, C::LS, w);
      vl_mat<N, false>(tab.Dg, w, gy);
      if (OP == kVcHelmholtz) {
        const double wxz = nu * v.det * W[x] * W[z];
        if (c == 0) {  // T01 partial
#pragma unroll
          for (int m = 0; m < N; ++m) gy[m] *= v.sc[1];
          vl_st<N>(cell + C::TT + 3 * C::CS + first, C::LS, gy);
        } else if (c == 1) {  // T11 final
#pragma unroll
          for (int m = 0; m < N; ++m) gy[m] = (v.sc[1] * gy[m] + v.sc[1] * gy[m]) * (wxz * tab.w[m]);
          vl_st<N>(cell + C::TT + 1 * C::CS + first, C::LS, gy);
        } else {  // T12 final = (d_z u_1 + d_y u_2) JxW nu
          double t[N];
          vl_ld<N>(cell + C::TT + 5 * C::CS + first, C::LS, t);
#pragma unroll
          for (int m = 0; m < N; ++m) t[m] = (t[m] + v.sc[1] * gy[m]) * (wxz * tab.w[m]);
          vl_st<N>(cell + C::TT + 5 * C::CS + first, C::LS, t);
        }
      } else {
        double t[N];
        vl_ld<N>(cell + C::TT + first, C::LS, t);
#pragma unroll
        for (int m = 0; m < N; ++m) t[m] += v.sc[1] * gy[m];
        vl_st<N>(cell + C::TT + first, C::LS, t);
      }
    }
    __syncthreads();
    // x lines: d/dx
    #pragma unroll
    for (int it = threadIdx.x; it < 3 * C::LINES; it += C::THREADS) {
      const int cs = it / (3 * NN), c = (it / NN) % 3, l = it % NN, y = l % N, z = l / N;
      if (OP == kVcProjection && c != 0) continue;
      const int64_t e = e0 + cs;
      const VlGeo &v = sgeo[cs];
      double *cell = cells + cs * C::CELL;
      const int first = vl_idx<N>(0, y, z);
      double w[N], gx[N];
      vl_ld<N>(cell + C::UG + c * C::CS + first, 1, w);
      vl_mat<N, false>(tab.Dg, w, gx);
      const double wyz = v.det * W[y] * W[z];
      if (OP == kVcHelmholtz) {
        if (c == 0) {  // T00 final
#pragma unroll
          for (int m = 0; m < N; ++m) gx[m] = (v.sc[0] * gx[m] + v.sc[0] * gx[m]) * (nu * wyz * tab.w[m]);
          vl_st<N>(cell + C::TT + 0 * C::CS + first, 1, gx);
        } else {  // T01 (c = 1) / T02 (c = 2) final
          double *tp = cell + C::TT + (c == 1 ? 3 : 4) * C::CS + first;
          double t[N];
          vl_ld<N>(tp, 1, t);
#pragma unroll
          for (int m = 0; m < N; ++m) t[m] = (t[m] + v.sc[0] * gx[m]) * (nu * wyz * tab.w[m]);
          vl_st<N>(tp, 1, t);
        }
      } else {
        const double td = e < ncells ? tau_d[e] : 0.0;
        double *tp = cell + C::TT + first;
        double t[N];
        vl_ld<N>(tp, 1, t);
#pragma unroll
        for (int m = 0; m < N; ++m) t[m] = td * (t[m] + v.sc[0] * gx[m]) * (wyz * tab.w[m]);
        vl_st<N>(tp, 1, t);
      }
    }
    __syncthreads();
  }

  // ---- volume + face tests, accumulated in place of u~ ------------------------
  const double mass = OP == kVcHelmholtz ? gamma0_dt : 1.0;
  // lifts of the two sides normal to axis `ax` onto a line through face point f
  auto lift = [&](const double *cell, int ax, int a, int f, double (&acc)[N]) {
    if (!faces) return;
    const double *JV = cell + C::JA, *AN = JV + 18 * F;
    const double j0 = JV[((2 * ax) * 3 + a) * F + f], j1 = JV[((2 * ax + 1) * 3 + a) * F + f];
    const double n0 = AN[((2 * ax) * 3 + a) * F + f], n1 = AN[((2 * ax + 1) * 3 + a) * F + f];
#pragma unroll
    for (int m = 0; m < N; ++m) {
      double t = fma(tab.eL[m], j0, acc[m]);
      t = fma(tab.eR[m], j1, t);
      if (OP == kVcHelmholtz) {
        t = fma(tab.gL[m], n0, t);
        t = fma(tab.gR[m], n1, t);
      }
      acc[m] = t;
    }
  };
  // T slot tested with d/dx_b for component a (-1: none)
  auto tslot = [&](int a, int b) -> int {
    if (OP == kVcProjection) return (divdiv && a == b) ? 0 : -1;
    if (a == b) return a;
    return a + b + 2;  // 01 -> 3, 02 -> 4, 12 -> 5
  };
  // x lines: mass + d/dx test + x-side lifts
  #pragma unroll
  for (int it = threadIdx.x; it < 3 * C::LINES; it += C::THREADS) {
    const int cs = it / (3 * NN), a = (it / NN) % 3, l = it % NN, y = l % N, z = l / N;
    const VlGeo &v = sgeo[cs];
    double *cell = cells + cs * C::CELL;
    const int first = vl_idx<N>(0, y, z);
    double w[N], acc[N];
    vl_ld<N>(cell + C::UG + a * C::CS + first, 1, w);
    const double wyz = mass * v.det * W[y] * W[z];
#pragma unroll
    for (int m = 0; m < N; ++m) acc[m] = w[m] * (wyz * tab.w[m]);
    const int k = tslot(a, 0);
    if (k >= 0) {
      double t[N], d[N];
      vl_ld<N>(cell + C::TT + k * C::CS + first, 1, t);
      vl_mat<N, true>(tab.Dg, t, d);
#pragma unroll
      for (int m = 0; m < N; ++m) acc[m] = fma(v.sc[0], d[m], acc[m]);
    }
    lift(cell, 0, a, z * N + y, acc);
    vl_st<N>(cell + C::UG + a * C::CS + first, 1, acc);
  }
  __syncthreads();
  // y lines: d/dy test + y-side lifts
  #pragma unroll
  for (int it = threadIdx.x; it < 3 * C::LINES; it += C::THREADS) {
    const int cs = it / (3 * NN), a = (it / NN) % 3, l = it % NN, x = l % N, z = l / N;
    const int k = tslot(a, 1);
    if (k < 0 && !faces) continue;
    const VlGeo &v = sgeo[cs];
    double *cell = cells + cs * C::CELL;
    const int first = vl_idx<N>(x, 0, z);
    double acc[N];
    vl_ld<N>(cell + C::UG + a * C::CS + first, C::LS, acc);
    if (k >= 0) {
      double t[N], d[N];
      vl_ld<N>(cell + C::TT + k * C::CS + first, C::LS, t);
      vl_mat<N, true>(tab.Dg, t, d);
#pragma unroll
      for (int m = 0; m < N; ++m) acc[m] = fma(v.sc[1], d[m], acc[m]);
    }
    lift(cell, 1, a, z * N + x, acc);
    vl_st<N>(cell + C::UG + a * C::CS + first, C::LS, acc);
  }
  __syncthreads();
  // z lines: d/dz test + z-side lifts, then S^T along z
  #pragma unroll
  for (int it = threadIdx.x; it < 3 * C::LINES; it += C::THREADS) {
    const int cs = it / (3 * NN), a = (it / NN) % 3, l = it % NN, x = l % N, y = l / N;
    const int k = tslot(a, 2);
    const VlGeo &v = sgeo[cs];
    double *cell = cells + cs * C::CELL;
    const int first = vl_idx<N>(x, y, 0);
    double acc[N], o[N];
    vl_ld<N>(cell + C::UG + a * C::CS + first, C::PS, acc);
    if (k >= 0) {
      double t[N], d[N];
      vl_ld<N>(cell + C::TT + k * C::CS + first, C::PS, t);
      vl_mat<N, true>(tab.Dg, t, d);
#pragma unroll
      for (int m = 0; m < N; ++m) acc[m] = fma(v.sc[2], d[m], acc[m]);
    }
    lift(cell, 2, a, y * N + x, acc);
    vl_mat<N, true>(tab.S, acc, o);
    vl_st<N>(cell + C::UG + a * C::CS + first, C::PS, o);
  }
  __syncthreads();
  // x lines: S^T (UG -> TT)
  #pragma unroll
  for (int it = threadIdx.x; it < 3 * C::LINES; it += C::THREADS) {
    const int cs = it / (3 * NN), a = (it / NN) % 3, l = it % NN, y = l % N, z = l / N;
    double *cell = cells + cs * C::CELL;
    const int first = vl_idx<N>(0, y, z);
    double w[N], o[N];
    vl_ld<N>(cell + C::UG + a * C::CS + first, 1, w);
    vl_mat<N, true>(tab.S, w, o);
    vl_st<N>(cell + C::TT + a * C::CS + first, 1, o);
  }
  __syncthreads();
  // y lines: S^T -> global (+ the CG product u . out of this line)
  double dacc = 0.0;
  #pragma unroll
  for (int it = threadIdx.x; it < 3 * C::LINES; it += C::THREADS) {
    const int cs = it / (3 * NN), a = (it / NN) % 3, l = it % NN, x = l % N, z = l / N;
    const int64_t e = e0 + cs;
    if (e >= ncells) continue;
    double *cell = cells + cs * C::CELL;
    double w[N], o[N];
    vl_ld<N>(cell + C::TT + a * C::CS + vl_idx<N>(x, 0, z), C::LS, w);
    vl_mat<N, true>(tab.S, w, o);
    double *dst = out + ((int64_t)a * ncells + e) * C::P + z * NN + x;
    vl_st<N>(dst, N, o);
    if (pdot) {
      const double *src = u + ((int64_t)a * ncells + e) * C::P + z * NN + x;
#pragma unroll
      for (int m = 0; m < N; ++m) dacc = fma(src[m * N], o[m], dacc);
    }
  }
  if (pdot) {  // deterministic CTA sum -> pdot[blockIdx.x]
    __shared__ double red[C::THREADS / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < C::THREADS / 32; ++w) t += red[w];
      pdot[blockIdx.x] = t;
    }
  }
}

}  // namespace dg
