// Fused cell+face SIPG Laplace vmult for Cartesian cells, fp64, sm_100a.
//
// Replaces apply_pressure_laplace (reference operators.py:187-238).  On an
// axis-aligned cell the reference's quadrature-point evaluation collapses to
// a separable form (exact up to rounding, Gauss rule n_q = k+1 integrates
// every product exactly):
//
//   out = M_z [ M_y ( s_x Kh_x u + s_x Lx ) + s_y Kh_y P + s_y Ly ]
//         + s_z Kh_z Q + s_z Lz,        P = M_x u,  Q = M_y P
//
// with M = S^T W S, Kh_d = (2/h_d) D^T W D (1D reference matrices),
// s_d = prod_{d' != d} h_d'/2, and L_d the face lifts of the SIP fluxes
// (operators.py:209-237) evaluated from the value/normal-derivative face
// functionals of u (x), P (y) and Q (z) -- linear functionals commute with
// the tangential masses, so face terms need no extra sweeps.
//
// CTA = brick of BX*BY*BZ cells held in shared memory; one thread per line
// per phase (x-lines, y-lines, z-lines).  Neighbour functionals come from
// the brick (shared memory) or, across the brick surface, from halo cells
// read once from L2 (global) with their tangential masses applied.
// No atomics: every output DoF is written once by its own cell
// (the reference's gather-then-scatter determinism, spaces.py:151-158).
#pragma once
#include <type_traits>

#include "common.cuh"

namespace dg {

template <int N>
__host__ __device__ constexpr int row_pitch() {
  return (N % 2 == 0) ? N + 1 : N;  // odd smem row pitch: conflict-free lines
}

struct NbrInfo {
  int kind;        // 0 in-brick, 1 halo, 2 boundary none, 3 boundary neumann
  int cb;          // in-brick cell index
  double h;        // neighbour size in the face-normal direction
  double tau;      // neighbour tau_e
  const double *src;  // halo: neighbour cell data (global)
};

// Resolve the neighbour of owned cell (ix,iy,iz) across side (D, s).
template <int D, int S, int DIM, int N, int BX, int BY, int BZ>
__device__ __forceinline__ NbrInfo resolve_nbr(const Geo &g, const double *u,
                                               int ix, int iy,
                                               int iz, int x0, int y0, int z0,
                                               int ex, int ey, int ez) {
  constexpr int NP = (DIM == 3) ? N * N * N : N * N;
  NbrInfo r;
  r.cb = 0;
  r.src = nullptr;
  r.h = 1.0;
  r.tau = 0.0;
  const int nd = D == 0 ? g.nx : D == 1 ? g.ny : g.nz;
  int cd = D == 0 ? ix : D == 1 ? iy : iz;
  int nc = cd + (S ? 1 : -1);
  if (nc < 0 || nc >= nd) {
    const int m = g.mode[2 * D + S];
    if (m == kWrap) {
      nc = S ? 0 : nd - 1;
    } else if (m == kGhost) {
      const int t = iy + g.ny * iz;
      r.kind = 1;
      r.src = g.ghost[S] + (size_t)t * NP;
      r.h = g.ghost_h[S];
      r.tau = g.ghost_tau[S][t];
      return r;
    } else {
      r.kind = m;  // kBndNone / kBndNeumann
      return r;
    }
  }
  const int cx = D == 0 ? nc : ix, cy = D == 1 ? nc : iy, cz = D == 2 ? nc : iz;
  const size_t e = (size_t)cx + (size_t)g.nx * (cy + (size_t)g.ny * cz);
  r.h = (D == 0) ? g.hx[cx] : (D == 1) ? g.hy[cy] : g.hz[cz];
  r.tau = g.tau[e];
  const int lo = D == 0 ? x0 : D == 1 ? y0 : z0;
  const int ext = D == 0 ? ex : D == 1 ? ey : ez;
  if (nc >= lo && nc < lo + ext) {
    r.kind = 0;
    r.cb = (cx - x0) + BX * ((cy - y0) + BY * (cz - z0));
  } else {
    r.kind = 1;
    r.src = u + e * NP;
  }
  return r;
}

// SIP face lift for one line.  vo/go: own value / reference derivative at
// the face end; vn/gn neighbour's; returns (cv, cd): the value-row and
// derivative-row coefficients (already including the own 1/h factors).
__device__ __forceinline__ void sip_coeffs(int kind, int s, double vo,
                                           double go, double vn, double gn,
                                           double h, double hn, double tau,
                                           double &cv, double &cd) {
  if (kind <= 1) {  // interior
    if (s) {          // own cell is the minus side
      const double jump = vo - vn;
      const double avg = go / h + gn / hn;
      cv = -(avg - tau * jump);
      cd = -jump / h;
    } else {          // own cell is the plus side
      const double jump = vn - vo;
      const double avg = gn / hn + go / h;
      cv = avg - tau * jump;
      cd = -jump / h;
    }
  } else if (kind == kBndNeumann) {  // pressure-Dirichlet (operators.py:227-233)
    if (s) {
      cv = -(2.0 / h * go - 2.0 * tau * vo);
      cd = -2.0 * vo / h;
    } else {
      cv = 2.0 / h * go + 2.0 * tau * vo;
      cd = 2.0 * vo / h;
    }
  } else {
    cv = 0.0;
    cd = 0.0;
  }
}

template <int DIM, int N, int BX, int BY, int BZ>
struct LapCfg {
  static constexpr int RP = row_pitch<N>();
  static constexpr int NC = BX * BY * BZ;
  static constexpr int LPC = (DIM == 3) ? N * N : N;      // lines per cell
  static constexpr int CS = (DIM == 3) ? N * N * RP : N * RP;  // smem cell stride
  static constexpr int NL = NC * LPC;
  static constexpr int THREADS = ((NL + 31) / 32) * 32;
  static constexpr int SIDE_CELLS_X = BY * BZ;
  static constexpr int SIDE_CELLS_Y = BX * BZ;
  static constexpr int SIDE_CELLS_Z = (DIM == 3) ? BX * BY : 0;
  // halo buffers: per side, cells * (v, g) * LPC
  static constexpr int HOFF_X = 0;
  static constexpr int HOFF_Y = HOFF_X + 2 * SIDE_CELLS_X * 2 * LPC;
  static constexpr int HOFF_Z = HOFF_Y + 2 * SIDE_CELLS_Y * 2 * LPC;
  static constexpr int HSIZE = HOFF_Z + 2 * SIDE_CELLS_Z * 2 * LPC;
  static constexpr int BUF = NC * CS;
  static constexpr int BUF1 = (BUF > HSIZE) ? BUF : HSIZE;  // aliases halo raw
  static constexpr int FBUF = NC * 4 * LPC;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(BUF + BUF1 + FBUF + HSIZE);
};

// halo slot offset of side (d, s) and tangential brick position t
template <int DIM, int N, int BX, int BY, int BZ>
__device__ __forceinline__ int halo_off(int d, int s, int pos) {
  using C = LapCfg<DIM, N, BX, BY, BZ>;
  const int base = d == 0 ? C::HOFF_X : d == 1 ? C::HOFF_Y : C::HOFF_Z;
  const int cells = d == 0 ? C::SIDE_CELLS_X : d == 1 ? C::SIDE_CELLS_Y : C::SIDE_CELLS_Z;
  return base + ((s * cells + pos) * 2) * C::LPC;
}

// part: 0 all cells, 1 skip cells touching a ghost side, 2 only those
template <int DIM, int N, int BX, int BY, int BZ>
__global__ void __launch_bounds__(LapCfg<DIM, N, BX, BY, BZ>::THREADS)
laplace_vmult_kernel(const double *__restrict__ u, double *__restrict__ out,
                     const Geo g, const LapTab<N> T, const double tau_scale,
                     const int part) {
  using C = LapCfg<DIM, N, BX, BY, BZ>;
  constexpr int RP = C::RP, LPC = C::LPC, CS = C::CS;
  constexpr int NP = (DIM == 3) ? N * N * N : N * N;
  extern __shared__ double smem[];
  double *buf0 = smem;
  double *buf1 = buf0 + C::BUF;
  double *fbuf = buf1 + C::BUF1;
  double *hbuf = fbuf + C::FBUF;
  double *hraw = buf1;  // aliased: consumed before buf1 is written

  const int nbx = (g.nx + BX - 1) / BX;
  const int nby = (g.ny + BY - 1) / BY;
  const int bid = blockIdx.x;
  const int bx = bid % nbx;
  const int by = (bid / nbx) % nby;
  const int bz = bid / (nbx * nby);
  const int x0 = bx * BX, y0 = by * BY, z0 = bz * BZ;
  const int ex = min(BX, g.nx - x0), ey = min(BY, g.ny - y0);
  const int ez = (DIM == 3) ? min(BZ, g.nz - z0) : 1;
  if (part != 0) {
    const bool touches = (g.mode[0] == kGhost && x0 == 0) ||
                         (g.mode[1] == kGhost && x0 + ex == g.nx);
    if ((part == 1 && touches) || (part == 2 && !touches)) return;
  }
  const int tid = threadIdx.x;

  // ---- phase 0a: own cells -> buf0 (padded rows) ---------------------------
  for (int i = tid; i < C::NC * NP; i += blockDim.x) {
    const int c = i / NP, o = i % NP;
    const int jx = c % BX, jy = (c / BX) % BY, jz = c / (BX * BY);
    const int x = o % N, y = (o / N) % N, z = (DIM == 3) ? o / (N * N) : 0;
    double v = 0.0;
    if (jx < ex && jy < ey && jz < ez) {
      const size_t e = (size_t)(x0 + jx) + (size_t)g.nx * ((y0 + jy) + (size_t)g.ny * (z0 + jz));
      v = u[e * NP + o];
    }
    buf0[c * CS + (z * N + y) * RP + x] = v;
  }
  // ---- phase 0b: raw face functionals of halo cells -> hraw ---------------
  {
    constexpr int NSX = C::SIDE_CELLS_X, NSY = C::SIDE_CELLS_Y, NSZ = C::SIDE_CELLS_Z;
    constexpr int TOT = 2 * (NSX + NSY + NSZ) * LPC;
    for (int i = tid; i < TOT; i += blockDim.x) {
      int r = i;
      int d, s, pos;
      const int p = r % LPC;
      r /= LPC;
      if (r < 2 * NSX) { d = 0; s = r / NSX; pos = r % NSX; }
      else if (r < 2 * (NSX + NSY)) { r -= 2 * NSX; d = 1; s = r / NSY; pos = r % NSY; }
      else { constexpr int NZ1 = NSZ > 0 ? NSZ : 1; r -= 2 * (NSX + NSY); d = 2; s = r / NZ1; pos = r % NZ1; }
      // brick-edge owned cell on this side
      int jx, jy, jz;
      if (d == 0) { jx = s ? ex - 1 : 0; jy = pos % BY; jz = pos / BY; }
      else if (d == 1) { jy = s ? ey - 1 : 0; jx = pos % BX; jz = pos / BX; }
      else { jz = s ? ez - 1 : 0; jx = pos % BX; jy = pos / BX; }
      if (jx >= ex || jy >= ey || jz >= ez) continue;
      NbrInfo nb;
#define DG_RES(DD, SS) resolve_nbr<DD, SS, DIM, N, BX, BY, BZ>(g, u, x0 + jx, y0 + jy, z0 + jz, x0, y0, z0, ex, ey, ez)
      if (d == 0) nb = s ? DG_RES(0, 1) : DG_RES(0, 0);
      else if (d == 1) nb = s ? DG_RES(1, 1) : DG_RES(1, 0);
      else nb = s ? DG_RES(2, 1) : DG_RES(2, 0);
#undef DG_RES
      if (nb.kind != 1) continue;
      // tangential coordinates of face point p
      int a, b;  // (slow, fast) tangential indices
      if (DIM == 3) { a = p / N; b = p % N; } else { a = 0; b = p; }
      const double *src = nb.src;
      int base, stride;
      if (d == 0) { base = (a * N + b) * N; stride = 1; }            // (z,y) line in x
      else if (d == 1) { base = a * N * N + b; stride = N; }          // (z,x) line in y
      else { base = a * N + b; stride = N * N; }                      // (y,x) line in z
      // neighbour on our hi side faces us with its LEFT end, and vice versa
      double gsum = 0.0;
      if (s) {
#pragma unroll
        for (int q = 0; q < N; ++q) gsum += T.dL[q] * src[base + q * stride];
      } else {
#pragma unroll
        for (int q = 0; q < N; ++q) gsum += T.dR[q] * src[base + q * stride];
      }
      const double v = src[base + (s ? 0 : N - 1) * stride];
      const int off = halo_off<DIM, N, BX, BY, BZ>(d, s, pos);
      hraw[off + p] = v;
      hraw[off + LPC + p] = gsum;
    }
  }
  __syncthreads();
  // ---- phase 0c: tangential masses on halo functionals -> hbuf -------------
  {
    constexpr int TOT = C::HSIZE;
    for (int i = tid; i < TOT; i += blockDim.x) {
      const int p = i % LPC;
      double acc;
      if (i < C::HOFF_Y) {
        acc = hraw[i];  // x-sides: raw functionals of u
      } else if (i < C::HOFF_Z) {
        // y-sides: P = M_x applied along the fast tangential index (x)
        const int rowbase = i - p;
        const int a = (DIM == 3) ? p / N : 0, b = (DIM == 3) ? p % N : p;
        acc = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) acc += T.M[b * N + q] * hraw[rowbase + a * N + q];
      } else {
        // z-sides: Q = M_y M_x (tangential (y, x))
        const int rowbase = i - p;
        const int a = p / N, b = p % N;
        acc = 0.0;
#pragma unroll
        for (int qa = 0; qa < N; ++qa) {
          double t = 0.0;
#pragma unroll
          for (int qb = 0; qb < N; ++qb) t += T.M[b * N + qb] * hraw[rowbase + qa * N + qb];
          acc += T.M[a * N + qa] * t;
        }
      }
      hbuf[i] = acc;
    }
  }

  const int l = tid;
  const bool has_line = l < C::NL;
  const int c = has_line ? l / LPC : 0;
  const int t = l % LPC;  // tangential position (slow*N + fast) in each phase
  const int jx = c % BX, jy = (c / BX) % BY, jz = c / (BX * BY);
  const bool active = has_line && jx < ex && jy < ey && jz < ez;
  const int ix = x0 + jx, iy = y0 + jy, iz = z0 + jz;
  const size_t e = (size_t)ix + (size_t)g.nx * (iy + (size_t)g.ny * iz);
  const double hxe = active ? g.hx[ix] : 1.0;
  const double hye = active ? g.hy[iy] : 1.0;
  const double hze = (DIM == 3 && active) ? g.hz[iz] : 2.0;
  const double taue = active ? g.tau[e] : 0.0;
  const double sx = 0.5 * hye * (DIM == 3 ? 0.5 * hze : 1.0);
  const double sy = 0.5 * hxe * (DIM == 3 ? 0.5 * hze : 1.0);
  const double sz = 0.25 * hxe * hye;
  double v[N], w[N];

  // generic: own functionals of the current line -> fbuf; then lifts
  auto store_functionals = [&](const double *line) {
    double g0 = 0.0, g1 = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      g0 += T.dL[q] * line[q];
      g1 += T.dR[q] * line[q];
    }
    fbuf[(c * 4 + 0) * LPC + t] = line[0];
    fbuf[(c * 4 + 1) * LPC + t] = g0;
    fbuf[(c * 4 + 2) * LPC + t] = line[N - 1];
    fbuf[(c * 4 + 3) * LPC + t] = g1;
  };
  // add s * lifts of direction d into acc[] given own line data `line`
  auto add_lifts = [&](auto dconst, const double *line, double h, double sfac,
                       double *acc) {
    constexpr int d = decltype(dconst)::value;
    double g0 = 0.0, g1 = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      g0 += T.dL[q] * line[q];
      g1 += T.dR[q] * line[q];
    }
    auto one_side = [&](auto sconst) {
      constexpr int s = decltype(sconst)::value;
      const NbrInfo nb = resolve_nbr<d, s, DIM, N, BX, BY, BZ>(g, u, ix, iy, iz,
                                                                x0, y0, z0, ex, ey, ez);
      double vn = 0.0, gn = 0.0;
      if (nb.kind == 0) {
        // neighbour's facing end: its left end if it is our +side neighbour
        vn = fbuf[(nb.cb * 4 + (s ? 0 : 2)) * LPC + t];
        gn = fbuf[(nb.cb * 4 + (s ? 1 : 3)) * LPC + t];
      } else if (nb.kind == 1) {
        int pos;
        if (d == 0) pos = jy + BY * jz;
        else if (d == 1) pos = jx + BX * jz;
        else pos = jx + BX * jy;
        const int off = halo_off<DIM, N, BX, BY, BZ>(d, s, pos);
        vn = hbuf[off + t];
        gn = hbuf[off + LPC + t];
      }
      const double tau = tau_scale * (nb.kind <= 1 ? fmax(taue, nb.tau) : taue);
      double cv, cd;
      sip_coeffs(nb.kind, s, s ? line[N - 1] : line[0], s ? g1 : g0, vn, gn, h,
                 nb.h, tau, cv, cd);
      cv *= sfac;
      cd *= sfac;
      acc[s ? N - 1 : 0] += cv;
#pragma unroll
      for (int q = 0; q < N; ++q) acc[q] += cd * (s ? T.dR[q] : T.dL[q]);
    };
    one_side(std::integral_constant<int, 0>());
    one_side(std::integral_constant<int, 1>());
  };

  // ---- phase X: x-lines of u ----------------------------------------------
  const int ta = (DIM == 3) ? t / N : 0, tb = (DIM == 3) ? t % N : t;
  const int xbase = c * CS + (ta * N + tb) * RP;  // (z, y) line along x
  if (has_line) {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = buf0[xbase + q];
    store_functionals(v);
  }
  __syncthreads();
  if (active) {
    const double kx = sx * 2.0 / hxe;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        a += T.K[i * N + q] * v[q];
        b += T.M[i * N + q] * v[q];
      }
      w[i] = kx * a;
      buf0[xbase + i] = b;  // P = M_x u (own line only)
    }
    add_lifts(std::integral_constant<int, 0>(), v, hxe, sx, w);
#pragma unroll
    for (int i = 0; i < N; ++i) buf1[xbase + i] = w[i];
  }
  __syncthreads();
  // ---- phase Y: y-lines of P and T ------------------------------------------
  const int ybase = c * CS + ta * N * RP + tb;  // (z, x) line along y, stride RP
  if (has_line) {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = buf0[ybase + q * RP];
    store_functionals(v);
  }
  __syncthreads();
  if (active) {
    double tl[N];
#pragma unroll
    for (int q = 0; q < N; ++q) tl[q] = buf1[ybase + q * RP];
    const double ky = sy * 2.0 / hye;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        a += T.K[i * N + q] * v[q];
        b += T.M[i * N + q] * tl[q];
      }
      w[i] = b + ky * a;
    }
    add_lifts(std::integral_constant<int, 1>(), v, hye, sy, w);
    if (DIM == 2) {
      // out[e][y][x]: this y-line is x = tb
#pragma unroll
      for (int i = 0; i < N; ++i) out[e * NP + i * N + tb] = w[i];
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double b = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) b += T.M[i * N + q] * v[q];
        buf0[ybase + i * RP] = b;  // Q = M_y P
        buf1[ybase + i * RP] = w[i];  // G
      }
    }
  }
  if (DIM == 2) return;
  __syncthreads();
  // ---- phase Z: z-lines of Q and G --------------------------------------------
  const int zbase = c * CS + ta * RP + tb;  // (y, x) line along z, stride N*RP
  if (has_line) {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = buf0[zbase + q * N * RP];
    store_functionals(v);
  }
  __syncthreads();
  if (active) {
    double gl[N];
#pragma unroll
    for (int q = 0; q < N; ++q) gl[q] = buf1[zbase + q * N * RP];
    const double kz = sz * 2.0 / hze;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        a += T.K[i * N + q] * v[q];
        b += T.M[i * N + q] * gl[q];
      }
      w[i] = b + kz * a;
    }
    add_lifts(std::integral_constant<int, 2>(), v, hze, sz, w);
#pragma unroll
    for (int i = 0; i < N; ++i) out[e * NP + (i * N + ta) * N + tb] = w[i];
  }
}

}  // namespace dg
