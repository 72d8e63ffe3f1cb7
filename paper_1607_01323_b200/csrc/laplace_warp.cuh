// Barrier-free SIPG Laplace vmult (3D, n = k+1 <= 5), fp64, sm_100a.
//
// Same separable operator as laplace.cuh (reference operators.py:187-238):
//   out = M_z [ M_y (s_x Kh_x u + s_x Lx) + s_y Kh_y P + s_y Ly ]
//         + s_z Kh_z Q + s_z Lz,      P = M_x u, Q = M_y P
// but organised for throughput on B200:
//  * the CTA's brick of cells is TMA-bulk-copied into shared memory once and
//    stays read-only -- the only CTA-wide barrier of the kernel;
//  * each warp then processes whole cells on its own (one lane per line,
//    32/n^2 cells per warp step): the x->y->z transposes go through a
//    warp-private scratch with __syncwarp only, and the face functionals of
//    neighbour cells are recomputed by the warp from the read-only brick
//    (shared memory) or, across the brick surface, from L2 -- there is no
//    cross-warp exchange and warps never wait for each other;
//  * every 1D product runs in even-odd (centro-symmetric) form.
// Each output DoF is written once by its own cell; no atomics.
#pragma once
#include "laplace.cuh"

namespace dg {

template <int N, int BX, int BY, int BZ, int NW>
struct WarpLapCfg {
  static constexpr int NP = N * N * N;
  static constexpr int LPC = N * N;          // lines (lanes) per cell
  static constexpr int CPW = 32 / LPC;       // cells per warp step
  static constexpr int RP = row_pitch<N>();  // scratch row pitch
  static constexpr int CS = N * N * RP;      // scratch cell stride
  static constexpr int NC = BX * BY * BZ;
  static constexpr int THREADS = 32 * NW;
  // shared: brick (NC*NP) | per warp: A, B (CPW*CS each), X (CPW*4*LPC), X2
  static constexpr int WARP_SCR = 2 * CPW * CS + 2 * CPW * 4 * LPC;
  static constexpr int OFF_BAR = NC * NP + NW * WARP_SCR;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(OFF_BAR + 1);
};

// neighbour of the own cell across side (D, S) as a data pointer: brick
// (shared) or global; h and tau of the neighbour; kind as in NbrInfo
struct NbrPtr {
  int kind;
  const double *p;
  double h, tau;
};

template <int D, int S, int N, int BX, int BY, int BZ>
__device__ __forceinline__ NbrPtr nbr_ptr(const Geo &g, const double *u, const double *brick,
                                          int ix, int iy, int iz, int x0, int y0, int z0, int ex,
                                          int ey, int ez) {
  constexpr int NP = N * N * N;
  const NbrInfo nb = resolve_nbr<D, S, 3, N, BX, BY, BZ>(g, u, ix, iy, iz, x0, y0, z0, ex, ey, ez);
  NbrPtr r;
  r.kind = nb.kind;
  r.h = nb.h;
  r.tau = nb.tau;
  r.p = nb.kind == 0 ? brick + nb.cb * NP : nb.src;
  return r;
}

template <int N, int BX, int BY, int BZ, int NW>
__global__ void __launch_bounds__(32 * NW, 3)
laplace_warp_kernel(const double *__restrict__ u, double *__restrict__ out, const Geo g,
                    const LapTab<N> T, const double tau_scale, const int part) {
  using C = WarpLapCfg<N, BX, BY, BZ, NW>;
  constexpr int NP = C::NP, LPC = C::LPC, CPW = C::CPW, RP = C::RP, CS = C::CS;
  constexpr int H = N / 2, NE = (N + 1) / 2;
  constexpr int HO = H > 0 ? H : 1;
  extern __shared__ double smem[];
  double *brick = smem;
  const int x0 = blockIdx.x * BX, y0 = blockIdx.y * BY, z0 = blockIdx.z * BZ;
  const int ex = min(BX, g.nx - x0), ey = min(BY, g.ny - y0), ez = min(BZ, g.nz - z0);
  if (part != 0) {
    const bool touches = (g.mode[0] == kGhost && x0 == 0) || (g.mode[1] == kGhost && x0 + ex == g.nx);
    if ((part == 1 && touches) || (part == 2 && !touches)) return;
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- the brick -> shared memory (rows of x-adjacent cells are contiguous) -
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
  constexpr int ROW = BX * NP;
  const bool tma = !(ex & 1) && !(g.nx & 1) && ((reinterpret_cast<uintptr_t>(u) & 15) == 0) &&
                   ((ROW * sizeof(double)) % 16 == 0);
  if (tma) {
    if (tid == 0) {
      mbar_init(bar, 1);
      int rows = 0;
      for (int r = 0; r < BY * BZ; ++r)
        if (r % BY < ey && r / BY < ez) ++rows;
      mbar_expect_tx(bar, (uint32_t)(rows * ex * NP * sizeof(double)));
      for (int r = 0; r < BY * BZ; ++r) {
        const int jy = r % BY, jz = r / BY;
        if (jy >= ey || jz >= ez) continue;
        const size_t e0 = (size_t)x0 + (size_t)g.nx * ((y0 + jy) + (size_t)g.ny * (z0 + jz));
        bulk_g2s(brick + r * ROW, u + e0 * NP, (uint32_t)(ex * NP * sizeof(double)), bar);
      }
    }
    __syncthreads();  // barrier init visible before anyone waits
    mbar_wait(bar, 0);
  } else {
    for (int i = tid; i < C::NC * NP; i += blockDim.x) {
      const int r = i / ROW, w = i - r * ROW;
      const int jx = w / NP;
      const int jy = r % BY, jz = r / BY;
      double v = 0.0;
      if (jx < ex && jy < ey && jz < ez)
        v = u[((size_t)x0 + (size_t)g.nx * ((y0 + jy) + (size_t)g.ny * (z0 + jz))) * NP + w];
      brick[i] = v;
    }
    __syncthreads();
  }

  // ---- per-warp scratch ------------------------------------------------------
  double *wA = smem + C::NC * NP + warp * C::WARP_SCR;  // P, then Q   [cell][z][y][RP]
  double *wB = wA + CPW * CS;                            // T, then G
  double *wX = wB + CPW * CS;                            // neighbour raw functionals
  double *wX2 = wX + CPW * 4 * LPC;                      // after M_x (z faces)
  const int cl = lane / LPC, p = lane - cl * LPC;
  const int a = p / N, b = p - (p / N) * N;  // (slow, fast) tangential index
  const bool lane_ok = cl < CPW;

  for (int grp = warp; grp * CPW < C::NC; grp += NW) {
    const int c = grp * CPW + (lane_ok ? cl : 0);
    const int jx = c % BX, jy = (c / BX) % BY, jz = c / (BX * BY);
    const bool active = lane_ok && c < C::NC && jx < ex && jy < ey && jz < ez;
    const int ix = x0 + jx, iy = y0 + jy, iz = z0 + jz;
    const size_t e = (size_t)ix + (size_t)g.nx * (iy + (size_t)g.ny * iz);
    double h0 = 1.0, h1 = 1.0, h2 = 1.0, taue = 0.0;
    if (active) {
      h0 = g.hx[ix];
      h1 = g.hy[iy];
      h2 = g.hz[iz];
      taue = g.tau[e];
    }
    const double *own = brick + c * NP;
    double *sA = wA + (lane_ok ? cl : 0) * CS, *sB = wB + (lane_ok ? cl : 0) * CS;
    double *sX = wX + (lane_ok ? cl : 0) * 4 * LPC, *sX2 = wX2 + (lane_ok ? cl : 0) * 4 * LPC;
    double v[N], ev[NE], ov[HO], E[NE], O[HO], y[N];

    // SIP lift of direction D into E/O given own line functionals and the
    // neighbour's (vn, gn) per side (operators.py:209-237); sfac = s_D
    auto lifts = [&](auto dconst, double hd, double sfac, double v0, double g0, double v1,
                     double g1, const NbrPtr *nb, const double *vn, const double *gn) {
      constexpr int D = decltype(dconst)::value;
      (void)D;
      const double hi = 1.0 / hd;
      double cv[2], cd[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double sg = s ? -1.0 : 1.0;
        const double vo = s ? v1 : v0, go = s ? g1 : g0;
        if (nb[s].kind <= 1) {
          const double tau = tau_scale * fmax(taue, nb[s].tau);
          const double hni = 1.0 / nb[s].h;
          cv[s] = tau * (vo - vn[s]) + sg * (hi * go + hni * gn[s]);
          cd[s] = sg * hi * (vo - vn[s]);
        } else if (nb[s].kind == kBndNeumann) {
          const double tau = tau_scale * taue;
          cv[s] = 2.0 * (tau * vo + sg * hi * go);
          cd[s] = 2.0 * sg * hi * vo;
        } else {
          cv[s] = 0.0;
          cd[s] = 0.0;
        }
        cv[s] *= sfac;
        cd[s] *= sfac;
      }
      E[0] += 0.5 * (cv[0] + cv[1]);
      O[0] += 0.5 * (cv[0] - cv[1]);
      const double dm = cd[0] - cd[1], dp = cd[0] + cd[1];
#pragma unroll
      for (int i = 0; i < NE; ++i) E[i] += T.dLe[i] * dm;
#pragma unroll
      for (int i = 0; i < H; ++i) O[i] += T.dLo[i] * dp;
    };
    auto own_functionals = [&](double &v0, double &g0, double &v1, double &g1) {
      double ge = 0.0, go = 0.0;
#pragma unroll
      for (int j = 0; j < NE; ++j) ge += T.dLe[j] * ev[j];
#pragma unroll
      for (int j = 0; j < H; ++j) go += T.dLo[j] * ov[j];
      v0 = v[0];
      v1 = v[N - 1];
      g0 = ge + go;
      g1 = go - ge;
    };
    // raw functionals of a neighbour line facing side s (its opposite end)
    auto raw_func = [&](const double *line, int stride, int s, double &vr, double &gr) {
      double x[N];
#pragma unroll
      for (int q = 0; q < N; ++q) x[q] = line[q * stride];
      gr = 0.0;
      if (s) {
        vr = x[0];
#pragma unroll
        for (int q = 0; q < N; ++q) gr += T.dL[q] * x[q];
      } else {
        vr = x[N - 1];
#pragma unroll
        for (int q = 0; q < N; ++q) gr += T.dR[q] * x[q];
      }
    };
    NbrPtr nb[2];

    // ================= phase X: x-lines (z = a, y = b) of u ==================
    double v0, g0, v1, g1, vn[2], gn[2];
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = own[(a * N + b) * N + q];
    eo_split<N>(v, ev, ov);
    own_functionals(v0, g0, v1, g1);
    if (active) {
      nb[0] = nbr_ptr<0, 0, N, BX, BY, BZ>(g, u, brick, ix, iy, iz, x0, y0, z0, ex, ey, ez);
      nb[1] = nbr_ptr<0, 1, N, BX, BY, BZ>(g, u, brick, ix, iy, iz, x0, y0, z0, ex, ey, ez);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        vn[s] = gn[s] = 0.0;
        if (nb[s].kind <= 1) raw_func(nb[s].p + (a * N + b) * N, 1, s, vn[s], gn[s]);
      }
      eo_apply<N, false>(T.Me, T.Mo, ev, ov, 1.0, E, O);
      eo_merge<N>(E, O, y);
#pragma unroll
      for (int i = 0; i < N; ++i) sA[(a * N + b) * RP + i] = y[i];  // P = M_x u
      eo_apply<N, false>(T.Ke, T.Ko, ev, ov, 0.5 * h1 * h2 / h0, E, O);
      lifts(std::integral_constant<int, 0>(), h0, 0.25 * h1 * h2, v0, g0, v1, g1, nb, vn, gn);
      eo_merge<N>(E, O, y);
#pragma unroll
      for (int i = 0; i < N; ++i) sB[(a * N + b) * RP + i] = y[i];  // T
    }
    __syncwarp();

    // ================= phase Y: y-lines (z = a, x = b) of P and T =============
    // neighbour P-functionals: raw y-functionals per (z, x), then M_x across
    // the lanes of the same z through the warp scratch
    if (active) {
      nb[0] = nbr_ptr<1, 0, N, BX, BY, BZ>(g, u, brick, ix, iy, iz, x0, y0, z0, ex, ey, ez);
      nb[1] = nbr_ptr<1, 1, N, BX, BY, BZ>(g, u, brick, ix, iy, iz, x0, y0, z0, ex, ey, ez);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        double vr = 0.0, gr = 0.0;
        if (nb[s].kind <= 1) raw_func(nb[s].p + a * N * N + b, N, s, vr, gr);
        sX[(s * 2 + 0) * LPC + p] = vr;
        sX[(s * 2 + 1) * LPC + p] = gr;
      }
    }
    __syncwarp();
    if (active) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        double av = 0.0, ag = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          av += T.M[b * N + q] * sX[(s * 2 + 0) * LPC + a * N + q];
          ag += T.M[b * N + q] * sX[(s * 2 + 1) * LPC + a * N + q];
        }
        vn[s] = av;
        gn[s] = ag;
      }
      double tl[N], te[NE], to[HO];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        v[q] = sA[(a * N + q) * RP + b];
        tl[q] = sB[(a * N + q) * RP + b];
      }
      eo_split<N>(v, ev, ov);
      eo_split<N>(tl, te, to);
      own_functionals(v0, g0, v1, g1);
      eo_apply<N, false>(T.Me, T.Mo, ev, ov, 1.0, E, O);  // Q = M_y P
      eo_merge<N>(E, O, y);
#pragma unroll
      for (int i = 0; i < N; ++i) sA[(a * N + i) * RP + b] = y[i];
      eo_apply<N, false>(T.Me, T.Mo, te, to, 1.0, E, O);  // G = M_y T
      eo_apply<N, true>(T.Ke, T.Ko, ev, ov, 0.5 * h0 * h2 / h1, E, O);
      lifts(std::integral_constant<int, 1>(), h1, 0.25 * h0 * h2, v0, g0, v1, g1, nb, vn, gn);
      eo_merge<N>(E, O, y);
#pragma unroll
      for (int i = 0; i < N; ++i) sB[(a * N + i) * RP + b] = y[i];
    }
    __syncwarp();

    // ================= phase Z: z-lines (y = a, x = b) of Q and G =============
    if (active) {
      nb[0] = nbr_ptr<2, 0, N, BX, BY, BZ>(g, u, brick, ix, iy, iz, x0, y0, z0, ex, ey, ez);
      nb[1] = nbr_ptr<2, 1, N, BX, BY, BZ>(g, u, brick, ix, iy, iz, x0, y0, z0, ex, ey, ez);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        double vr = 0.0, gr = 0.0;
        if (nb[s].kind <= 1) raw_func(nb[s].p + a * N + b, N * N, s, vr, gr);
        sX[(s * 2 + 0) * LPC + p] = vr;
        sX[(s * 2 + 1) * LPC + p] = gr;
      }
    }
    __syncwarp();
    if (active) {  // M_x along the fast index
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int w2 = 0; w2 < 2; ++w2) {
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < N; ++q) acc += T.M[b * N + q] * sX[(s * 2 + w2) * LPC + a * N + q];
          sX2[(s * 2 + w2) * LPC + p] = acc;
        }
    }
    __syncwarp();
    if (active) {  // M_y along the slow index
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        double av = 0.0, ag = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          av += T.M[a * N + q] * sX2[(s * 2 + 0) * LPC + q * N + b];
          ag += T.M[a * N + q] * sX2[(s * 2 + 1) * LPC + q * N + b];
        }
        vn[s] = av;
        gn[s] = ag;
      }
      double gl[N], ge[NE], go[HO];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        v[q] = sA[(q * N + a) * RP + b];
        gl[q] = sB[(q * N + a) * RP + b];
      }
      eo_split<N>(v, ev, ov);
      eo_split<N>(gl, ge, go);
      own_functionals(v0, g0, v1, g1);
      eo_apply<N, false>(T.Me, T.Mo, ge, go, 1.0, E, O);  // M_z G
      eo_apply<N, true>(T.Ke, T.Ko, ev, ov, 0.5 * h0 * h1 / h2, E, O);
      lifts(std::integral_constant<int, 2>(), h2, 0.25 * h0 * h1, v0, g0, v1, g1, nb, vn, gn);
      eo_merge<N>(E, O, y);
#pragma unroll
      for (int i = 0; i < N; ++i) out[e * NP + (i * N + a) * N + b] = y[i];
    }
    __syncwarp();
  }
}

}  // namespace dg
