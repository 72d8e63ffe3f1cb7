// SIP Laplace vmult, 3D Cartesian cells: warp-column kernel (sm_100a, fp64).
// Same operator, z-first factorisation, plane-per-thread sweeps, TMA ring,
// look-ahead and face coefficients as laplace7.cuh (reference
// operators.py:187-238), but every WARP marches its own column -- a TX x TY
// tile of cells (TX * TY * N <= 32 lanes: lane = cell * N + plane) over a
// range of z layers -- with its own ring slots, transpose buffer, halo block
// and mbarriers.  All exchanges (the Z -> XY transpose, x / y neighbour face
// functionals inside the tile) stay inside the warp, so there is no CTA
// barrier at all: warps never wait for each other, and warps of a persistent
// CTA pull columns from a global work counter (dynamic balance across the
// SM sub-partitions).  The price: a smaller tile, so more neighbour cells are
// read as halo (from L2: the neighbouring columns are processed at the same
// time) -- all of it inside the z phase, where registers are free.
#pragma once
#include "laplace7.cuh"

namespace dg {

template <int N, int TX, int TY, int NRING, int WPB>
struct Lap9Cfg {
  static constexpr int NCW = TX * TY;  // cells per warp tile
  static_assert(NCW * N <= 32, "one warp per tile");
  static constexpr bool IDLE = NCW * N < 32;
  static constexpr int NP = N * N * N;
  static constexpr int CSTR = L7Stride<N>::value;
  static constexpr int LAYER = (((NCW + (IDLE ? 1 : 0)) * CSTR + 1) / 2) * 2;
  static constexpr int LCMAX = 32;
  static constexpr int HXN = 2 * TY * N * N * 2;  // [side][jy][y][z][v|g]
  static constexpr int HYN = 2 * TX * N * N * 2;  // [side][jx][x][z][v|g]
  static constexpr int CCS = 15;
  // per-warp region (doubles)
  static constexpr int OFF_R = NRING * LAYER;
  static constexpr int OFF_HX = OFF_R + LAYER;
  static constexpr int OFF_HY = OFF_HX + HXN;
  static constexpr int OFF_CC = OFF_HY + HYN;
  static constexpr int OFF_ZD = OFF_CC + (NCW + 1) * CCS;
  static constexpr int OFF_ZERO = OFF_ZD + 4 * (LCMAX + 2);
  static constexpr int OFF_BAR = OFF_ZERO + 2 * N * N;
  static constexpr int WSTRIDE = ((OFF_BAR + NRING + 1) / 2) * 2;  // 16-byte multiple
  static constexpr int THREADS = 32 * WPB;
  static constexpr size_t SMEM = sizeof(double) * (size_t)WSTRIDE * WPB;
  static constexpr int HITEMS = 2 * N * (TX + TY);
  static constexpr int HROWS = 2 * TX * N * 2;
};

template <int N, int TX, int TY, int NRING, int WPB>
__global__ void __launch_bounds__(32 * WPB, 1)
laplace9_kernel(const double *__restrict__ u, double *__restrict__ out, const Geo g,
                const __grid_constant__ LapTab<N> T, const double ts, const int part,
                const int zlo, const int zhi, const int lc, const int ntx, const int nty,
                const int nunits, unsigned *__restrict__ counter) {
  using C = Lap9Cfg<N, TX, TY, NRING, WPB>;
  constexpr int NCW = C::NCW, NP = C::NP, CSTR = C::CSTR, H = N / 2, NE = (N + 1) / 2;
  constexpr int HO = H > 0 ? H : 1;
  constexpr int N2 = N * N;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *const wbase = smem + (size_t)warp * C::WSTRIDE;
  double *const ring = wbase;
  double *const rbuf = wbase + C::OFF_R;
  double *const hxb = wbase + C::OFF_HX;
  double *const hyb = wbase + C::OFF_HY;
  double *const cc = wbase + C::OFF_CC;
  double *const zd = wbase + C::OFF_ZD;
  const double *const zero = wbase + C::OFF_ZERO;
  uint64_t *const bar = reinterpret_cast<uint64_t *>(wbase + C::OFF_BAR);
  for (int i = lane; i < 2 * N * N; i += 32) wbase[C::OFF_ZERO + i] = 0.0;
  if (lane == 0)
    for (int i = 0; i < NRING; ++i) mbar_init(&bar[i], 1);
  __syncwarp();

  const bool live = lane < NCW * N;
  const int c = live ? lane / N : NCW - 1;   // idle lanes shadow the last cell ...
  const int s = live ? lane % N : N - 1;
  const int cs = live ? c : NCW;             // ... on a scratch slot
  const int jx = c % TX, jy = c / TX;
  const size_t nxy = (size_t)g.nx * g.ny;
  const bool aligned = !(reinterpret_cast<uintptr_t>(u) & 15) && !(reinterpret_cast<uintptr_t>(out) & 15);
  unsigned uphase[NRING];  // completed phases per slot (parity of the next wait)
#pragma unroll
  for (int i = 0; i < NRING; ++i) uphase[i] = 0;

  for (;;) {
    int unit = 0;
    if (lane == 0) unit = (int)atomicAdd(counter, 1u);
    unit = __shfl_sync(FULL, unit, 0);
    if (unit >= nunits) break;
    // ---- unit: tile (tx, ty) x z-chunk -----------------------------------
    const int tix = unit % ntx;
    const int tiy = (unit / ntx) % nty;
    const int chunk = unit / (ntx * nty);
    const int x0 = tix * TX, y0 = tiy * TY;
    const int ex = min(TX, g.nx - x0), ey = min(TY, g.ny - y0);
    const int z0 = zlo + chunk * lc, z1 = min(zhi, z0 + lc);
    if (z0 >= z1) continue;
    if (part != 0) {
      const bool touches = (g.mode[0] == kGhost && x0 == 0) || (g.mode[1] == kGhost && x0 + ex == g.nx);
      if ((part == 1 && touches) || (part == 2 && !touches)) continue;
    }
    const int nlay = z1 - z0;
    const int ix = x0 + min(jx, ex - 1), iy = y0 + min(jy, ey - 1);

    // ---- neighbour kinds / lanes, column constants, z data ------------------
    int kx0, kx1, ky0, ky1, lx0, lx1, ly0, ly1;
    {
      int nb = 0;
      kx0 = kind7<0>(g, 0, ix, g.nx, x0, ex, nb);
      lx0 = (nb + TX * jy) * N + s;
      kx1 = kind7<1>(g, 0, ix, g.nx, x0, ex, nb);
      lx1 = (nb + TX * jy) * N + s;
      ky0 = kind7<0>(g, 1, iy, g.ny, y0, ey, nb);
      ly0 = (jx + TX * nb) * N + s;
      ky1 = kind7<1>(g, 1, iy, g.ny, y0, ey, nb);
      ly1 = (jx + TX * nb) * N + s;
      if (kx0 != 0) lx0 = lane;
      if (kx1 != 0) lx1 = lane;
      if (ky0 != 0) ly0 = lane;
      if (ky1 != 0) ly1 = lane;
    }
    if (live && s == 0) {
      const double *ax = g.ax[0] + 4 * ix, *ay = g.ax[1] + 4 * iy;
      const double hx = ax[0], hxi = ax[1], tx = ax[2];
      const double hy = ay[0], hyi = ay[1], ty = ay[2];
      double *q = cc + c * C::CCS;
      q[0] = 0.25 * hx * hy;
      q[1] = 0.5 * hx * hy;
      q[2] = tx + ty;
      q[3] = hy;
      q[4] = hxi;
      q[5] = fmax(tx, ax[-4 + 2]) + ty;
      q[6] = fmax(tx, ax[4 + 2]) + ty;
      q[7] = ax[-4 + 1];
      q[8] = ax[4 + 1];
      q[9] = hx;
      q[10] = hyi;
      q[11] = tx + fmax(ty, ay[-4 + 2]);
      q[12] = tx + fmax(ty, ay[4 + 2]);
      q[13] = ay[-4 + 1];
      q[14] = ay[4 + 1];
    }
    for (int i = lane; i < 4 * (nlay + 2); i += 32) zd[i] = g.ax[2][4 * (z0 - 1) + i];

    // ---- ring (positions: 0 below, 1..nlay column, nlay + 1 above) ----------
    auto layer_of = [&](int r) -> int {
      const int z = z0 + r - 1;
      if (z < 0) return g.mode[4] == kWrap ? g.nz - 1 : -1;
      if (z >= g.nz) return g.mode[5] == kWrap ? 0 : -1;
      return z;
    };
    const bool rows_ok = (N & 1) ? (!(g.nx & 1) && !(ex & 1)) : true;
    const bool tma = rows_ok && aligned;
    auto issue = [&](int r) {
      if (r > nlay + 1) return;
      const int lay = layer_of(r);
      uint64_t *b = &bar[r % NRING];
      if (lay < 0) {
        if (tma && lane == 0) mbar_arrive(b);
        return;
      }
      double *dst = ring + (r % NRING) * C::LAYER;
      if (tma) {
        if (lane == 0) mbar_expect_tx(b, (uint32_t)(ex * ey * NP * sizeof(double)));
        __syncwarp();
        const int nitem = (N & 1) ? ey : ex * ey;
        for (int i = lane; i < nitem; i += 32) {
          const int xx = (N & 1) ? 0 : i % ex, yy = (N & 1) ? i : i / ex;
          const size_t e0 = (size_t)x0 + xx + (size_t)g.nx * (y0 + yy) + nxy * lay;
          bulk_g2s(dst + (xx + TX * yy) * CSTR, u + e0 * NP,
                   (uint32_t)(((N & 1) ? ex : 1) * NP * sizeof(double)), b);
        }
      } else {
        for (int i = lane; i < ex * ey * NP; i += 32) {
          const int cl = i / NP, w = i - cl * NP;
          const int xx = cl % ex, yy = cl / ex;
          dst[(xx + TX * yy) * CSTR + w] =
              u[((size_t)x0 + xx + (size_t)g.nx * (y0 + yy) + nxy * lay) * NP + w];
        }
      }
    };
    // the r-th position of THIS unit uses slot r % NRING for the
    // (uphase[slot])-th time since the kernel started
    int pos_phase[NRING];
#pragma unroll
    for (int i = 0; i < NRING; ++i) pos_phase[i] = (int)uphase[i];
    auto wait_slot = [&](int r) {
      const int sl = r % NRING;
      if (tma && layer_of(r) >= 0) mbar_wait(&bar[sl], (pos_phase[sl] + r / NRING) & 1);
    };

    // ---- halo (laplace7.cuh items, two rounds over the 32 lanes) -----------
    int hside = 0, hrow = 0, hpos = 0, htrace = 0;
    bool hx_item = false;
    double hreg[N][N];
    const double *hsrc = nullptr;
    auto halo_load = [&](int it, int lay) {
      hsrc = nullptr;
      htrace = 0;
      if (it >= C::HITEMS || lay < 0) return;
      hx_item = it < 2 * TY * N;
      const int i2 = hx_item ? it : it - 2 * TY * N;
      const int per = hx_item ? TY * N : TX * N;
      hside = i2 / per;
      const int rem = i2 - hside * per;
      hrow = rem / N;
      hpos = rem - hrow * N;
      if (hx_item) {
        if (hrow >= ey) return;
        const int yy = y0 + hrow;
        int nc = hside ? x0 + ex : x0 - 1;
        if (nc < 0 || nc >= g.nx) {
          const int m = g.mode[hside];
          if (m == kWrap) nc = hside ? 0 : g.nx - 1;
          else if (m == kGhost) {
            htrace = g.ghost_traces;
            hsrc = g.ghost[hside] + ((size_t)yy + (size_t)g.ny * lay) * (htrace ? 2 * N2 : NP);
          } else return;
        }
        if (!hsrc) {
          if (nc >= x0 && nc < x0 + ex) return;
          hsrc = u + ((size_t)nc + (size_t)g.nx * yy + nxy * lay) * NP;
        }
      } else {
        if (hrow >= ex) return;
        const int xx = x0 + hrow;
        int nc = hside ? y0 + ey : y0 - 1;
        if (nc < 0 || nc >= g.ny) {
          const int m = g.mode[2 + hside];
          if (m == kWrap) nc = hside ? 0 : g.ny - 1;
          else return;
        }
        if (nc >= y0 && nc < y0 + ey) return;
        hsrc = u + ((size_t)xx + (size_t)g.nx * nc + nxy * lay) * NP;
      }
      if (htrace) {
#pragma unroll
        for (int z = 0; z < N; ++z) {
          hreg[z][0] = __ldg(hsrc + (z * N + hpos) * 2);
          hreg[z][1] = __ldg(hsrc + (z * N + hpos) * 2 + 1);
        }
        return;
      }
#pragma unroll
      for (int z = 0; z < N; ++z)
#pragma unroll
        for (int q = 0; q < N; ++q)
          hreg[z][q] = __ldg(hsrc + z * N2 + (hx_item ? hpos * N + q : q * N + hpos));
    };
    auto halo_stage1 = [&]() {
      if (!hsrc) return;
      double v[N], gg[N], mv[N], mg[N];
#pragma unroll
      for (int z = 0; z < N; ++z) {
        double e[NE], o[HO], g0, g1;
        eo_split<N>(hreg[z], e, o);
        l7_ends<N>(T, e, o, g0, g1);
        v[z] = htrace ? hreg[z][0] : (hside ? hreg[z][0] : hreg[z][N - 1]);
        gg[z] = htrace ? hreg[z][1] : (hside ? g0 : g1);
      }
      l7_mass<N>(T, v, mv);
      l7_mass<N>(T, gg, mg);
      double *hp = hx_item ? hxb + ((hside * TY + hrow) * N + hpos) * N * 2
                           : hyb + ((hside * TX + hrow) * N + hpos) * N * 2;
#pragma unroll
      for (int z = 0; z < N; ++z) {
        hp[2 * z] = mv[z];
        hp[2 * z + 1] = mg[z];
      }
    };
    auto halo_stage2 = [&]() {  // y halo: M_x along x
      for (int i = lane; i < C::HROWS; i += 32) {
        const int vg = i & 1, rz = i >> 1;
        const int z = rz % N, sj = rz / N;
        if ((sj % TX) >= ex) continue;
        double *row = hyb + sj * N * N * 2 + z * 2 + vg;
        double v[N], y[N];
#pragma unroll
        for (int x = 0; x < N; ++x) v[x] = row[x * N * 2];
        l7_mass<N>(T, v, y);
#pragma unroll
        for (int x = 0; x < N; ++x) row[x * N * 2] = y[x];
      }
    };

    // ---- prologue of the unit -------------------------------------------------
    for (int r = 0; r < NRING; ++r) issue(r);
    if (!tma) __syncwarp();
    double ztv[N], ztg[N];
#pragma unroll
    for (int x = 0; x < N; ++x) {
      ztv[x] = 0.0;
      ztg[x] = 0.0;
    }
    if (layer_of(0) >= 0) {
      wait_slot(0);
      const double *p = ring + cs * CSTR + s * N;
#pragma unroll
      for (int x = 0; x < N; ++x) {
        double w[N], e[NE], o[HO], g0, g1;
#pragma unroll
        for (int z = 0; z < N; ++z) w[z] = p[z * N2 + x];
        eo_split<N>(w, e, o);
        l7_ends<N>(T, e, o, g0, g1);
        ztv[x] = w[N - 1];
        ztg[x] = g1;
      }
    }
    __syncwarp();  // slot 0 consumed (refilled below), cc / zd visible

    // ---- march -------------------------------------------------------------------
    for (int p = 0; p < nlay; ++p) {
      const int r = p + 1;
      const int iz = z0 + p;
      double *const slot = ring + (r % NRING) * C::LAYER;
      const double *az = zd + 4 * (p + 1);
      const double hz = az[0], hzi = az[1], tz = az[2];
      auto refill = [&]() {
        if (tma) bulk_wait_read();  // every lane that issued a store of this slot
        issue(r + NRING - 1);
      };
      if (NRING == 2) {
        refill();
        if (!tma) __syncwarp();
      }
      wait_slot(r);
      const int lay_up = layer_of(r + 1);
      wait_slot(r + 1);
      // ===== z phase: W = M_z u (in place), R = A_z u; halo of THIS layer =====
      halo_load(lane, iz);
      {
        const double *q = cc + c * C::CCS;
        const double sfz = q[0], kz = q[1] * hzi, txy = q[2];
        const double taue = txy + tz;
        const int kz0 = iz == 0 ? (g.mode[4] == kWrap ? 0 : g.mode[4]) : 0;
        const int kz1 = iz == g.nz - 1 ? (g.mode[5] == kWrap ? 0 : g.mode[5]) : 0;
        const Side7 s0 = side7(kz0, txy + fmax(tz, az[-4 + 2]), taue, sfz, hzi, az[-4 + 1], 1.0, ts);
        const Side7 s1 = side7(kz1, txy + fmax(tz, az[4 + 2]), taue, sfz, hzi, az[4 + 1], -1.0, ts);
        double *up = slot + cs * CSTR + s * N;
        double *rp = rbuf + cs * CSTR + s * N;
        const double *lp = ring + ((r + 1) % NRING) * C::LAYER + cs * CSTR + s * N;
        const bool la_ok = lay_up >= 0;
#pragma unroll
        for (int x = 0; x < N; ++x) {
          double w[N], e[NE], o[HO], E[NE], O[HO], g0, g1;
#pragma unroll
          for (int z = 0; z < N; ++z) w[z] = up[z * N2 + x];
          double la0 = lp[x], lg = T.dL[0] * la0;
#pragma unroll
          for (int z = 1; z < N; ++z) lg += T.dL[z] * lp[z * N2 + x];
          const double vn1 = la_ok ? la0 : 0.0, gn1 = la_ok ? lg : 0.0;
          eo_split<N>(w, e, o);
          l7_ends<N>(T, e, o, g0, g1);
          const double vn0 = ztv[x], gn0 = ztg[x];
          ztv[x] = w[N - 1];
          ztg[x] = g1;
          eo_apply<N, false>(T.Ke, T.Ko, e, o, kz, E, O);
          l7_lift<N>(T, s0, s1, w[0], g0, vn0, gn0, w[N - 1], g1, vn1, gn1, E, O);
          double y[N];
          eo_merge<N>(E, O, y);
#pragma unroll
          for (int z = 0; z < N; ++z) rp[z * N2 + x] = y[z];
          eo_apply<N, false>(T.Me, T.Mo, e, o, 1.0, E, O);
          eo_merge<N>(E, O, y);
#pragma unroll
          for (int z = 0; z < N; ++z) up[z * N2 + x] = y[z];
          if (x == N / 2 && C::HITEMS > 32) {  // halo round 2 (items 32..)
            halo_stage1();
            halo_load(lane + 32, iz);
          }
        }
      }
      halo_stage1();
      if (NRING >= 3) refill();
      __syncwarp();  // W, R, halo stage 1 visible
      halo_stage2();
      __syncwarp();
      // ===== xy phase: T = A_x W + M_x R, V = M_x W; out = M_y T + A_y V =====
      {
        const double *q = cc + c * C::CCS;
        const double hy = q[3], hxi = q[4], hx = q[9], hyi = q[10];
        const double taue = q[2] + tz;
        double Tp[N][N], Vp[N][N];
        {
          const double sfx = 0.25 * hy * hz, kx = 0.5 * hy * hz * hxi;
          const Side7 s0 = side7(kx0, q[5] + tz, taue, sfx, hxi, q[7], 1.0, ts);
          const Side7 s1 = side7(kx1, q[6] + tz, taue, sfx, hxi, q[8], -1.0, ts);
          const double *wp = slot + cs * CSTR + s * N2;
          const double *rp = rbuf + cs * CSTR + s * N2;
          const double *h0 = kx0 == 1 ? hxb + (jy * N) * N * 2 + 2 * s : zero;
          const double *h1 = kx1 == 1 ? hxb + ((TY + jy) * N) * N * 2 + 2 * s : zero;
#pragma unroll
          for (int y = 0; y < N; ++y) {
            double w[N], rr[N], e[NE], o[HO], re[NE], ro[HO], E[NE], O[HO], g0, g1;
#pragma unroll
            for (int x = 0; x < N; ++x) {
              w[x] = wp[y * N + x];
              rr[x] = rp[y * N + x];
            }
            eo_split<N>(w, e, o);
            eo_split<N>(rr, re, ro);
            l7_ends<N>(T, e, o, g0, g1);
            const double v0 = w[0], v1 = w[N - 1];
            const double vn0 = l7_pick(kx0, __shfl_sync(FULL, v1, lx0), h0[y * N * 2]);
            const double gn0 = l7_pick(kx0, __shfl_sync(FULL, g1, lx0), h0[y * N * 2 + 1]);
            const double vn1 = l7_pick(kx1, __shfl_sync(FULL, v0, lx1), h1[y * N * 2]);
            const double gn1 = l7_pick(kx1, __shfl_sync(FULL, g0, lx1), h1[y * N * 2 + 1]);
            eo_apply<N, false>(T.Ke, T.Ko, e, o, kx, E, O);
            eo_apply<N, true>(T.Me, T.Mo, re, ro, 1.0, E, O);
            l7_lift<N>(T, s0, s1, v0, g0, vn0, gn0, v1, g1, vn1, gn1, E, O);
            eo_merge<N>(E, O, Tp[y]);
            eo_apply<N, false>(T.Me, T.Mo, e, o, 1.0, E, O);
            eo_merge<N>(E, O, Vp[y]);
          }
        }
        {
          const double sfy = 0.25 * hx * hz, ky = 0.5 * hx * hz * hyi;
          const Side7 s0 = side7(ky0, q[11] + tz, taue, sfy, hyi, q[13], 1.0, ts);
          const Side7 s1 = side7(ky1, q[12] + tz, taue, sfy, hyi, q[14], -1.0, ts);
          const double *h0 = ky0 == 1 ? hyb + (jx * N) * N * 2 + 2 * s : zero;
          const double *h1 = ky1 == 1 ? hyb + ((TX + jx) * N) * N * 2 + 2 * s : zero;
          double *op = slot + cs * CSTR + s * N2;
#pragma unroll
          for (int x = 0; x < N; ++x) {
            double vc[N], tc[N], e[NE], o[HO], te[NE], to[HO], E[NE], O[HO], g0, g1;
#pragma unroll
            for (int y = 0; y < N; ++y) {
              vc[y] = Vp[y][x];
              tc[y] = Tp[y][x];
            }
            eo_split<N>(vc, e, o);
            eo_split<N>(tc, te, to);
            l7_ends<N>(T, e, o, g0, g1);
            const double v0 = vc[0], v1 = vc[N - 1];
            const double vn0 = l7_pick(ky0, __shfl_sync(FULL, v1, ly0), h0[x * N * 2]);
            const double gn0 = l7_pick(ky0, __shfl_sync(FULL, g1, ly0), h0[x * N * 2 + 1]);
            const double vn1 = l7_pick(ky1, __shfl_sync(FULL, v0, ly1), h1[x * N * 2]);
            const double gn1 = l7_pick(ky1, __shfl_sync(FULL, g0, ly1), h1[x * N * 2 + 1]);
            eo_apply<N, false>(T.Me, T.Mo, te, to, 1.0, E, O);
            eo_apply<N, true>(T.Ke, T.Ko, e, o, ky, E, O);
            l7_lift<N>(T, s0, s1, v0, g0, vn0, gn0, v1, g1, vn1, gn1, E, O);
            double yv[N];
            eo_merge<N>(E, O, yv);
#pragma unroll
            for (int yy = 0; yy < N; ++yy) op[yy * N + x] = yv[yy];
          }
        }
      }
      if (tma) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();  // out complete in the slot
      if (tma) {
        const int nitem = (N & 1) ? ey : ex * ey;
        for (int i = lane; i < nitem; i += 32) {
          const int xx = (N & 1) ? 0 : i % ex, yy = (N & 1) ? i : i / ex;
          const size_t e0 = (size_t)x0 + xx + (size_t)g.nx * (y0 + yy) + nxy * iz;
          bulk_s2g(out + e0 * NP, slot + (xx + TX * yy) * CSTR,
                   (uint32_t)(((N & 1) ? ex : 1) * NP * sizeof(double)));
        }
      } else {
        for (int i = lane; i < ex * ey * NP; i += 32) {
          const int cl = i / NP, w = i - cl * NP;
          const int xx = cl % ex, yy = cl / ex;
          out[((size_t)x0 + xx + (size_t)g.nx * (y0 + yy) + nxy * iz) * NP + w] =
              slot[(xx + TX * yy) * CSTR + w];
        }
        __syncwarp();
      }
    }
    // positions issued for this unit: 0 .. nlay + 1 (the last ones maybe
    // beyond the issue window); account the barrier phases they completed
    const int npos = nlay + 2;
    if (tma) {  // (plain-copy units never touch the barriers)
#pragma unroll
      for (int i = 0; i < NRING; ++i) {
        const int uses = npos > i ? (npos - 1 - i) / NRING + 1 : 0;
        uphase[i] += (unsigned)uses;
      }
    }
    // every position of this unit was waited for (all copies landed); the
    // stores must have read their slots before the next unit refills them
    if (tma) bulk_wait_read();
    __syncwarp();
  }
  bulk_wait_read();
}

}  // namespace dg
