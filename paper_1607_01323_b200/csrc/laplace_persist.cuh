// Persistent, software-pipelined SIPG Laplace vmult (3D), fp64, sm_100a.
//
// Same operator and per-brick algorithm as laplace_vmult_kernel
// (laplace.cuh: separable even-odd sweeps, shared-memory brick, halo face
// functionals), restructured so the per-brick prologue is off the critical
// path: a fixed grid of CTAs (2 per SM) walks the bricks; while brick i is
// computed,
//   * the TMA bulk copy of brick i+1 streams into the second raw buffer,
//   * the face-coefficient table of brick i+1 (neighbour kinds, 1/h, tau:
//     the dependent L2 loads of the setup) is built into the second table
//     slot during the long phase-Y segment.
// Only the halo face functionals (L2 reads of neighbour lines) remain in the
// per-brick critical path.
#pragma once
#include "laplace.cuh"

namespace dg {

template <int N, int BX, int BY, int BZ>
struct PersistCfg {
  using L = LapCfg<3, N, BX, BY, BZ>;
  static constexpr int BUF = L::BUF, FBUF = L::FBUF, HSIZE = L::HSIZE;
  static constexpr int NC = L::NC, NSIDE = 6, SIDEC = 6;
  static constexpr int TAB = SIDEC * NC * NSIDE + 4 * NC;  // one table slot (doubles)
  static constexpr int OFF_RAW0 = 0;
  static constexpr int OFF_RAW1 = BUF;
  static constexpr int OFF_BUF1 = 2 * BUF;
  static constexpr int OFF_FBUF = 3 * BUF;
  static constexpr int OFF_HRAW = OFF_FBUF + FBUF;
  static constexpr int OFF_HBUF = OFF_HRAW + HSIZE;
  static constexpr int OFF_TAB = OFF_HBUF + HSIZE;           // 2 slots
  static constexpr int OFF_BAR = OFF_TAB + 2 * TAB;           // 2 mbarriers
  static constexpr int NDBL = OFF_BAR + 2;
  static constexpr size_t SMEM = sizeof(double) * (size_t)NDBL + sizeof(int) * 2 * NC * NSIDE;
};

struct BrickPos {
  int x0, y0, z0, ex, ey, ez;
};

__device__ __forceinline__ BrickPos brick_pos(const Geo &g, int b, int nbx, int nby, int BX,
                                              int BY, int BZ) {
  BrickPos p;
  const int bx = b % nbx, by = (b / nbx) % nby, bz = b / (nbx * nby);
  p.x0 = bx * BX;
  p.y0 = by * BY;
  p.z0 = bz * BZ;
  p.ex = min(BX, g.nx - p.x0);
  p.ey = min(BY, g.ny - p.y0);
  p.ez = min(BZ, g.nz - p.z0);
  return p;
}

// Source cell of halo slot (d, s, pos) of brick bp by index arithmetic only:
// the neighbour of the slot's brick-edge cell if it lies outside the brick,
// nullptr if inside, a boundary, or the edge cell is idle.
template <int N, int BX, int BY, int BZ>
__device__ __forceinline__ const double *halo_src3(const Geo &g, const double *u, int d, int s,
                                                   int pos, const BrickPos &bp) {
  constexpr int NP = N * N * N;
  int jx, jy, jz;
  if (d == 0) { jx = s ? bp.ex - 1 : 0; jy = pos % BY; jz = pos / BY; }
  else if (d == 1) { jy = s ? bp.ey - 1 : 0; jx = pos % BX; jz = pos / BX; }
  else { jz = s ? bp.ez - 1 : 0; jx = pos % BX; jy = pos / BX; }
  if (jx >= bp.ex || jy >= bp.ey || jz >= bp.ez) return nullptr;
  const int ix = bp.x0 + jx, iy = bp.y0 + jy, iz = bp.z0 + jz;
  const int n = d == 0 ? g.nx : (d == 1 ? g.ny : g.nz);
  int nc = (d == 0 ? ix : (d == 1 ? iy : iz)) + (s ? 1 : -1);
  if (nc < 0 || nc >= n) {
    const int m = g.mode[2 * d + s];
    if (m == kGhost) return (s ? g.ghost[1] : g.ghost[0]) + (size_t)(iy + g.ny * iz) * NP;
    if (m != kWrap) return nullptr;
    nc = s ? 0 : n - 1;
  }
  const int lo = d == 0 ? bp.x0 : (d == 1 ? bp.y0 : bp.z0);
  const int ext = d == 0 ? bp.ex : (d == 1 ? bp.ey : bp.ez);
  if (nc >= lo && nc < lo + ext) return nullptr;  // in the brick
  const int cx = d == 0 ? nc : ix, cy = d == 1 ? nc : iy, cz = d == 2 ? nc : iz;
  return u + ((size_t)cx + (size_t)g.nx * (cy + (size_t)g.ny * cz)) * NP;
}

template <int N, int BX, int BY, int BZ>
__global__ void __launch_bounds__(LapCfg<3, N, BX, BY, BZ>::THREADS, 2)
laplace_persist_kernel(const double *__restrict__ u, double *__restrict__ out, const Geo g,
                       const LapTab<N> T, const double tau_scale, const int nbx, const int nby,
                       const int nbricks) {
  using L = LapCfg<3, N, BX, BY, BZ>;
  using C = PersistCfg<N, BX, BY, BZ>;
  constexpr int RP = L::RP, LPC = L::LPC, CS = L::CS, NP = L::NP, NSIDE = 6;
  constexpr int H = N / 2, NE = (N + 1) / 2, HO = H > 0 ? H : 1;
  static_assert(RP == N, "persistent kernel: odd N (unpadded TMA rows)");
  extern __shared__ double smem[];
  double *buf1 = smem + C::OFF_BUF1;
  double *fbuf = smem + C::OFF_FBUF;
  double *hraw = smem + C::OFF_HRAW;
  double *hbuf = smem + C::OFF_HBUF;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
  int *soff_all = reinterpret_cast<int *>(smem + C::NDBL);
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  if ((int)blockIdx.x >= nbricks) return;
  const bool tma_ok = !(g.nx & 1) && ((reinterpret_cast<uintptr_t>(u) & 15) == 0);

  // TMA (or cooperative fallback) copy of brick b into raw buffer `rb`
  auto load_brick = [&](int b, double *rb, uint64_t *bar, bool coop) {
    const BrickPos bp = brick_pos(g, b, nbx, nby, BX, BY, BZ);
    constexpr int ROW = BX * NP;
    if (tma_ok && !(bp.ex & 1)) {
      if (tid == 0) {
        // order earlier generic-proxy accesses of this buffer before the
        // async-proxy (TMA) writes into it
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        int rows = 0;
        for (int r = 0; r < BY * BZ; ++r)
          if (r % BY < bp.ey && r / BY < bp.ez) ++rows;
        mbar_expect_tx(bar, (uint32_t)(rows * bp.ex * NP * sizeof(double)));
        for (int r = 0; r < BY * BZ; ++r) {
          const int jy = r % BY, jz = r / BY;
          if (jy >= bp.ey || jz >= bp.ez) continue;
          const size_t e0 = (size_t)bp.x0 + (size_t)g.nx * ((bp.y0 + jy) + (size_t)g.ny * (bp.z0 + jz));
          bulk_g2s(rb + r * ROW, u + e0 * NP, (uint32_t)(bp.ex * NP * sizeof(double)), bar);
        }
      }
      return true;
    }
    if (coop) {
      for (int i = tid; i < L::NC * NP; i += blockDim.x) {
        const int r = i / ROW, w = i - r * ROW;
        const int jx = w / NP, jy = r % BY, jz = r / BY;
        double v = 0.0;
        if (jx < bp.ex && jy < bp.ey && jz < bp.ez)
          v = u[((size_t)bp.x0 + (size_t)g.nx * ((bp.y0 + jy) + (size_t)g.ny * (bp.z0 + jz))) * NP + w];
        rb[i] = v;
      }
    }
    return false;
  };

  // face-coefficient table of brick b into slot ts (threads < NC*6 and < NC)
  auto build_table = [&](int b, int ts) {
    const BrickPos bp = brick_pos(g, b, nbx, nby, BX, BY, BZ);
    double *tab = smem + C::OFF_TAB + ts * C::TAB;
    double *sside = tab;
    double *scell = tab + C::SIDEC * C::NC * NSIDE;
    int *soff = soff_all + ts * C::NC * NSIDE;
    for (int it = tid; it < C::NC * NSIDE; it += blockDim.x) {
      const int c = it / NSIDE, side = it % NSIDE;
      const int d = side >> 1, s = side & 1;
      const int jx = c % BX, jy = (c / BX) % BY, jz = c / (BX * BY);
      double a_vo = 0.0, a_go = 0.0, a_vn = 0.0, a_gn = 0.0, b_vo = 0.0, b_vn = 0.0;
      int off = C::OFF_FBUF + (c * 4 + (s ? 2 : 0)) * LPC;
      if (jx < bp.ex && jy < bp.ey && jz < bp.ez) {
        const int ix = bp.x0 + jx, iy = bp.y0 + jy, iz = bp.z0 + jz;
        NbrInfo nb;
#define DG_RES(DD, SS)                                                                           \
  resolve_nbr<DD, SS, 3, N, BX, BY, BZ>(g, u, ix, iy, iz, bp.x0, bp.y0, bp.z0, bp.ex, bp.ey, \
                                        bp.ez)
        switch (side) {
          case 0: nb = DG_RES(0, 0); break;
          case 1: nb = DG_RES(0, 1); break;
          case 2: nb = DG_RES(1, 0); break;
          case 3: nb = DG_RES(1, 1); break;
          case 4: nb = DG_RES(2, 0); break;
          default: nb = DG_RES(2, 1); break;
        }
#undef DG_RES
        const double taue = g.tau[(size_t)ix + (size_t)g.nx * (iy + (size_t)g.ny * iz)];
        const double h0 = g.hx[ix], h1 = g.hy[iy], h2 = g.hz[iz];
        const double hd = d == 0 ? h0 : (d == 1 ? h1 : h2);
        const double sfac = d == 0 ? 0.25 * h1 * h2 : (d == 1 ? 0.25 * h0 * h2 : 0.25 * h0 * h1);
        const double hi = 1.0 / hd;
        const double sg = s ? -1.0 : 1.0;
        if (nb.kind <= 1) {
          const double hni = 1.0 / nb.h;
          const double tau = tau_scale * fmax(taue, nb.tau);
          a_vo = tau; a_go = sg * hi; a_vn = -tau; a_gn = sg * hni;
          b_vo = sg * hi; b_vn = -sg * hi;
          if (nb.kind == 0) {
            off = C::OFF_FBUF + (nb.cb * 4 + (s ? 0 : 2)) * LPC;
          } else {
            const int pos = d == 0 ? jy + BY * jz : (d == 1 ? jx + BX * jz : jx + BX * jy);
            const int slot = slot_of<L>(d, s, pos);
            off = (d == 0 ? C::OFF_HRAW : C::OFF_HBUF) + slot * 2 * LPC;
          }
        } else if (nb.kind == kBndNeumann) {
          const double tau = tau_scale * taue;
          a_vo = 2.0 * tau; a_go = 2.0 * sg * hi;
          b_vo = 2.0 * sg * hi;
        }
        a_vo *= sfac; a_go *= sfac; a_vn *= sfac; a_gn *= sfac; b_vo *= sfac; b_vn *= sfac;
      }
      double *sc = sside + C::SIDEC * it;
      sc[0] = a_vo; sc[1] = a_go; sc[2] = a_vn; sc[3] = a_gn; sc[4] = b_vo; sc[5] = b_vn;
      soff[it] = off;
    }
    for (int cc = tid; cc < C::NC; cc += blockDim.x) {
      const int jx = cc % BX, jy = (cc / BX) % BY, jz = cc / (BX * BY);
      double h0 = 1.0, h1 = 1.0, h2 = 1.0;
      if (jx < bp.ex && jy < bp.ey && jz < bp.ez) {
        h0 = g.hx[bp.x0 + jx];
        h1 = g.hy[bp.y0 + jy];
        h2 = g.hz[bp.z0 + jz];
      }
      double *ct = scell + 4 * cc;
      ct[0] = 0.5 * h1 * h2 / h0;
      ct[1] = 0.5 * h0 * h2 / h1;
      ct[2] = 0.5 * h0 * h1 / h2;
    }
  };

  // raw face functionals of the halo cells of brick b -> hraw
  auto halo = [&](int b) {
    const BrickPos bp = brick_pos(g, b, nbx, nby, BX, BY, BZ);
    constexpr int NIT = L::NSLOT * LPC;
    constexpr int THR = L::THREADS;
    constexpr int ROUNDS = (NIT + THR - 1) / THR;
    double x[ROUNDS][N];
    int item[ROUNDS], sd[ROUNDS];
#pragma unroll
    for (int k = 0; k < ROUNDS; ++k) {
      const int i = tid + k * THR;
      item[k] = -1;
      sd[k] = 0;
      if (i < NIT) {
        const int slot = i / LPC, p = i - slot * LPC;
        int d, s, pos;
        if (slot < L::SLOT1) { d = 0; s = slot >= L::NS0; pos = slot - s * L::NS0; }
        else if (slot < L::SLOT2) { d = 1; s = slot >= L::SLOT1 + L::NS1; pos = slot - L::SLOT1 - s * L::NS1; }
        else { d = 2; s = slot >= L::SLOT2 + L::NS2; pos = slot - L::SLOT2 - s * L::NS2; }
        const double *src = halo_src3<N, BX, BY, BZ>(g, u, d, s, pos, bp);
        if (src != nullptr) {
          const int a = p / N, bb = p - a * N;
          int base, stride;
          if (d == 0) { base = (a * N + bb) * N; stride = 1; }
          else if (d == 1) { base = a * N * N + bb; stride = N; }
          else { base = a * N + bb; stride = N * N; }
#pragma unroll
          for (int q = 0; q < N; ++q) x[k][q] = __ldg(src + base + q * stride);
          item[k] = i;
          sd[k] = s;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < ROUNDS; ++k) {
      if (item[k] < 0) continue;
      const int slot = item[k] / LPC, p = item[k] - slot * LPC;
      double v, gsum = 0.0;
      if (sd[k]) {
        v = x[k][0];
#pragma unroll
        for (int q = 0; q < N; ++q) gsum += T.dL[q] * x[k][q];
      } else {
        v = x[k][N - 1];
#pragma unroll
        for (int q = 0; q < N; ++q) gsum += T.dR[q] * x[k][q];
      }
      hraw[(slot * 2 + 0) * LPC + p] = v;
      hraw[(slot * 2 + 1) * LPC + p] = gsum;
    }
  };

  // ---- prologue: first brick -------------------------------------------------
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  __syncthreads();
  const int b_first = blockIdx.x;
  bool tma_cur = load_brick(b_first, smem + C::OFF_RAW0, &bars[0], true);
  build_table(b_first, 0);
  uint32_t parity[2] = {0u, 0u};  // mbarrier phase per raw buffer

  for (int it = 0;; ++it) {
    const int b = b_first + it * G;
    if (b >= nbricks) break;
    const int rb = it & 1;
    double *buf0 = smem + (rb ? C::OFF_RAW1 : C::OFF_RAW0);
    const double *tab = smem + C::OFF_TAB + rb * C::TAB;
    const double *sside = tab;
    const double *scell = tab + C::SIDEC * C::NC * NSIDE;
    const int *soff = soff_all + rb * C::NC * NSIDE;
    const BrickPos bp = brick_pos(g, b, nbx, nby, BX, BY, BZ);
    const int bn = b + G;
    halo(b);
    __syncthreads();  // #1: tables of b, halo raw, (fallback) raw loads visible
    if (tma_cur) {
      mbar_wait(&bars[rb], parity[rb]);
      parity[rb] ^= 1u;
    }
    // prefetch brick b+G into the other raw buffer (freed at the end of b-G)
    bool tma_next = false;
    if (bn < nbricks) tma_next = load_brick(bn, smem + (rb ? C::OFF_RAW0 : C::OFF_RAW1), &bars[rb ^ 1], false);

    // ---- per-thread line coordinates ----------------------------------------
    const int l = tid;
    const bool has_line = l < L::NL;
    const int c = has_line ? l / LPC : 0;
    const int t = l - c * LPC;
    const int jx = c % BX, jy = (c / BX) % BY, jz = c / (BX * BY);
    const bool active = has_line && jx < bp.ex && jy < bp.ey && jz < bp.ez;
    const size_t e = (size_t)(bp.x0 + jx) + (size_t)g.nx * ((bp.y0 + jy) + (size_t)g.ny * (bp.z0 + jz));
    const int ta = t / N, tb = t - ta * N;
    double v[N], ev[NE], ov[HO], E[NE], O[HO];
    double v0 = 0.0, v1 = 0.0, g0 = 0.0, g1 = 0.0;
    auto functionals = [&]() {
      double ge = 0.0, go = 0.0;
#pragma unroll
      for (int j = 0; j < NE; ++j) ge += T.dLe[j] * ev[j];
#pragma unroll
      for (int j = 0; j < H; ++j) go += T.dLo[j] * ov[j];
      v0 = v[0];
      v1 = v[N - 1];
      g0 = ge + go;
      g1 = go - ge;
      fbuf[(c * 4 + 0) * LPC + t] = v0;
      fbuf[(c * 4 + 1) * LPC + t] = g0;
      fbuf[(c * 4 + 2) * LPC + t] = v1;
      fbuf[(c * 4 + 3) * LPC + t] = g1;
    };
    auto add_lifts = [&](auto dconst) {
      constexpr int d = decltype(dconst)::value;
      const int s0 = c * NSIDE + 2 * d, s1 = s0 + 1;
      const double *c0 = sside + C::SIDEC * s0, *c1 = sside + C::SIDEC * s1;
      const double vn0 = smem[soff[s0] + t], gn0 = smem[soff[s0] + LPC + t];
      const double vn1 = smem[soff[s1] + t], gn1 = smem[soff[s1] + LPC + t];
      const double cv0 = c0[0] * v0 + c0[1] * g0 + c0[2] * vn0 + c0[3] * gn0;
      const double cd0 = c0[4] * v0 + c0[5] * vn0;
      const double cv1 = c1[0] * v1 + c1[1] * g1 + c1[2] * vn1 + c1[3] * gn1;
      const double cd1 = c1[4] * v1 + c1[5] * vn1;
      E[0] += 0.5 * (cv0 + cv1);
      O[0] += 0.5 * (cv0 - cv1);
      const double dm = cd0 - cd1, dp = cd0 + cd1;
#pragma unroll
      for (int i = 0; i < NE; ++i) E[i] += T.dLe[i] * dm;
#pragma unroll
      for (int i = 0; i < H; ++i) O[i] += T.dLo[i] * dp;
    };

    // ---- phase X ----------------------------------------------------------------
    const int xbase = c * CS + (ta * N + tb) * RP;
    if (has_line) {
#pragma unroll
      for (int q = 0; q < N; ++q) v[q] = buf0[xbase + q];
      eo_split<N>(v, ev, ov);
      functionals();
    }
    __syncthreads();  // #2
    {  // halo step A: y, z sides M_x on raw rows
      constexpr int ROWS = LPC / N;
      for (int i = tid; i < (L::NSLOT - L::SLOT1) * 2 * ROWS; i += blockDim.x) {
        const int sw = i / ROWS, a = i - sw * ROWS;
        const int off = (L::SLOT1 * 2 + sw) * LPC + a * N;
        double x[N];
#pragma unroll
        for (int q = 0; q < N; ++q) x[q] = hraw[off + q];
#pragma unroll
        for (int i2 = 0; i2 < N; ++i2) {
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < N; ++q) acc += T.M[i2 * N + q] * x[q];
          hbuf[off + i2] = acc;
        }
      }
    }
    if (active) {
      double y[N];
      eo_apply<N, false>(T.Me, T.Mo, ev, ov, 1.0, E, O);
      eo_merge<N>(E, O, y);
#pragma unroll
      for (int i = 0; i < N; ++i) buf0[xbase + i] = y[i];
      eo_apply<N, false>(T.Ke, T.Ko, ev, ov, scell[4 * c + 0], E, O);
      add_lifts(std::integral_constant<int, 0>());
      eo_merge<N>(E, O, y);
#pragma unroll
      for (int i = 0; i < N; ++i) buf1[xbase + i] = y[i];
    }
    __syncthreads();  // #3
    {  // halo step B: z sides M_y in place (columns)
      for (int i = tid; i < 2 * L::NS2 * 2 * N; i += blockDim.x) {
        const int sw = i / N, xcol = i - sw * N;
        double *col = hbuf + (L::SLOT2 * 2 + sw) * LPC + xcol;
        double x[N];
#pragma unroll
        for (int q = 0; q < N; ++q) x[q] = col[q * N];
#pragma unroll
        for (int i2 = 0; i2 < N; ++i2) {
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < N; ++q) acc += T.M[i2 * N + q] * x[q];
          col[i2 * N] = acc;
        }
      }
    }
    // ---- phase Y ----------------------------------------------------------------
    const int ybase = c * CS + ta * N * RP + tb;
    if (has_line) {
#pragma unroll
      for (int q = 0; q < N; ++q) v[q] = buf0[ybase + q * RP];
      eo_split<N>(v, ev, ov);
      functionals();
    }
    __syncthreads();  // #4
    if (active) {
      double y[N], te[NE], to[HO];
#pragma unroll
      for (int q = 0; q < N; ++q) y[q] = buf1[ybase + q * RP];
      eo_split<N>(y, te, to);
      eo_apply<N, false>(T.Me, T.Mo, ev, ov, 1.0, E, O);
      eo_merge<N>(E, O, y);
#pragma unroll
      for (int i = 0; i < N; ++i) buf0[ybase + i * RP] = y[i];
      eo_apply<N, false>(T.Me, T.Mo, te, to, 1.0, E, O);
      eo_apply<N, true>(T.Ke, T.Ko, ev, ov, scell[4 * c + 1], E, O);
      add_lifts(std::integral_constant<int, 1>());
      eo_merge<N>(E, O, y);
#pragma unroll
      for (int i = 0; i < N; ++i) buf1[ybase + i * RP] = y[i];
    }
    // table of the next brick (its loads overlap the rest of this brick)
    if (bn < nbricks) build_table(bn, rb ^ 1);
    __syncthreads();  // #5
    // ---- phase Z ----------------------------------------------------------------
    const int zbase = c * CS + ta * RP + tb;
    if (has_line) {
#pragma unroll
      for (int q = 0; q < N; ++q) v[q] = buf0[zbase + q * N * RP];
      eo_split<N>(v, ev, ov);
      functionals();
    }
    __syncthreads();  // #6
    if (active) {
      double y[N], ge[NE], go[HO];
#pragma unroll
      for (int q = 0; q < N; ++q) y[q] = buf1[zbase + q * N * RP];
      eo_split<N>(y, ge, go);
      eo_apply<N, false>(T.Me, T.Mo, ge, go, 1.0, E, O);
      eo_apply<N, true>(T.Ke, T.Ko, ev, ov, scell[4 * c + 2], E, O);
      add_lifts(std::integral_constant<int, 2>());
      eo_merge<N>(E, O, y);
#pragma unroll
      for (int i = 0; i < N; ++i) out[e * NP + (i * N + ta) * N + tb] = y[i];
    }
    tma_cur = tma_next;
    if (!tma_next && bn < nbricks) {
      __syncthreads();  // fallback path: cooperative load of the next brick
      load_brick(bn, smem + (rb ? C::OFF_RAW0 : C::OFF_RAW1), &bars[rb ^ 1], true);
    }
    __syncthreads();  // #7: fbuf / hraw / buf1 free for the next brick
  }
}

}  // namespace dg
