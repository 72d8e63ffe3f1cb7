// Fused cell+face SIPG Laplace vmult for Cartesian cells, fp64, sm_100a.
//
// Replaces apply_pressure_laplace (reference operators.py:187-238).  On an
// axis-aligned cell the reference's quadrature-point evaluation collapses to
// a separable form (exact up to rounding: the Gauss rule n_q = k+1
// integrates every product exactly):
//
//   out = M_z [ M_y ( s_x Kh_x u + s_x Lx ) + s_y Kh_y P + s_y Ly ]
//         + s_z Kh_z Q + s_z Lz,        P = M_x u,  Q = M_y P
//
// with M = S^T W S, Kh_d = (2/h_d) D^T W D (1D reference matrices),
// s_d = prod_{d' != d} h_d'/2, and L_d the face lifts of the SIP fluxes
// (operators.py:209-237) evaluated from the value/normal-derivative face
// functionals of u (x), P (y) and Q (z): linear functionals commute with the
// tangential masses, so face terms need no extra sweeps.  7 one-dimensional
// sweeps per cell in 3D (4 in 2D) plus rank-2 face lifts.
//
// CTA = brick of BX*BY*BZ cells in shared memory; one thread per line per
// phase (x-, y-, z-lines).  Neighbour functionals come from the brick or,
// across the brick surface, from halo cells read once from L2 with their
// tangential masses applied.  Per-cell side data (neighbour kind/index,
// 1/h of the neighbour, face penalty) is resolved once per CTA into a small
// shared table, so the face arithmetic is divide-free.
// No atomics: every output DoF is written once by its own cell
// (the reference's gather-then-scatter determinism, spaces.py:151-158).
#pragma once
#include <type_traits>

#include "common.cuh"

namespace dg {

template <int N>
__host__ __device__ constexpr int row_pitch() {
  return (N % 2 == 0) ? N + 1 : N;  // odd shared-memory row pitch
}

struct NbrInfo {
  int kind;           // 0 in-brick, 1 halo, 2 boundary none, 3 boundary neumann
  int cb;             // in-brick cell index
  double h;           // neighbour size in the face-normal direction
  double tau;         // neighbour tau_e
  const double *src;  // halo: neighbour cell data (global)
};

// Resolve the neighbour of owned cell (ix,iy,iz) across side (D, S).
template <int D, int S, int DIM, int N, int BX, int BY, int BZ>
__device__ __forceinline__ NbrInfo resolve_nbr(const Geo &g, const double *u, int ix, int iy,
                                               int iz, int x0, int y0, int z0, int ex, int ey,
                                               int ez) {
  constexpr int NP = (DIM == 3) ? N * N * N : N * N;
  NbrInfo r;
  r.cb = 0;
  r.src = nullptr;
  r.h = 1.0;
  r.tau = 0.0;
  const int nd = D == 0 ? g.nx : D == 1 ? g.ny : g.nz;
  const int cd = D == 0 ? ix : D == 1 ? iy : iz;
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

template <int DIM, int N, int BX, int BY, int BZ>
struct LapCfg {
  static constexpr int RP = row_pitch<N>();
  static constexpr int NC = BX * BY * BZ;
  static constexpr int NP = (DIM == 3) ? N * N * N : N * N;
  static constexpr int LPC = (DIM == 3) ? N * N : N;           // lines per cell
  static constexpr int CS = (DIM == 3) ? N * N * RP : N * RP;  // smem cell stride
  static constexpr int NL = NC * LPC;
  static constexpr int THREADS = ((NL + 31) / 32) * 32;
  static constexpr int NSIDE = 2 * DIM;
  static constexpr int NS0 = BY * BZ, NS1 = BX * BZ, NS2 = (DIM == 3) ? BX * BY : 0;
  static constexpr int SLOT0 = 0, SLOT1 = 2 * NS0, SLOT2 = 2 * NS0 + 2 * NS1;
  static constexpr int NSLOT = 2 * (NS0 + NS1 + NS2);
  static constexpr int HSIZE = NSLOT * 2 * LPC;  // [slot][v|g][LPC]
  static constexpr int BUF = NC * CS;
  static constexpr int FBUF = NC * 4 * LPC;      // [cell][v0,g0,v1,g1][LPC]
  static constexpr int CELLT = 8;                // per cell: 1/h_d, s_d
  // shared memory carve-up (doubles, then pointers, then ints)
  static constexpr int OFF_BUF1 = BUF;
  static constexpr int OFF_FBUF = 2 * BUF;
  static constexpr int OFF_HRAW = OFF_FBUF + FBUF;
  static constexpr int OFF_HBUF = OFF_HRAW + HSIZE;
  static constexpr int OFF_SIDE = OFF_HBUF + HSIZE;          // [cell][side] (1/hn, tau)
  static constexpr int OFF_CELL = OFF_SIDE + 2 * NC * NSIDE;
  static constexpr int OFF_PTR = OFF_CELL + CELLT * NC;       // halo sources
  static constexpr int OFF_BAR = OFF_PTR + NSLOT;             // mbarrier (TMA)
  static constexpr int NDBL = OFF_BAR + 1;
  static constexpr size_t SMEM = sizeof(double) * (size_t)NDBL + sizeof(int) * NC * NSIDE;
};

// ---- TMA bulk copy (cp.async.bulk) + mbarrier helpers -----------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, int phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// slot index of side (d, s) at tangential brick position pos
template <class C>
__device__ __forceinline__ int slot_of(int d, int s, int pos) {
  return d == 0 ? C::SLOT0 + s * C::NS0 + pos
                : (d == 1 ? C::SLOT1 + s * C::NS1 + pos : C::SLOT2 + s * C::NS2 + pos);
}

// SIP face coefficients (value row cv, derivative row cd) for one line end.
// vo/go own value / reference derivative at the face, vn/gn neighbour's,
// hi = 1/h own, hni = 1/h neighbour, tau = scaled face penalty.
__device__ __forceinline__ void sip_coeffs(int kind, int s, double vo, double go, double vn,
                                           double gn, double hi, double hni, double tau,
                                           double &cv, double &cd) {
  if (kind <= 1) {  // interior face (operators.py:217-225)
    if (s) {          // own cell is the minus side
      const double jump = vo - vn;
      const double avg = go * hi + gn * hni;
      cv = tau * jump - avg;
      cd = -jump * hi;
    } else {          // own cell is the plus side
      const double jump = vn - vo;
      const double avg = gn * hni + go * hi;
      cv = avg - tau * jump;
      cd = -jump * hi;
    }
  } else if (kind == kBndNeumann) {  // pressure-Dirichlet face (operators.py:227-233)
    if (s) {
      cv = 2.0 * (tau * vo - hi * go);
      cd = -2.0 * vo * hi;
    } else {
      cv = 2.0 * (hi * go + tau * vo);
      cd = 2.0 * vo * hi;
    }
  } else {
    cv = 0.0;
    cd = 0.0;
  }
}

// part: 0 all cells, 1 skip bricks touching a ghost side, 2 only those
template <int DIM, int N, int BX, int BY, int BZ>
__global__ void __launch_bounds__(LapCfg<DIM, N, BX, BY, BZ>::THREADS, (N >= 7 ? 1 : 2))
laplace_vmult_kernel(const double *__restrict__ u, double *__restrict__ out, const Geo g,
                     const LapTab<N> T, const double tau_scale, const int part) {
  using C = LapCfg<DIM, N, BX, BY, BZ>;
  constexpr int RP = C::RP, LPC = C::LPC, CS = C::CS, NP = C::NP, NSIDE = C::NSIDE;
  extern __shared__ double smem[];
  double *buf0 = smem;
  double *buf1 = smem + C::OFF_BUF1;
  double *fbuf = smem + C::OFF_FBUF;
  double *hraw = smem + C::OFF_HRAW;
  double *hbuf = smem + C::OFF_HBUF;
  double *sside = smem + C::OFF_SIDE;
  double *scell = smem + C::OFF_CELL;
  const double **hsrc = reinterpret_cast<const double **>(smem + C::OFF_PTR);
  int *skind = reinterpret_cast<int *>(smem + C::NDBL);

  const int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  const int x0 = bx * BX, y0 = by * BY, z0 = bz * BZ;
  const int ex = min(BX, g.nx - x0), ey = min(BY, g.ny - y0);
  const int ez = (DIM == 3) ? min(BZ, g.nz - z0) : 1;
  if (part != 0) {
    const bool touches = (g.mode[0] == kGhost && x0 == 0) || (g.mode[1] == kGhost && x0 + ex == g.nx);
    if ((part == 1 && touches) || (part == 2 && !touches)) return;
  }
  const int tid = threadIdx.x;

  // ---- setup: per (cell, side) neighbour table; per cell geometry ---------
  for (int it = tid; it < C::NC * NSIDE; it += blockDim.x) {
    const int c = it / NSIDE, side = it % NSIDE;
    const int jx = c % BX, jy = (c / BX) % BY, jz = c / (BX * BY);
    int kind = 2, idx = 0;
    double hni = 0.0, tau = 0.0;
    const double *hsrc_cell = nullptr;
    if (jx < ex && jy < ey && jz < ez) {
      const int ix = x0 + jx, iy = y0 + jy, iz = z0 + jz;
      NbrInfo nb;
#define DG_RES(DD, SS) \
  resolve_nbr<DD, SS, DIM, N, BX, BY, BZ>(g, u, ix, iy, iz, x0, y0, z0, ex, ey, ez)
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
      kind = nb.kind;
      if (kind == 0) idx = nb.cb;
      if (kind == 1) {
        const int d = side >> 1, s = side & 1;
        const int pos = d == 0 ? jy + BY * jz : (d == 1 ? jx + BX * jz : jx + BX * jy);
        idx = slot_of<C>(d, s, pos);
        hsrc_cell = nb.src;
      }
      if (kind <= 1) {
        hni = 1.0 / nb.h;
        tau = tau_scale * fmax(taue, nb.tau);
      } else {
        tau = tau_scale * taue;
      }
    }
    skind[it] = kind | (idx << 4);
    sside[2 * it] = hni;
    sside[2 * it + 1] = tau;
    {  // every halo slot is written exactly once, by its brick-edge cell
      const int d = side >> 1, s = side & 1;
      const bool edge = d == 0 ? jx == (s ? ex - 1 : 0)
                               : (d == 1 ? jy == (s ? ey - 1 : 0) : jz == (s ? ez - 1 : 0));
      if (edge) {
        const int pos = d == 0 ? jy + BY * jz : (d == 1 ? jx + BX * jz : jx + BX * jy);
        hsrc[slot_of<C>(d, s, pos)] = hsrc_cell;
      }
    }
  }
  for (int cc = tid; cc < C::NC; cc += blockDim.x) {
    const int jx = cc % BX, jy = (cc / BX) % BY, jz = cc / (BX * BY);
    double h0 = 1.0, h1 = 1.0, h2 = 2.0;
    if (jx < ex && jy < ey && jz < ez) {
      h0 = g.hx[x0 + jx];
      h1 = g.hy[y0 + jy];
      if (DIM == 3) h2 = g.hz[z0 + jz];
    }
    double *ct = scell + C::CELLT * cc;
    ct[0] = 1.0 / h0;
    ct[1] = 1.0 / h1;
    ct[2] = 1.0 / h2;
    ct[3] = 0.5 * h1 * (DIM == 3 ? 0.5 * h2 : 1.0);
    ct[4] = 0.5 * h0 * (DIM == 3 ? 0.5 * h2 : 1.0);
    ct[5] = 0.25 * h0 * h1;
  }
  // ---- own cells -> buf0: rows of x-adjacent cells are contiguous in both
  // global and (odd N, unpadded) shared memory -> one TMA bulk copy per row
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
  constexpr int ROW = BX * NP;
  const bool tma = (RP == N) && !(ex & 1) && !(g.nx & 1) &&
                   ((reinterpret_cast<uintptr_t>(u) & 15) == 0);
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
        bulk_g2s(buf0 + r * ROW, u + e0 * NP, (uint32_t)(ex * NP * sizeof(double)), bar);
      }
    }
  } else {
    for (int i = tid; i < C::NC * NP; i += blockDim.x) {
      const int r = i / ROW, w = i - r * ROW;
      const int jx = w / NP, o = w - jx * NP;
      const int jy = r % BY, jz = r / BY;
      double v = 0.0;
      if (jx < ex && jy < ey && jz < ez)
        v = u[((size_t)x0 + (size_t)g.nx * ((y0 + jy) + (size_t)g.ny * (z0 + jz))) * NP + w];
      int so;
      if (RP == N) {
        so = o;
      } else {
        const int x = o % N, yz = o / N;
        so = yz * RP + x;
      }
      buf0[(r * BX + jx) * CS + so] = v;
    }
  }
  __syncthreads();  // #1

  // ---- halo: raw face functionals of neighbour cells outside the brick ----
  // flat (slot, face point) items spread over all threads; every thread
  // issues all of its L2 loads before consuming any (memory-level parallelism)
  {
    constexpr int NIT = C::NSLOT * LPC;
    constexpr int ROUNDS = (NIT + C::THREADS - 1) / C::THREADS;
    double x[ROUNDS][N];
    int item[ROUNDS], sd[ROUNDS];
#pragma unroll
    for (int k = 0; k < ROUNDS; ++k) {
      const int i = tid + k * C::THREADS;
      item[k] = -1;
      sd[k] = 0;
      if (i < NIT) {
        const int slot = i / LPC, p = i - slot * LPC;
        const double *src = hsrc[slot];
        if (src != nullptr) {
          int d, s;
          if (slot < C::SLOT1) { d = 0; s = slot >= C::NS0; }
          else if (slot < C::SLOT2) { d = 1; s = slot >= C::SLOT1 + C::NS1; }
          else { d = 2; s = slot >= C::SLOT2 + C::NS2; }
          const int a = (DIM == 3) ? p / N : 0, b = (DIM == 3) ? p - a * N : p;
          int base, stride;
          if (d == 0) { base = (a * N + b) * N; stride = 1; }     // (z,y) line along x
          else if (d == 1) { base = a * N * N + b; stride = N; }  // (z,x) line along y
          else { base = a * N + b; stride = N * N; }              // (y,x) line along z
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
      if (sd[k]) {  // neighbour on our hi side faces us with its LEFT end
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
  }
  if (tma) mbar_wait(bar, 0);

  // ---- per-thread line coordinates ------------------------------------------
  const int l = tid;
  const bool has_line = l < C::NL;
  const int c = has_line ? l / LPC : 0;
  const int t = l - c * LPC;  // tangential position (slow*N + fast) in each phase
  const int jx = c % BX, jy = (c / BX) % BY, jz = c / (BX * BY);
  const bool active = has_line && jx < ex && jy < ey && jz < ez;
  const size_t e = (size_t)(x0 + jx) + (size_t)g.nx * ((y0 + jy) + (size_t)g.ny * (z0 + jz));
  const int ta = (DIM == 3) ? t / N : 0, tb = (DIM == 3) ? t - ta * N : t;
  double v[N], w[N], g0 = 0.0, g1 = 0.0;

  auto functionals = [&]() {
    g0 = 0.0;
    g1 = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      g0 += T.dL[q] * v[q];
      g1 += T.dR[q] * v[q];
    }
    fbuf[(c * 4 + 0) * LPC + t] = v[0];
    fbuf[(c * 4 + 1) * LPC + t] = g0;
    fbuf[(c * 4 + 2) * LPC + t] = v[N - 1];
    fbuf[(c * 4 + 3) * LPC + t] = g1;
  };
  // w += sfac * (SIP lifts of direction d) for the own line v (functionals
  // g0/g1 from the first pass); halo data of x-sides is raw, y/z mass-applied
  auto add_lifts = [&](auto dconst, double hi, double sfac) {
    constexpr int d = decltype(dconst)::value;
    const double *hb = (d == 0) ? hraw : hbuf;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int st = c * NSIDE + 2 * d + s;
      const int kv = skind[st];
      const int kind = kv & 15, idx = kv >> 4;
      double vn = 0.0, gn = 0.0;
      if (kind == 0) {
        vn = fbuf[(idx * 4 + (s ? 0 : 2)) * LPC + t];
        gn = fbuf[(idx * 4 + (s ? 1 : 3)) * LPC + t];
      } else if (kind == 1) {
        vn = hb[(idx * 2 + 0) * LPC + t];
        gn = hb[(idx * 2 + 1) * LPC + t];
      }
      double cv, cd;
      sip_coeffs(kind, s, s ? v[N - 1] : v[0], s ? g1 : g0, vn, gn, hi, sside[2 * st],
                 sside[2 * st + 1], cv, cd);
      cv *= sfac;
      cd *= sfac;
      w[s ? N - 1 : 0] += cv;
#pragma unroll
      for (int q = 0; q < N; ++q) w[q] += cd * (s ? T.dR[q] : T.dL[q]);
    }
  };

  // ---- phase X: x-lines of u --------------------------------------------------
  const int xbase = c * CS + (ta * N + tb) * RP;  // (z, y) line along x
  if (has_line) {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = buf0[xbase + q];
    functionals();
  }
  __syncthreads();  // #2
  // halo step A: y-sides P = M_x raw (rows along x); z-sides first M_x
  {
    constexpr int ROWS = LPC / N;  // rows per (slot, which)
    for (int i = tid; i < (C::NSLOT - C::SLOT1) * 2 * ROWS; i += blockDim.x) {
      const int sw = i / ROWS, a = i - sw * ROWS;  // sw = (slot - SLOT1)*2 + which
      const int off = (C::SLOT1 * 2 + sw) * LPC + a * N;
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
    const double *ct = scell + C::CELLT * c;
    const double ihx = ct[0], sx = ct[3];
    const double kx = 2.0 * sx * ihx;
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
    add_lifts(std::integral_constant<int, 0>(), ihx, sx);
#pragma unroll
    for (int i = 0; i < N; ++i) buf1[xbase + i] = w[i];
  }
  __syncthreads();  // #3
  // halo step B (3D): z-sides Q = M_y (M_x raw), columns along y, in place
  if (DIM == 3) {
    for (int i = tid; i < 2 * C::NS2 * 2 * N; i += blockDim.x) {
      const int sw = i / N, xcol = i - sw * N;  // sw = (slot - SLOT2)*2 + which
      double *col = hbuf + (C::SLOT2 * 2 + sw) * LPC + xcol;
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
  // ---- phase Y: y-lines of P and T ------------------------------------------
  const int ybase = c * CS + ta * N * RP + tb;  // (z, x) line along y, stride RP
  if (has_line) {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = buf0[ybase + q * RP];
    functionals();
  }
  __syncthreads();  // #4
  if (active) {
    const double *ct = scell + C::CELLT * c;
    const double ihy = ct[1], sy = ct[4];
    const double ky = 2.0 * sy * ihy;
    double tl[N];
#pragma unroll
    for (int q = 0; q < N; ++q) tl[q] = buf1[ybase + q * RP];
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
    add_lifts(std::integral_constant<int, 1>(), ihy, sy);
    if (DIM == 2) {
#pragma unroll
      for (int i = 0; i < N; ++i) out[e * NP + i * N + tb] = w[i];
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double b = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) b += T.M[i * N + q] * v[q];
        buf0[ybase + i * RP] = b;     // Q = M_y P
        buf1[ybase + i * RP] = w[i];  // G
      }
    }
  }
  if (DIM == 2) return;
  __syncthreads();  // #5
  // ---- phase Z: z-lines of Q and G --------------------------------------------
  const int zbase = c * CS + ta * RP + tb;  // (y, x) line along z, stride N*RP
  if (has_line) {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = buf0[zbase + q * N * RP];
    functionals();
  }
  __syncthreads();  // #6
  if (active) {
    const double *ct = scell + C::CELLT * c;
    const double ihz = ct[2], sz = ct[5];
    const double kz = 2.0 * sz * ihz;
    double gl[N];
#pragma unroll
    for (int q = 0; q < N; ++q) gl[q] = buf1[zbase + q * N * RP];
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
    add_lifts(std::integral_constant<int, 2>(), ihz, sz);
#pragma unroll
    for (int i = 0; i < N; ++i) out[e * NP + (i * N + ta) * N + tb] = w[i];
  }
}

}  // namespace dg
