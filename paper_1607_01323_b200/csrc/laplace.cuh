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
// Every 1D sweep runs in even-odd form: M and K are centro-symmetric and the
// endpoint derivative rows anti-symmetric, so each n x n product becomes a
// ceil(n/2)^2 + floor(n/2)^2 product on the even/odd halves of the line --
// fewer fp64 operations and a coefficient set small enough to stay in
// uniform registers.  Face lifts are applied in the same even/odd domain.
//
// CTA = brick of BX*BY*BZ cells in shared memory; one thread per line per
// phase (x-, y-, z-lines).  Neighbour functionals come from the brick or,
// across the brick surface, from halo cells read once from L2 with their
// tangential masses applied.  The face coupling of every (cell, side) is
// reduced once per CTA to six coefficients (own value/derivative,
// neighbour value/derivative) and one shared-memory offset, so the face
// arithmetic is branch- and divide-free.
// No atomics: every output DoF is written once by its own cell
// (the reference's gather-then-scatter determinism, spaces.py:151-158).
#pragma once
#include <type_traits>
#include "tma.cuh"

#include "common.cuh"

namespace dg {

template <int N>
__host__ __device__ constexpr int row_pitch() {
  return (N % 2 == 0) ? N + 1 : N;  // odd shared-memory row pitch
}

template <class R>
struct NbrInfoT {
  int kind;           // 0 in-brick, 1 halo, 2 boundary none, 3 boundary neumann
  int cb;             // in-brick cell index
  R h;                // neighbour size in the face-normal direction
  R hi;               // its inverse
  R tau;              // neighbour tau_e
  const R *src;       // halo: neighbour cell data (global)
};
using NbrInfo = NbrInfoT<double>;

// Resolve the neighbour of owned cell (ix,iy,iz) across side (D, S).
template <int D, int S, int DIM, int N, int BX, int BY, int BZ, class R>
__device__ __forceinline__ NbrInfoT<R> resolve_nbr(const Geo &g, const R *u, int ix, int iy,
                                                   int iz, int x0, int y0, int z0, int ex,
                                                   int ey, int ez) {
  constexpr int NP = (DIM == 3) ? N * N * N : N * N;
  NbrInfoT<R> r;
  r.cb = 0;
  r.src = nullptr;
  r.h = 1.0;
  r.hi = 1.0;
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
      // x-slab ghost layers are fp64 (the fp32 V-cycle runs on whole meshes)
      r.src = reinterpret_cast<const R *>(g.ghost[S]) + (size_t)t * NP;
      r.h = g.ghost_h[S];
      r.hi = g.ghost_hi[S];
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
  r.hi = (D == 0) ? g.hxi[cx] : (D == 1) ? g.hyi[cy] : g.hzi[cz];
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

template <int DIM, int N, int BX, int BY, int BZ, class R = double>
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
  static constexpr int SIDEC = 6;                // face coefficients per (cell, side)
  // shared memory carve-up (R values, then pointers, the mbarrier, ints)
  static constexpr int OFF_BUF1 = BUF;
  static constexpr int OFF_FBUF = 2 * BUF;
  static constexpr int OFF_HRAW = OFF_FBUF + FBUF;
  static constexpr int OFF_HBUF = OFF_HRAW + HSIZE;
  static constexpr int OFF_SIDE = OFF_HBUF + HSIZE;          // [cell][side][6]
  static constexpr int OFF_CELL = OFF_SIDE + SIDEC * NC * NSIDE;  // [cell][4]: s_d scaled K
  static constexpr int NDAT = OFF_CELL + 4 * NC;             // R values
  static constexpr size_t PTR_B = ((sizeof(R) * NDAT + 7) / 8) * 8;  // halo sources (bytes)
  static constexpr size_t BAR_B = PTR_B + 8 * (size_t)NSLOT;         // mbarrier (TMA)
  static constexpr size_t INT_B = BAR_B + 8;                         // side offsets
  static constexpr size_t SMEM = INT_B + sizeof(int) * NC * NSIDE;
};

// slot index of side (d, s) at tangential brick position pos
template <class C>
__device__ __forceinline__ int slot_of(int d, int s, int pos) {
  return d == 0 ? C::SLOT0 + s * C::NS0 + pos
                : (d == 1 ? C::SLOT1 + s * C::NS1 + pos : C::SLOT2 + s * C::NS2 + pos);
}

// Global source of halo slot `slot` (neighbour cell across the brick surface)
// or nullptr when that neighbour is a boundary, lies in the brick (periodic
// wrap onto the brick itself) or the slot is outside a partial brick.  Pure
// index arithmetic, the same resolution as resolve_nbr.
template <class C, int N, int BX, int BY, int BZ, class R = double>
__device__ __forceinline__ const R *halo_slot_src(const Geo &g, const R *u, int slot,
                                                       int x0, int y0, int z0, int ex, int ey,
                                                       int ez, int &d, int &s) {
  constexpr int NP = N * N * N;
  int loc;
  if (slot < C::SLOT1) { d = 0; loc = slot; }
  else if (slot < C::SLOT2) { d = 1; loc = slot - C::SLOT1; }
  else { d = 2; loc = slot - C::SLOT2; }
  const int ns = d == 0 ? C::NS0 : (d == 1 ? C::NS1 : C::NS2);
  s = loc >= ns;
  const int pos = loc - s * ns;
  int ix, iy, iz;
  if (d == 0) { iy = pos % BY; iz = pos / BY; if (iy >= ey || iz >= ez) return nullptr; ix = s ? ex - 1 : 0; }
  else if (d == 1) { ix = pos % BX; iz = pos / BX; if (ix >= ex || iz >= ez) return nullptr; iy = s ? ey - 1 : 0; }
  else { ix = pos % BX; iy = pos / BX; if (ix >= ex || iy >= ey) return nullptr; iz = s ? ez - 1 : 0; }
  ix += x0; iy += y0; iz += z0;
  const int nd = d == 0 ? g.nx : (d == 1 ? g.ny : g.nz);
  const int lo = d == 0 ? x0 : (d == 1 ? y0 : z0);
  const int ext = d == 0 ? ex : (d == 1 ? ey : ez);
  int nc = (d == 0 ? ix : (d == 1 ? iy : iz)) + (s ? 1 : -1);
  if (nc < 0 || nc >= nd) {
    const int m = g.mode[2 * d + s];
    if (m == kGhost) return reinterpret_cast<const R *>(g.ghost[s]) + (size_t)(iy + g.ny * iz) * NP;
    if (m != kWrap) return nullptr;
    nc = s ? 0 : nd - 1;
  }
  if (nc >= lo && nc < lo + ext) return nullptr;
  const int cx = d == 0 ? nc : ix, cy = d == 1 ? nc : iy, cz = d == 2 ? nc : iz;
  return u + ((size_t)cx + (size_t)g.nx * (cy + (size_t)g.ny * cz)) * NP;
}

// ---- even-odd helpers on register arrays ------------------------------------
template <int N, class R>
__device__ __forceinline__ void eo_split(const R *v, R *e, R *o) {
  constexpr int H = N / 2;
#pragma unroll
  for (int j = 0; j < H; ++j) {
    e[j] = v[j] + v[N - 1 - j];
    o[j] = v[j] - v[N - 1 - j];
  }
  if (N & 1) e[H] = v[H];
}
// E = sc * Ae e ; O = sc * Ao o  (accumulate = false) or E += ..., O += ...
template <int N, bool ACC, class R>
__device__ __forceinline__ void eo_apply(const R *Ae, const R *Ao, const R *e, const R *o,
                                         typename Ident<R>::type sc, R *E, R *O) {
  constexpr int H = N / 2, NE = (N + 1) / 2;
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    R a = 0.0;
#pragma unroll
    for (int j = 0; j < NE; ++j) a += Ae[i * NE + j] * e[j];
    E[i] = ACC ? E[i] + sc * a : sc * a;
  }
#pragma unroll
  for (int i = 0; i < H; ++i) {
    R a = 0.0;
#pragma unroll
    for (int j = 0; j < H; ++j) a += Ao[i * H + j] * o[j];
    O[i] = ACC ? O[i] + sc * a : sc * a;
  }
}
template <int N, class R>
__device__ __forceinline__ void eo_merge(const R *E, const R *O, R *y) {
  constexpr int H = N / 2;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    y[i] = E[i] + O[i];
    y[N - 1 - i] = E[i] - O[i];
  }
  if (N & 1) y[H] = E[H];
}

// Epilogues fused into the vmult's output loop (CG / Chebyshev vector phases,
// reference solvers.py:56-71 and :121-128):
//   kEpiStore  out = L u
//   kEpiCheb   rc -= L u ; dnew = a*u + b*(rc/diag) ; x += dnew   (one
//              Chebyshev step; u is the current direction d, out unused)
//   kEpiDot    out = L u and per-CTA partial sums of u.Lu, sum(Lu), u.w
//              (w = integrals of the basis functions, the dual zero-mean
//              weights) for pAp of the projected operator
//   kEpiDotS   (laplace8 only) as kEpiDot, but out leaves by the TMA bulk
//              stores of kEpiStore and the sums are formed in the y phase
//              from a shared-memory copy of the layer's u (no global
//              re-read of u, no extra barrier)
enum LapEpi : int { kEpiStore = 0, kEpiCheb = 1, kEpiDot = 2, kEpiDotS = 3 };
template <class R>
struct EpiArgsT {
  R *rc;
  const R *diag;
  R *x;
  R *dnew;
  double a, b;
  double *partials;      // [brick][4]
  double wint[kMaxN];    // integrals of the 1D basis functions on [-1,1]
};
using EpiArgs = EpiArgsT<double>;

template <int EPI, int DIM, int N, class R>
__device__ __forceinline__ void epi_store(const R *__restrict__ u, R *__restrict__ out,
                                          const EpiArgsT<R> &ea, size_t gi, R y, double wq,
                                          double *acc) {
  if (EPI == kEpiStore) {
    out[gi] = y;
  } else if (EPI == kEpiCheb) {
    if constexpr (std::is_same<R, double>::value) {
      const double r = __dsub_rn(ea.rc[gi], y);
      const double dn = __dadd_rn(__dmul_rn(ea.a, u[gi]), __dmul_rn(ea.b, __ddiv_rn(r, ea.diag[gi])));
      ea.rc[gi] = r;
      ea.dnew[gi] = dn;
      ea.x[gi] = __dadd_rn(ea.x[gi], dn);
    } else {
      const R r = ea.rc[gi] - y;
      const R dn = (R)ea.a * u[gi] + (R)ea.b * (r / ea.diag[gi]);
      ea.rc[gi] = r;
      ea.dnew[gi] = dn;
      ea.x[gi] = ea.x[gi] + dn;
    }
  } else {
    out[gi] = y;
    const double p = u[gi];
    acc[0] += p * y;
    acc[1] += y;
    acc[2] += p * wq;
  }
}

// deterministic CTA reduction of acc[0..2] -> ea.partials[blk*4 + k]
template <class EA>
__device__ __forceinline__ void epi_reduce(double *acc, double *red, const EA &ea, int blk) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc[k] = v;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();  // red may alias data of the last phase
  if (lane == 0)
    for (int k = 0; k < 3; ++k) red[k * 32 + w] = acc[k];
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += red[threadIdx.x * 32 + i];
    ea.partials[(size_t)blk * 4 + threadIdx.x] = s;
  }
}

// part: 0 all cells, 1 skip bricks touching a ghost side, 2 only those
template <int DIM, int N, int BX, int BY, int BZ, int EPI = kEpiStore, class R = double>
__global__ void __launch_bounds__(LapCfg<DIM, N, BX, BY, BZ, R>::THREADS, (N >= 7 ? 1 : 2))
laplace_vmult_kernel(const R *__restrict__ u, R *__restrict__ out, const Geo g,
                     const LapTab<N, R> T, const double tau_scale, const int part,
                     const EpiArgsT<R> ea = EpiArgsT<R>{}) {
  static_assert(EPI != kEpiDot || std::is_same<R, double>::value, "fused dot epilogue: fp64 only");
  using C = LapCfg<DIM, N, BX, BY, BZ, R>;
  constexpr int RP = C::RP, LPC = C::LPC, CS = C::CS, NP = C::NP, NSIDE = C::NSIDE;
  constexpr int H = N / 2, NE = (N + 1) / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R *smem = reinterpret_cast<R *>(smem_raw);
  R *buf0 = smem;
  R *buf1 = smem + C::OFF_BUF1;
  R *fbuf = smem + C::OFF_FBUF;
  R *hraw = smem + C::OFF_HRAW;
  R *hbuf = smem + C::OFF_HBUF;
  R *sside = smem + C::OFF_SIDE;
  R *scell = smem + C::OFF_CELL;
  const R **hsrc = reinterpret_cast<const R **>(smem_raw + C::PTR_B);
  int *soff = reinterpret_cast<int *>(smem_raw + C::INT_B);

  const int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z + g.bz0;
  const int x0 = bx * BX, y0 = by * BY, z0 = bz * BZ;
  const int ex = min(BX, g.nx - x0), ey = min(BY, g.ny - y0);
  const int ez = (DIM == 3) ? min(BZ, g.nz - z0) : 1;
  if (part != 0) {
    const bool touches = (g.mode[0] == kGhost && x0 == 0) || (g.mode[1] == kGhost && x0 + ex == g.nx);
    if ((part == 1 && touches) || (part == 2 && !touches)) return;
  }
  const int tid = threadIdx.x;

  // ---- own cells -> buf0 (issued first: the copy overlaps the setup) ------
  // rows of x-adjacent cells are contiguous in both
  // global and (odd N, unpadded) shared memory -> one TMA bulk copy per row
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + C::BAR_B);
  constexpr int ROW = BX * NP;
  const bool tma = std::is_same<R, double>::value && (RP == N) && !(ex & 1) && !(g.nx & 1) &&
                   ((reinterpret_cast<uintptr_t>(u) & 15) == 0);
  if (tma) {
    if (tid == 0) {
      mbar_init(bar, 1);
      int rows = 0;
      for (int r = 0; r < BY * BZ; ++r)
        if (r % BY < ey && r / BY < ez) ++rows;
      mbar_expect_tx(bar, (uint32_t)(rows * ex * NP * sizeof(R)));
      for (int r = 0; r < BY * BZ; ++r) {
        const int jy = r % BY, jz = r / BY;
        if (jy >= ey || jz >= ez) continue;
        const size_t e0 = (size_t)x0 + (size_t)g.nx * ((y0 + jy) + (size_t)g.ny * (z0 + jz));
        bulk_g2s(buf0 + r * ROW, u + e0 * NP, (uint32_t)(ex * NP * sizeof(R)), bar);
      }
    }
  } else {
    for (int i = tid; i < C::NC * NP; i += blockDim.x) {
      const int r = i / ROW, w = i - r * ROW;
      const int jx = w / NP, o = w - jx * NP;
      const int jy = r % BY, jz = r / BY;
      R v = 0.0;
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
  // ---- setup: per (cell, side) face coefficients + neighbour data offset ---
  for (int it = tid; it < C::NC * NSIDE; it += blockDim.x) {
    const int c = it / NSIDE, side = it % NSIDE;
    const int d = side >> 1, s = side & 1;
    const int jx = c % BX, jy = (c / BX) % BY, jz = c / (BX * BY);
    R a_vo = 0.0, a_go = 0.0, a_vn = 0.0, a_gn = 0.0, b_vo = 0.0, b_vn = 0.0;
    int off = C::OFF_FBUF + (c * 4 + (s ? 2 : 0)) * LPC;  // own data (any valid)
    const R *hsrc_cell = nullptr;
    if (DIM == 3 && g.ctab != nullptr) {
      // coefficients from the context's cell table (laplace6.cuh), neighbour
      // kind by index arithmetic: no dependent loads, no divisions
      if (jx < ex && jy < ey && jz < ez) {
        const size_t e = (size_t)(x0 + jx) + (size_t)g.nx * ((y0 + jy) + (size_t)g.ny * (z0 + jz));
        const double *tr = g.ctab + e * kCellTab + 3 * side;
        const R A = (R)(tau_scale * tr[0]), B = (R)tr[1], Dn = (R)tr[2];
        const int nd = d == 0 ? g.nx : (d == 1 ? g.ny : g.nz);
        const int lo = d == 0 ? x0 : (d == 1 ? y0 : z0);
        const int ext = d == 0 ? ex : (d == 1 ? ey : ez);
        int nc = (d == 0 ? x0 + jx : (d == 1 ? y0 + jy : z0 + jz)) + (s ? 1 : -1);
        int kind = 1;  // 0 in-brick, 1 halo, 2 boundary
        bool ghost = false;
        if (nc < 0 || nc >= nd) {
          const int m = g.mode[2 * d + s];
          if (m == kWrap) nc = s ? 0 : nd - 1;
          else if (m == kGhost) ghost = true;
          else kind = 2;
        }
        a_vo = A; a_go = B; b_vo = B;
        if (kind == 1) {
          a_vn = -A; a_gn = Dn; b_vn = -B;
          if (!ghost && nc >= lo && nc < lo + ext) {
            const int cb = d == 0 ? (nc - x0) + BX * (jy + BY * jz)
                                  : (d == 1 ? jx + BX * ((nc - y0) + BY * jz)
                                            : jx + BX * (jy + BY * (nc - z0)));
            off = C::OFF_FBUF + (cb * 4 + (s ? 0 : 2)) * LPC;
          } else {
            const int pos = d == 0 ? jy + BY * jz : (d == 1 ? jx + BX * jz : jx + BX * jy);
            off = (d == 0 ? C::OFF_HRAW : C::OFF_HBUF) + slot_of<C>(d, s, pos) * 2 * LPC;
          }
        }
      }
      const bool edge = d == 0 ? jx == (s ? ex - 1 : 0)
                               : (d == 1 ? jy == (s ? ey - 1 : 0) : jz == (s ? ez - 1 : 0));
      if (edge) {
        const int pos = d == 0 ? jy + BY * jz : (d == 1 ? jx + BX * jz : jx + BX * jy);
        const int slot = slot_of<C>(d, s, pos);
        int dd, ss;
        hsrc[slot] = halo_slot_src<C, N, BX, BY, BZ, R>(g, u, slot, x0, y0, z0, ex, ey, ez, dd, ss);
      }
      R *sc = sside + C::SIDEC * it;
      sc[0] = a_vo; sc[1] = a_go; sc[2] = a_vn; sc[3] = a_gn; sc[4] = b_vo; sc[5] = b_vn;
      soff[it] = off;
      continue;
    }
    if (jx < ex && jy < ey && jz < ez) {
      const int ix = x0 + jx, iy = y0 + jy, iz = z0 + jz;
      NbrInfoT<R> nb;
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
      const R taue = g.tau[(size_t)ix + (size_t)g.nx * (iy + (size_t)g.ny * iz)];
      const R h0 = g.hx[ix], h1 = g.hy[iy], h2 = (DIM == 3) ? g.hz[iz] : 2.0;
      const R hd = d == 0 ? h0 : (d == 1 ? h1 : h2);
      R sfac;  // s_d = prod of the other half sizes
      if (DIM == 3) sfac = d == 0 ? 0.25 * h1 * h2 : (d == 1 ? 0.25 * h0 * h2 : 0.25 * h0 * h1);
      else sfac = d == 0 ? 0.5 * h1 : 0.5 * h0;
      const R hi = 1.0 / hd;
      const R sg = s ? -1.0 : 1.0;  // sign of the own outward normal flips go terms
      if (nb.kind <= 1) {                // interior face (operators.py:217-225)
        const R hni = 1.0 / nb.h;
        const R tau = tau_scale * fmax(taue, nb.tau);
        a_vo = tau; a_go = sg * hi; a_vn = -tau; a_gn = sg * hni;
        b_vo = sg * hi; b_vn = -sg * hi;
        if (nb.kind == 0) {
          off = C::OFF_FBUF + (nb.cb * 4 + (s ? 0 : 2)) * LPC;
        } else {
          const int pos = d == 0 ? jy + BY * jz : (d == 1 ? jx + BX * jz : jx + BX * jy);
          const int slot = slot_of<C>(d, s, pos);
          off = (d == 0 ? C::OFF_HRAW : C::OFF_HBUF) + slot * 2 * LPC;
          hsrc_cell = nb.src;
        }
      } else if (nb.kind == kBndNeumann) {  // pressure-Dirichlet face (operators.py:227-233)
        const R tau = tau_scale * taue;
        a_vo = 2.0 * tau; a_go = 2.0 * sg * hi;
        b_vo = 2.0 * sg * hi;
      }
      a_vo *= sfac; a_go *= sfac; a_vn *= sfac; a_gn *= sfac; b_vo *= sfac; b_vn *= sfac;
    }
    R *sc = sside + C::SIDEC * it;
    sc[0] = a_vo; sc[1] = a_go; sc[2] = a_vn; sc[3] = a_gn; sc[4] = b_vo; sc[5] = b_vn;
    soff[it] = off;
    {  // every halo slot is written exactly once, by its brick-edge cell
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
    R h0 = 1.0, h1 = 1.0, h2 = 2.0;
    if (jx < ex && jy < ey && jz < ez) {
      h0 = g.hx[x0 + jx];
      h1 = g.hy[y0 + jy];
      if (DIM == 3) h2 = g.hz[z0 + jz];
    }
    R *ct = scell + 4 * cc;  // (2/h_d) s_d: scale of K along d
    if (DIM == 3 && g.ctab != nullptr) {
      if (jx < ex && jy < ey && jz < ez) {
        const double *tr =
            g.ctab + ((size_t)(x0 + jx) + (size_t)g.nx * ((y0 + jy) + (size_t)g.ny * (z0 + jz))) * kCellTab;
        ct[0] = (R)tr[18];
        ct[1] = (R)tr[19];
        ct[2] = (R)tr[20];
      } else {
        ct[0] = ct[1] = ct[2] = 0.0;
      }
    } else if (DIM == 3) {
      ct[0] = 0.5 * h1 * h2 / h0;
      ct[1] = 0.5 * h0 * h2 / h1;
      ct[2] = 0.5 * h0 * h1 / h2;
    } else {
      ct[0] = h1 / h0;
      ct[1] = h0 / h1;
      ct[2] = 0.0;
    }
  }
  __syncthreads();  // #1

  // ---- halo: raw face functionals of neighbour cells outside the brick ----
  // flat (slot, face point) items spread over all threads; every thread
  // issues all of its L2 loads before consuming any (memory-level parallelism)
  if (!(g.exp_flags & 1)) {  // exp_flags bit 0: skip halo (timing experiments only)
    constexpr int NIT = C::NSLOT * LPC;
    constexpr int ROUNDS = (NIT + C::THREADS - 1) / C::THREADS;
    R x[ROUNDS][N];
    int item[ROUNDS], sd[ROUNDS];
#pragma unroll
    for (int k = 0; k < ROUNDS; ++k) {
      const int i = tid + k * C::THREADS;
      item[k] = -1;
      sd[k] = 0;
      if (i < NIT) {
        const int slot = i / LPC, p = i - slot * LPC;
        const R *src = hsrc[slot];
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
          // read from the facing end inwards: one derivative row for both
          // sides (dR_q = -dL_{N-1-q})
          if (!s) { base += (N - 1) * stride; stride = -stride; }
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
      R v, gsum = 0.0;
      v = x[k][0];  // the facing end (hi side: the neighbour's LEFT end)
#pragma unroll
      for (int q = 0; q < N; ++q) gsum += T.dL[q] * x[k][q];
      if (!sd[k]) gsum = -gsum;
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
  R v[N], ev[NE], ov[H > 0 ? H : 1], E[NE], O[H > 0 ? H : 1];
  R v0 = 0.0, v1 = 0.0, g0 = 0.0, g1 = 0.0;
  double eacc[3] = {0.0, 0.0, 0.0};  // kEpiDot partial sums

  // own face functionals of line v (even/odd split ev/ov): values and
  // reference derivatives at both ends -> fbuf
  auto functionals = [&]() {
    R ge = 0.0, go = 0.0;
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
  // E/O += even/odd form of the SIP lifts of direction d (coefficients and
  // neighbour locations from the per-CTA side table)
  auto add_lifts = [&](auto dconst) {
    constexpr int d = decltype(dconst)::value;
    if (g.exp_flags & 2) return;  // timing experiment: no face terms
    const int s0 = c * NSIDE + 2 * d, s1 = s0 + 1;
    const R *c0 = sside + C::SIDEC * s0, *c1 = sside + C::SIDEC * s1;
    const R vn0 = smem[soff[s0] + t], gn0 = smem[soff[s0] + LPC + t];
    const R vn1 = smem[soff[s1] + t], gn1 = smem[soff[s1] + LPC + t];
    const R cv0 = c0[0] * v0 + c0[1] * g0 + c0[2] * vn0 + c0[3] * gn0;
    const R cd0 = c0[4] * v0 + c0[5] * vn0;
    const R cv1 = c1[0] * v1 + c1[1] * g1 + c1[2] * vn1 + c1[3] * gn1;
    const R cd1 = c1[4] * v1 + c1[5] * vn1;
    // value rows e_0 / e_{N-1}; derivative rows dL, dR = -reverse(dL)
    E[0] += 0.5 * (cv0 + cv1);
    if (H > 0) O[0] += 0.5 * (cv0 - cv1);
    const R dm = cd0 - cd1, dp = cd0 + cd1;
#pragma unroll
    for (int i = 0; i < NE; ++i) E[i] += T.dLe[i] * dm;
#pragma unroll
    for (int i = 0; i < H; ++i) O[i] += T.dLo[i] * dp;
  };

  // ---- phase X: x-lines of u --------------------------------------------------
  const int xbase = c * CS + (ta * N + tb) * RP;  // (z, y) line along x
  if (has_line) {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = buf0[xbase + q];
    eo_split<N>(v, ev, ov);
    functionals();
  }
  __syncthreads();  // #2
  // halo step A: y-sides P = M_x raw (rows along x); z-sides first M_x
  if (!(g.exp_flags & 4)) {
    constexpr int ROWS = LPC / N;  // rows per (slot, which)
    for (int i = tid; i < (C::NSLOT - C::SLOT1) * 2 * ROWS; i += blockDim.x) {
      const int sw = i / ROWS, a = i - sw * ROWS;  // sw = (slot - SLOT1)*2 + which
      const int off = (C::SLOT1 * 2 + sw) * LPC + a * N;
      R x[N];
#pragma unroll
      for (int q = 0; q < N; ++q) x[q] = hraw[off + q];
#pragma unroll
      for (int i2 = 0; i2 < N; ++i2) {
        R acc = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) acc += T.M[i2 * N + q] * x[q];
        hbuf[off + i2] = acc;
      }
    }
  }
  if (active) {
    R y[N];
    eo_apply<N, false>(T.Me, T.Mo, ev, ov, 1.0, E, O);
    eo_merge<N>(E, O, y);
#pragma unroll
    for (int i = 0; i < N; ++i) buf0[xbase + i] = y[i];  // P = M_x u (own line only)
    eo_apply<N, false>(T.Ke, T.Ko, ev, ov, scell[4 * c + 0], E, O);
    add_lifts(std::integral_constant<int, 0>());
    eo_merge<N>(E, O, y);
#pragma unroll
    for (int i = 0; i < N; ++i) buf1[xbase + i] = y[i];
  }
  __syncthreads();  // #3
  // halo step B (3D): z-sides Q = M_y (M_x raw), columns along y, in place
  if (DIM == 3 && !(g.exp_flags & 4)) {
    for (int i = tid; i < 2 * C::NS2 * 2 * N; i += blockDim.x) {
      const int sw = i / N, xcol = i - sw * N;  // sw = (slot - SLOT2)*2 + which
      R *col = hbuf + (C::SLOT2 * 2 + sw) * LPC + xcol;
      R x[N];
#pragma unroll
      for (int q = 0; q < N; ++q) x[q] = col[q * N];
#pragma unroll
      for (int i2 = 0; i2 < N; ++i2) {
        R acc = 0.0;
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
    eo_split<N>(v, ev, ov);
    functionals();
  }
  __syncthreads();  // #4
  if (active) {
    R y[N], te[NE], to[H > 0 ? H : 1];
#pragma unroll
    for (int q = 0; q < N; ++q) y[q] = buf1[ybase + q * RP];
    eo_split<N>(y, te, to);
    if (DIM == 3) {  // Q = M_y P (own line; P was read before barrier #4)
      eo_apply<N, false>(T.Me, T.Mo, ev, ov, 1.0, E, O);
      eo_merge<N>(E, O, y);
#pragma unroll
      for (int i = 0; i < N; ++i) buf0[ybase + i * RP] = y[i];
    }
    eo_apply<N, false>(T.Me, T.Mo, te, to, 1.0, E, O);           // M_y T
    eo_apply<N, true>(T.Ke, T.Ko, ev, ov, scell[4 * c + 1], E, O);  // + s_y Kh_y P
    add_lifts(std::integral_constant<int, 1>());
    eo_merge<N>(E, O, y);
    if (DIM == 2) {
      const double wx = EPI == kEpiDot ? 0.25 * g.hx[x0 + jx] * g.hy[y0 + jy] * ea.wint[tb] : 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i)
        epi_store<EPI, DIM, N>(u, out, ea, e * NP + i * N + tb, y[i], wx * ea.wint[i], eacc);
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) buf1[ybase + i * RP] = y[i];  // G
    }
  }
  if (DIM == 2) {
    if (EPI == kEpiDot) epi_reduce(eacc, reinterpret_cast<double *>(fbuf), ea, bx + gridDim.x * (by + gridDim.y * bz));
    return;
  }
  __syncthreads();  // #5
  // ---- phase Z: z-lines of Q and G --------------------------------------------
  const int zbase = c * CS + ta * RP + tb;  // (y, x) line along z, stride N*RP
  if (EPI == kEpiCheb && active && !(g.exp_flags & 8)) {  // DG_EXP=8: off (timing A/B)
    // the Chebyshev epilogue reads rc, diag and x at this line's points:
    // start their L2 fetches now so they overlap the z functionals / sweep
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const size_t gi = e * NP + (i * N + ta) * N + tb;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(ea.rc + gi));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(ea.diag + gi));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(ea.x + gi));
    }
  }
  if (has_line) {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = buf0[zbase + q * N * RP];
    eo_split<N>(v, ev, ov);
    functionals();
  }
  __syncthreads();  // #6
  if (active) {
    R y[N], ge[NE], go[H > 0 ? H : 1];
#pragma unroll
    for (int q = 0; q < N; ++q) y[q] = buf1[zbase + q * N * RP];
    eo_split<N>(y, ge, go);
    eo_apply<N, false>(T.Me, T.Mo, ge, go, 1.0, E, O);           // M_z G
    eo_apply<N, true>(T.Ke, T.Ko, ev, ov, scell[4 * c + 2], E, O);  // + s_z Kh_z Q
    add_lifts(std::integral_constant<int, 2>());
    eo_merge<N>(E, O, y);
    const double wxy = EPI == kEpiDot ? 0.125 * g.hx[x0 + jx] * g.hy[y0 + jy] * g.hz[z0 + jz] *
                                            ea.wint[tb] * ea.wint[ta]
                                      : 0.0;
    if constexpr (EPI == kEpiCheb && !std::is_same<R, double>::value) {  // fp32 levels: same batching
      R rc[N], dg[N], xv[N], uv[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const size_t gi = e * NP + (i * N + ta) * N + tb;
        rc[i] = ea.rc[gi];
        dg[i] = ea.diag[gi];
        xv[i] = ea.x[gi];
        uv[i] = u[gi];
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const size_t gi = e * NP + (i * N + ta) * N + tb;
        const R r = rc[i] - y[i];
        const R dn = (R)ea.a * uv[i] + (R)ea.b * (r / dg[i]);
        ea.rc[gi] = r;
        ea.dnew[gi] = dn;
        ea.x[gi] = xv[i] + dn;
      }
    } else if constexpr (EPI == kEpiDot) {  // u of the line's points loaded before the out stores
      double pv[N];
#pragma unroll
      for (int i = 0; i < N; ++i) pv[i] = u[e * NP + (i * N + ta) * N + tb];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        out[e * NP + (i * N + ta) * N + tb] = y[i];
        eacc[0] += pv[i] * y[i];
        eacc[1] += y[i];
        eacc[2] += pv[i] * (wxy * ea.wint[i]);
      }
    } else if constexpr (EPI == kEpiCheb && std::is_same<R, double>::value) {
      // all operands of the line's N points loaded before any store (the
      // epilogue pointers may alias as far as the compiler knows, so per-point
      // load / store pairs serialised the L2 latency); same arithmetic as
      // epi_store
      double rc[N], dg[N], xv[N], uv[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const size_t gi = e * NP + (i * N + ta) * N + tb;
        rc[i] = ea.rc[gi];
        dg[i] = ea.diag[gi];
        xv[i] = ea.x[gi];
        uv[i] = u[gi];
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const size_t gi = e * NP + (i * N + ta) * N + tb;
        const double r = __dsub_rn(rc[i], y[i]);
        const double dn = __dadd_rn(__dmul_rn(ea.a, uv[i]), __dmul_rn(ea.b, __ddiv_rn(r, dg[i])));
        ea.rc[gi] = r;
        ea.dnew[gi] = dn;
        ea.x[gi] = __dadd_rn(xv[i], dn);
      }
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i)
        epi_store<EPI, DIM, N>(u, out, ea, e * NP + (i * N + ta) * N + tb, y[i], wxy * ea.wint[i],
                               eacc);
    }
  }
  if (EPI == kEpiDot) epi_reduce(eacc, reinterpret_cast<double *>(fbuf), ea, bx + gridDim.x * (by + gridDim.y * bz));
}

}  // namespace dg
