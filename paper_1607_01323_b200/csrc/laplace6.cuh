// SIP Laplace vmult, 3D Cartesian cells, register-plane variant (sm_100a, fp64).
//
// Same operator and separable form as laplace.cuh (reference
// operators.py:187-238):
//
//   out = M_z [ M_y ( s_x Kh_x u + s_x Lx ) + s_y Kh_y P + s_y Ly ]
//         + s_z Kh_z Q + s_z Lz,        P = M_x u,  Q = M_y P
//
// but with N threads per cell instead of N^2: in the XY phase thread (c, s)
// holds the z-slab s of cell c (an N x N plane) in registers and runs both
// the x-sweeps and the y-sweeps there, so only the z-sweep needs a
// shared-memory transpose (thread (c, s) then holds the y = s plane).  The
// even/odd 1D coefficients are held in registers for the whole kernel.
//
// Face coupling: each thread publishes the value / reference-derivative
// functionals of its lines' ends (u for x, P for y, Q for z) to shared
// memory and reads its neighbours' from there (in-brick), from the halo
// (neighbour cells across the brick surface, read once from L2 with their
// tangential masses applied in place), or from a zero block (boundary).
// Per (cell, side) the SIP flux collapses to three coefficients
//   cv = A (v_o - v_n) + B g_o + Dn g_n,   cd = B (v_o - v_n)
// (interior: A = tau s, B = sg s/h, Dn = sg s/h_n; velocity-Neumann: A = 2
// tau s, B = 2 sg s/h, Dn = 0; velocity-Dirichlet: 0), all division-free in
// the kernel (1/h per axis index precomputed on the host).
#pragma once
#include "laplace.cuh"
#include "tensor_fast.cuh"

namespace dg {

template <int N, int BX, int BY, int BZ>
struct Lap6Cfg {
  static constexpr int NC = BX * BY * BZ;
  static constexpr int NP = N * N * N;
  static constexpr int LPC = N * N;                        // lines per cell per direction
  static constexpr int PS = (N % 2 == 0) ? N * N + 1 : N * N;  // z-slab stride (pad even N)
  static constexpr int CS = N * PS;                        // cell stride
  static constexpr int NT = NC * N;                        // working threads
  static constexpr int THREADS = ((NT + 31) / 32) * 32;
  static constexpr int NS0 = BY * BZ, NS1 = BX * BZ, NS2 = BX * BY;
  static constexpr int SLOT0 = 0, SLOT1 = 2 * NS0, SLOT2 = 2 * NS0 + 2 * NS1;
  static constexpr int NSLOT = 2 * (NS0 + NS1 + NS2);
  static constexpr int HSIZE = NSLOT * 2 * LPC;           // [slot][v|g][LPC]
  static constexpr int BUF = NC * CS;
  // [cell][v0,g0,v1,g1][LPC], cell stride odd: the threads of a half-warp
  // (16 cells, same slab index) hit distinct banks
  static constexpr int FSTR = 4 * LPC + 1;
  static constexpr int FBUF = NC * FSTR;
  // whenever they fit (N >= 4): x functionals in buf1 (free until the G
  // planes), y and z functionals in buf0 (its planes are in registers by
  // then), the dot-product reduction scratch in fbz; else their own regions
  static constexpr bool FX_IN_BUF0 = FBUF <= BUF;
  static constexpr bool FY_IN_BUF1 = FBUF <= BUF;
  static constexpr int OFF_BUF1 = BUF;
  // x functionals go to buf1 (free until the G planes), y and z functionals
  // to buf0 (its planes are in registers by then): publishing the x
  // functionals needs no barrier after the u planes leave buf0
  static constexpr int OFF_FBX = FX_IN_BUF0 ? OFF_BUF1 : 2 * BUF;
  static constexpr int OFF_FBY = FY_IN_BUF1 ? 0 : 2 * BUF + (FX_IN_BUF0 ? 0 : FBUF);
  static constexpr int OFF_FBZ = FX_IN_BUF0 ? 0 : OFF_FBX;
  static constexpr int OFF_HRAW = 2 * BUF + (FX_IN_BUF0 ? 0 : FBUF) + (FY_IN_BUF1 ? 0 : FBUF);
  static constexpr int OFF_ZERO = OFF_HRAW + HSIZE;        // 2*LPC zeros (boundary neighbours)
  // per-cell tables with odd cell strides (a half-warp reads 16 cells' entries)
  // the context's cell table, brick rows as stored in global memory:
  // [cell][kCellTab] = side coefficients [side][A/tau_scale, B, Dn], then
  // s_d Kh scales (x, y, z), |cell|/8, pad (odd stride: conflict-free)
  static constexpr int SSTR = kCellTab;
  static constexpr int OFF_SIDE = OFF_ZERO + 2 * LPC;
  static constexpr int OFF_PTR = OFF_SIDE + SSTR * NC;     // halo sources
  static constexpr int OFF_BAR = OFF_PTR + NSLOT;
  static constexpr int NDBL = OFF_BAR + 1;
  static constexpr size_t SMEM = sizeof(double) * (size_t)NDBL + sizeof(int) * NC * 6;
  // the TMA row copies (PS == N*N) need 16-byte aligned shared addresses and
  // sizes: cell-table rows, brick rows and the table offset in doubles even
  static_assert(PS != N * N || (OFF_SIDE % 2 == 0 && (BX * SSTR) % 2 == 0 && (BX * NP) % 2 == 0),
                "TMA alignment of the brick rows");
};

// The context's cell table (once per context, one thread per (cell, side) and
// one per cell for the scales): the face coupling of every (cell, side) as
// three coefficients, A without tau_scale,
//   interior (operators.py:217-225): A = max(tau_e, tau_n) s, B = sg s/h, Dn = sg s/h_n
//   velocity-Neumann (:227-233):    A = 2 tau_e s,         B = 2 sg s/h, Dn = 0
//   velocity-Dirichlet (:189-193):  0
// with s the tangential face scale, then the per-cell stiffness scales and
// |cell|/8.  The vmult copies a brick's rows with its cells (TMA), so its
// prologue does index arithmetic only.
static __global__ void lap6_cell_table_kernel(const Geo g, double *tab) {
  const int64_t ncell = (int64_t)g.nx * g.ny * g.nz;
  const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (it >= ncell * 7) return;
  const int64_t e = it / 7;
  const int side = (int)(it - 7 * e);
  const int ix = (int)(e % g.nx), iy = (int)((e / g.nx) % g.ny), iz = (int)(e / ((int64_t)g.nx * g.ny));
  double *row = tab + e * kCellTab;
  const double h0 = g.hx[ix], h1 = g.hy[iy], h2 = g.hz[iz];
  if (side == 6) {
    row[18] = 0.5 * h1 * h2 * g.hxi[ix];
    row[19] = 0.5 * h0 * h2 * g.hyi[iy];
    row[20] = 0.5 * h0 * h1 * g.hzi[iz];
    row[21] = 0.125 * h0 * h1 * h2;
    row[22] = 0.0;
    return;
  }
  const int d = side >> 1, s = side & 1;
  const double *dummy = tab;  // resolve_nbr forms (never dereferenced) source pointers
  NbrInfo nb;
#define DG_RES(DD, SS) resolve_nbr<DD, SS, 3, 2, 1, 1, 1>(g, dummy, ix, iy, iz, 0, 0, 0, 0, 0, 0)
  switch (side) {
    case 0: nb = DG_RES(0, 0); break;
    case 1: nb = DG_RES(0, 1); break;
    case 2: nb = DG_RES(1, 0); break;
    case 3: nb = DG_RES(1, 1); break;
    case 4: nb = DG_RES(2, 0); break;
    default: nb = DG_RES(2, 1); break;
  }
#undef DG_RES
  const double taue = g.tau[e];
  const double hid = d == 0 ? g.hxi[ix] : (d == 1 ? g.hyi[iy] : g.hzi[iz]);
  const double sfac = d == 0 ? 0.25 * h1 * h2 : (d == 1 ? 0.25 * h0 * h2 : 0.25 * h0 * h1);
  const double sg = s ? -1.0 : 1.0;
  double A = 0.0, B = 0.0, Dn = 0.0;
  if (nb.kind <= 1) {
    A = fmax(taue, nb.tau) * sfac;
    B = sg * sfac * hid;
    Dn = sg * sfac * nb.hi;
  } else if (nb.kind == kBndNeumann) {
    A = 2.0 * taue * sfac;
    B = 2.0 * sg * sfac * hid;
  }
  row[3 * side] = A;
  row[3 * side + 1] = B;
  row[3 * side + 2] = Dn;
}

// 4 CTAs per SM need <= 168 registers at 96 threads: one more register drops
// the occupancy to 3 CTAs and costs ~30 % (measured)
template <int N, int BX, int BY, int BZ, int EPI = kEpiStore>
__global__ void __launch_bounds__(Lap6Cfg<N, BX, BY, BZ>::THREADS, 4)
laplace6_kernel(const double *__restrict__ u, double *__restrict__ out, const Geo g,
                const LapTab<N> T, const double tau_scale, const int part,
                const EpiArgs ea = EpiArgs{}) {
  using C = Lap6Cfg<N, BX, BY, BZ>;
  constexpr int LPC = C::LPC, CS = C::CS, PS = C::PS, NP = C::NP;
  constexpr int H = N / 2, NE = (N + 1) / 2, HO = H > 0 ? H : 1;
  extern __shared__ double smem[];
  double *buf0 = smem;
  double *buf1 = smem + C::OFF_BUF1;
  double *fbx = smem + C::OFF_FBX;
  double *fby = smem + C::OFF_FBY;
  double *fbz = smem + C::OFF_FBZ;
  double *hraw = smem + C::OFF_HRAW;
  double *sside = smem + C::OFF_SIDE;
  double *scell = sside + 18;  // per-cell scales at offset 18 of each table row
  const double **hsrc = reinterpret_cast<const double **>(smem + C::OFF_PTR);
  int *soff = reinterpret_cast<int *>(smem + C::NDBL);

  const int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z + g.bz0;
  const int x0 = bx * BX, y0 = by * BY, z0 = bz * BZ;
  const int ex = min(BX, g.nx - x0), ey = min(BY, g.ny - y0), ez = min(BZ, g.nz - z0);
  if (part != 0) {
    const bool touches = (g.mode[0] == kGhost && x0 == 0) || (g.mode[1] == kGhost && x0 + ex == g.nx);
    if ((part == 1 && touches) || (part == 2 && !touches)) return;
  }
  const int tid = threadIdx.x;

  // ---- own cells -> buf0 (TMA row copies for odd N) --------------------------
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
  constexpr int ROW = BX * NP;
  const bool tma = (PS == N * N) && !(ex & 1) && !(g.nx & 1) &&
                   ((reinterpret_cast<uintptr_t>(u) & 15) == 0);
  if (tma) {
    if (tid == 0) {
      mbar_init(bar, 1);
      mbar_expect_tx(bar, (uint32_t)(ey * ez * ex * (NP + C::SSTR) * sizeof(double)));
      for (int r = 0; r < BY * BZ; ++r) {
        const int jy = r % BY, jz = r / BY;
        if (jy >= ey || jz >= ez) continue;
        const size_t e0 = (size_t)x0 + (size_t)g.nx * ((y0 + jy) + (size_t)g.ny * (z0 + jz));
        bulk_g2s(buf0 + r * ROW, u + e0 * NP, (uint32_t)(ex * NP * sizeof(double)), bar);
        bulk_g2s(sside + r * BX * C::SSTR, g.ctab + e0 * C::SSTR,
                 (uint32_t)(ex * C::SSTR * sizeof(double)), bar);
      }
    }
  } else {
    for (int i = tid; i < C::NC * C::SSTR; i += blockDim.x) {
      const int cb = i / C::SSTR, w = i - cb * C::SSTR;
      const int jx = cb % BX, jy = (cb / BX) % BY, jz = cb / (BX * BY);
      sside[i] = (jx < ex && jy < ey && jz < ez)
                     ? g.ctab[((size_t)x0 + jx + (size_t)g.nx * ((y0 + jy) + (size_t)g.ny * (z0 + jz))) *
                                  C::SSTR + w]
                     : 0.0;
    }
    for (int i = tid; i < C::NC * NP; i += blockDim.x) {
      const int r = i / ROW, w = i - r * ROW;
      const int jx = w / NP, o = w - jx * NP;
      const int jy = r % BY, jz = r / BY;
      double v = 0.0;
      if (jx < ex && jy < ey && jz < ez)
        v = u[((size_t)x0 + (size_t)g.nx * ((y0 + jy) + (size_t)g.ny * (z0 + jz))) * NP + w];
      const int z = o / LPC;
      buf0[(r * BX + jx) * CS + z * PS + (o - z * LPC)] = v;
    }
  }

  // ---- setup: neighbour functional offsets and halo sources (index math only;
  // the coefficients arrive with the cells from the context's cell table)
  for (int it = tid; it < C::NC * 6; it += blockDim.x) {
    const int c = it / 6, side = it - 6 * c;
    const int d = side >> 1, s = side & 1;
    const int jx = c % BX, jy = (c / BX) % BY, jz = c / (BX * BY);
    const int pos = d == 0 ? jy + BY * jz : (d == 1 ? jx + BX * jz : jx + BX * jy);
    int off = C::OFF_ZERO;
    if (jx < ex && jy < ey && jz < ez) {
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
      if (kind == 1 && !ghost && nc >= lo && nc < lo + ext) {
        const int cb = d == 0 ? (nc - x0) + BX * (jy + BY * jz)
                              : (d == 1 ? jx + BX * ((nc - y0) + BY * jz)
                                        : jx + BX * (jy + BY * (nc - z0)));
        off = (d == 0 ? C::OFF_FBX : (d == 1 ? C::OFF_FBY : C::OFF_FBZ)) + cb * C::FSTR + (s ? 0 : 2) * LPC;
      } else if (kind == 1) {
        off = C::OFF_HRAW + slot_of<C>(d, s, pos) * 2 * LPC;
      }
    }
    soff[it] = off;
    const bool edge = d == 0 ? jx == (s ? ex - 1 : 0)
                             : (d == 1 ? jy == (s ? ey - 1 : 0) : jz == (s ? ez - 1 : 0));
    if (edge) {
      const int slot = slot_of<C>(d, s, pos);
      int dd, ss;
      hsrc[slot] = halo_slot_src<C, N, BX, BY, BZ>(g, u, slot, x0, y0, z0, ex, ey, ez, dd, ss);
    }
  }
  for (int i = tid; i < 2 * LPC; i += blockDim.x) smem[C::OFF_ZERO + i] = 0.0;
  __syncthreads();  // #1 tables, halo pointers

  // ---- halo: raw face functionals of neighbour cells across the brick -------
  // one item = (slot, a): an N x N tile of the neighbour cell (z-slab a for
  // x/y faces, y-row a for z faces; rows contiguous in global memory) ->
  // value and reference derivative at the facing end of its N normal lines
  if (!(g.exp_flags & 1)) {
    // one normal line per item, consecutive items = consecutive lines of one
    // neighbour cell: z faces read 25 contiguous doubles per position, y and x
    // faces a few cache lines per warp load (a tile per thread touches one
    // line per lane: 2 % slower, measured)
    constexpr int NIT = C::NSLOT * LPC;
    constexpr int U = (NIT + C::THREADS - 1) / C::THREADS;  // every load in flight at once
#pragma unroll 1
    for (int base = tid; base < NIT; base += U * C::THREADS) {
      double x[U][N];
      int dst[U], sd[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int it = base + k * C::THREADS;
        dst[k] = -1;
        sd[k] = 0;
        const int slot = it / LPC, t = it - slot * LPC;
        const double *src = it < NIT ? hsrc[slot] : nullptr;
        if (src != nullptr) {
          const int d = slot < C::SLOT1 ? 0 : (slot < C::SLOT2 ? 1 : 2);
          const int s = d == 0 ? slot >= C::NS0
                               : (d == 1 ? slot >= C::SLOT1 + C::NS1 : slot >= C::SLOT2 + C::NS2);
          const int a = t / N, b = t - a * N;
          // x line (y=b, z=a) | y line (x=b, z=a) | z line (x=b, y=a)
          // read the line from its facing end inwards (y[p], p = 0 at the face):
          // one derivative row for both sides, dR_q = -dL_{N-1-q}
          const int qs0 = d == 0 ? 1 : (d == 1 ? N : N * N);
          const int qs = s ? qs0 : -qs0;
          const double *l = (d == 2 ? src + t : src + a * N * N + (d == 0 ? b * N : b)) +
                            (s ? 0 : (N - 1) * qs0);
#pragma unroll
          for (int q = 0; q < N; ++q) x[k][q] = __ldg(l + q * qs);
          dst[k] = slot * 2 * LPC + t;
          sd[k] = s;
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if (dst[k] < 0) continue;
        double gs = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) gs += T.dL[q] * x[k][q];
        hraw[dst[k]] = x[k][0];
        hraw[dst[k] + LPC] = sd[k] ? gs : -gs;
      }
    }
  }
  if (tma) mbar_wait(bar, 0);
  else __syncthreads();

  // ---- per-thread coordinates ---------------------------------------------
  const bool has = tid < C::NT;
  // slab-major thread order: consecutive threads are different cells with the
  // same slab index, so the plane loads / stores (cell stride CS = N^3, odd
  // for odd N) and the functional buffers (odd stride) are bank-conflict free
  const int c = has ? tid % C::NC : 0;
  const int s = has ? tid / C::NC : 0;  // z-slab in the XY phase, y index in the Z phase
  // 1D coefficients in registers (indices are compile-time constants)
  double cMe[NE * NE], cMo[HO * HO], cKe[NE * NE], cKo[HO * HO], cLe[NE], cLo[HO];
#pragma unroll
  for (int i = 0; i < NE * NE; ++i) {
    cMe[i] = T.Me[i];
    cKe[i] = T.Ke[i];
  }
#pragma unroll
  for (int i = 0; i < HO * HO; ++i) {
    cMo[i] = H > 0 ? T.Mo[i] : 0.0;
    cKo[i] = H > 0 ? T.Ko[i] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < NE; ++i) cLe[i] = T.dLe[i];
#pragma unroll
  for (int i = 0; i < HO; ++i) cLo[i] = H > 0 ? T.dLo[i] : 0.0;

  double P[N][N], Tm[N][N];  // planes [row][col]

  // end functionals of a split line
  auto ends = [&](const double *e, const double *o, double &g0, double &g1) {
    double ge = 0.0, go = 0.0;
#pragma unroll
    for (int j = 0; j < NE; ++j) ge += cLe[j] * e[j];
#pragma unroll
    for (int j = 0; j < H; ++j) go += cLo[j] * o[j];
    g0 = ge + go;
    g1 = go - ge;
  };
  // publish the end functionals of the N lines get(l, q) (line l, position q)
  auto publish = [&](double *fb, int t0, auto get) {
    double *p = fb + c * C::FSTR + t0;
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double v[N], e[NE], o[HO], g0, g1;
#pragma unroll
      for (int q = 0; q < N; ++q) v[q] = get(l, q);
      eo_split<N>(v, e, o);
      ends(e, o, g0, g1);
      p[l] = v[0];
      p[LPC + l] = g0;
      p[2 * LPC + l] = v[N - 1];
      p[3 * LPC + l] = g1;
    }
  };
  // SIP face lifts of one line into its even/odd accumulators
  struct Side2 {
    double A0, B0, D0, A1, B1, D1;
    int o0, o1;
  };
  auto side2 = [&](int side0, int t0) {
    const double *c0 = sside + C::SSTR * c + 3 * side0;
    Side2 r;
    r.A0 = tau_scale * c0[0]; r.B0 = c0[1]; r.D0 = c0[2];
    r.A1 = tau_scale * c0[3]; r.B1 = c0[4]; r.D1 = c0[5];
    r.o0 = soff[c * 6 + side0] + t0;
    r.o1 = soff[c * 6 + side0 + 1] + t0;
    return r;
  };
  auto lift = [&](const Side2 &sd, int l, double v0, double g0, double v1, double g1, double *E,
                  double *O) {
    const double vn0 = smem[sd.o0 + l], gn0 = smem[sd.o0 + LPC + l];
    const double vn1 = smem[sd.o1 + l], gn1 = smem[sd.o1 + LPC + l];
    const double j0 = v0 - vn0, j1 = v1 - vn1;
    const double cv0 = sd.A0 * j0 + sd.B0 * g0 + sd.D0 * gn0, cd0 = sd.B0 * j0;
    const double cv1 = sd.A1 * j1 + sd.B1 * g1 + sd.D1 * gn1, cd1 = sd.B1 * j1;
    E[0] += 0.5 * (cv0 + cv1);
    if (H > 0) O[0] += 0.5 * (cv0 - cv1);
    const double dm = cd0 - cd1, dp = cd0 + cd1;
#pragma unroll
    for (int i = 0; i < NE; ++i) E[i] += cLe[i] * dm;
#pragma unroll
    for (int i = 0; i < H; ++i) O[i] += cLo[i] * dp;
  };

  // ---- XY-a: load the z-slab s (rows y, cols x); x-line functionals -------
  if (has) {
    const double *up = buf0 + c * CS + s * PS;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) P[j][i] = up[j * N + i];
  }
  if (has) publish(fbx, s * N, [&](int l, int q) { return P[l][q]; });  // x-lines t = z*N + y
  __syncthreads();  // #2
  // halo step A: y/z slots M_x in place (rows along x)
  if (!(g.exp_flags & 4)) {
    constexpr int ROWS = LPC / N;
    for (int i = tid; i < (C::NSLOT - C::SLOT1) * 2 * ROWS; i += blockDim.x) {
      const int sw = i / ROWS, a = i - sw * ROWS;
      double *row = hraw + (C::SLOT1 * 2 + sw) * LPC + a * N;
      double xr[N];
#pragma unroll
      for (int q = 0; q < N; ++q) xr[q] = row[q];
#pragma unroll
      for (int i2 = 0; i2 < N; ++i2) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) acc += T.M[i2 * N + q] * xr[q];
        row[i2] = acc;
      }
    }
  }
  // ---- XY-b: x-sweeps (rows): T = s_x Kh_x u + Lx, P = M_x u ----------------
  if (has) {
    const Side2 sd = side2(0, s * N);
    const double kx = scell[C::SSTR * c + 0];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double e[NE], o[HO], E[NE], O[HO], g0, g1;
      eo_split<N>(P[l], e, o);
      ends(e, o, g0, g1);
      eo_apply<N, false>(cKe, cKo, e, o, kx, E, O);
      lift(sd, l, P[l][0], g0, P[l][N - 1], g1, E, O);
      eo_merge<N>(E, O, Tm[l]);
      eo_apply<N, false>(cMe, cMo, e, o, 1.0, E, O);
      eo_merge<N>(E, O, P[l]);
    }
    publish(fby, s * N, [&](int l, int q) { return P[q][l]; });  // y-lines t = z*N + x
  }
  __syncthreads();  // #3
  // halo step B: z slots M_y in place (columns along y)
  if (!(g.exp_flags & 4)) {
    for (int i = tid; i < 2 * C::NS2 * 2 * N; i += blockDim.x) {
      const int sw = i / N, xcol = i - sw * N;
      double *col = hraw + (C::SLOT2 * 2 + sw) * LPC + xcol;
      double xr[N];
#pragma unroll
      for (int q = 0; q < N; ++q) xr[q] = col[q * N];
#pragma unroll
      for (int i2 = 0; i2 < N; ++i2) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) acc += T.M[i2 * N + q] * xr[q];
        col[i2 * N] = acc;
      }
    }
  }
  // ---- XY-c: y-sweeps (columns): G = M_y T + s_y Kh_y P + Ly, Q = M_y P ------
  if (has) {
    const Side2 sd = side2(2, s * N);
    const double ky = scell[C::SSTR * c + 1];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double v[N], w[N], e[NE], o[HO], te[NE], to[HO], E[NE], O[HO], g0, g1;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        v[q] = P[q][l];
        w[q] = Tm[q][l];
      }
      eo_split<N>(v, e, o);
      eo_split<N>(w, te, to);
      ends(e, o, g0, g1);
      eo_apply<N, false>(cMe, cMo, te, to, 1.0, E, O);
      eo_apply<N, true>(cKe, cKo, e, o, ky, E, O);
      lift(sd, l, v[0], g0, v[N - 1], g1, E, O);
      eo_merge<N>(E, O, w);
#pragma unroll
      for (int q = 0; q < N; ++q) Tm[q][l] = w[q];
      eo_apply<N, false>(cMe, cMo, e, o, 1.0, E, O);
      eo_merge<N>(E, O, v);
#pragma unroll
      for (int q = 0; q < N; ++q) P[q][l] = v[q];
    }
  }
  if (C::FY_IN_BUF1) __syncthreads();  // #3b: y functionals live in buf0 (Q goes there)
  if (has) {  // Q -> buf0 (z-slab s), G -> buf1
    double *q = buf0 + c * CS + s * PS, *gp = buf1 + c * CS + s * PS;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        q[j * N + i] = P[j][i];
        gp[j * N + i] = Tm[j][i];
      }
  }
  __syncthreads();  // #4
  // ---- Z-a: thread (c, s) takes the y = s plane [z][x]; z-line functionals --
  if (has) {
    const double *q = buf0 + c * CS + s * N, *gp = buf1 + c * CS + s * N;
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        P[z][i] = q[z * PS + i];
        Tm[z][i] = gp[z * PS + i];
      }
  }
  if (C::FX_IN_BUF0) __syncthreads();  // #4b: Q and G planes are in registers
  if (has) publish(fbz, s * N, [&](int l, int q2) { return P[q2][l]; });  // z-lines t = y*N + x
  __syncthreads();  // #5
  // ---- Z-b: out = M_z G + s_z Kh_z Q + Lz -> buf1 (y = s plane) ------------
  if (has) {
    const Side2 sd = side2(4, s * N);
    const double kz = scell[C::SSTR * c + 2];
    double *op = buf1 + c * CS + s * N;
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double v[N], w[N], e[NE], o[HO], ge[NE], go[HO], E[NE], O[HO], g0, g1;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        v[q] = P[q][l];
        w[q] = Tm[q][l];
      }
      eo_split<N>(v, e, o);
      eo_split<N>(w, ge, go);
      ends(e, o, g0, g1);
      eo_apply<N, false>(cMe, cMo, ge, go, 1.0, E, O);
      eo_apply<N, true>(cKe, cKo, e, o, kz, E, O);
      lift(sd, l, v[0], g0, v[N - 1], g1, E, O);
      eo_merge<N>(E, O, w);
#pragma unroll
      for (int q = 0; q < N; ++q) op[q * PS + l] = w[q];
    }
  }
  if (EPI == kEpiStore && tma && !(reinterpret_cast<uintptr_t>(out) & 15)) {
    // output rows are contiguous in shared and global memory: TMA bulk store
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // #6
    if (tid == 0) {
      for (int r = 0; r < BY * BZ; ++r) {
        const int ry = r % BY, rz = r / BY;
        if (ry >= ey || rz >= ez) continue;
        const size_t e0 = (size_t)x0 + (size_t)g.nx * ((y0 + ry) + (size_t)g.ny * (z0 + rz));
        bulk_s2g(out + e0 * NP, buf1 + r * ROW, (uint32_t)(ex * NP * sizeof(double)));
      }
      bulk_wait_read();
    }
    return;
  }
  __syncthreads();  // #6
  // ---- epilogue: per brick row, contiguous in global memory ----------------
  double eacc[3] = {0.0, 0.0, 0.0};
  for (int r = 0; r < BY * BZ; ++r) {
    const int ry = r % BY, rz = r / BY;
    if (ry >= ey || rz >= ez) continue;
    const size_t g0 = ((size_t)x0 + (size_t)g.nx * ((y0 + ry) + (size_t)g.ny * (z0 + rz))) * NP;
    for (int w = tid; w < ex * NP; w += blockDim.x) {
      int si, cb = 0, z = 0, yx = 0;
      if (PS == N * N && EPI != kEpiDot) {
        si = r * ROW + w;  // unpadded: the row is contiguous in shared memory too
      } else {
        const int cx = w / NP, o = w - cx * NP;
        cb = r * BX + cx;
        z = o / LPC;
        yx = o - z * LPC;
        si = cb * CS + z * PS + yx;
      }
      double wq = 0.0;
      if (EPI == kEpiDot) {
        const int yy = yx / N, xx = yx - yy * N;
        wq = scell[C::SSTR * cb + 3] * ea.wint[xx] * ea.wint[yy] * ea.wint[z];
      }
      epi_store<EPI, 3, N>(u, out, ea, g0 + w, buf1[si], wq, eacc);
    }
  }
  if (EPI == kEpiDot) epi_reduce(eacc, fbz, ea, bx + gridDim.x * (by + gridDim.y * bz));
}

}  // namespace dg
