// SIP Laplace vmult, 3D Cartesian cells: z-marching column kernel (sm_100a,
// fp64).  Replaces apply_pressure_laplace (reference operators.py:187-238).
//
// Operator (exact on axis-aligned cells, Gauss rule n_q = N):
//   L u = Ax (x) My (x) Mz u + Mx (x) Ay (x) Mz u + Mx (x) My (x) Az u
// with M = S^T W S, A_d = s_d Kh_d + (SIP face lifts along d), factored
// z-first so that every cell needs only the RAW face functionals of its
// z-neighbours:
//   W = Mz u,  R = Az u              (z-lines; lifts from raw u functionals)
//   T = Ax W + Mx R,  V = Mx W       (x-lines; lifts from W functionals)
//   out = My T + Ay V                (y-lines; lifts from V functionals)
// 7 one-dimensional sweeps per cell, all in even-odd form.
//
// Work decomposition.  A CTA owns a column: a TX x TY tile of cells in x-y
// and a range of z layers, and marches through it layer by layer.
// * Layers arrive by TMA bulk copies into an NRING-slot ring, issued
//   NRING - 2 layers ahead of the look-ahead use.  The z-neighbour below is
//   carried in registers (the top functionals of the previous layer), the one
//   above is read from the next ring slot, so no z halo is ever re-read.
// * z phase: thread (c, s) takes the ZX plane y = s of tile cell c, runs the
//   z-lines and writes W in place over u and R to a transpose buffer.
// * xy phase (one CTA barrier later): thread (c, s) takes the XY plane z = s,
//   runs the x-lines (rows) and the y-lines (columns) in registers and writes
//   out in place over W; the ring slot leaves by TMA bulk stores.
//   The threads of one plane index s are one group of NCT consecutive lanes,
//   so x- and y-neighbour face functionals inside the tile move by warp
//   shuffles.
// * Neighbours across the tile edge (halo): loads issued at the start of the
//   z phase, reduced at its end to facing-end value/derivative with M_z
//   (stage 1); y-halo rows get their M_x one layer later (stage 2), always
//   before the xy phase that reads them.
// Two CTA barriers per layer.  Face coefficients come from per-axis cell
// data (Geo::ax) and per-column constants computed once; no per-cell table.
// No atomics: every output DoF is written once.
#pragma once
#include "laplace.cuh"
#include "tensor_fast.cuh"

namespace dg {

template <int N>
struct L7Stride {  // shared-memory cell stride (doubles): odd N unpadded (rows
                   // contiguous, conflict-free 8-byte lanes), even N padded to
                   // a 16-byte multiple that is conflict-free for 16-byte lanes
  static constexpr int NP = N * N * N;
  static constexpr int value = (N & 1) ? NP : (N == 4 ? 66 : (N == 6 ? 218 : NP + 2));
};

template <int N, int TX, int TY, int NRING>
struct Lap7Cfg {
  static constexpr int NCT = TX * TY;  // cells per tile layer = lanes per plane group
  static_assert(NCT == 16 || NCT == 32, "plane group of 16 or 32 lanes");
  static_assert(NRING >= 2 && NRING <= 4, "ring depth");
  static constexpr int NP = N * N * N;
  static constexpr int CSTR = L7Stride<N>::value;
  static constexpr int THREADS = ((N * NCT + 31) / 32) * 32;
  // plane groups s >= N (when N * NCT is not a warp multiple) are idle: they
  // run the same code on a scratch cell slot and store nothing that is read
  static constexpr bool IDLE = THREADS > N * NCT;
  static constexpr int LAYER = (((NCT + (IDLE ? 1 : 0)) * CSTR + 1) / 2) * 2;  // 16-byte multiple
  static constexpr int OFF_R = NRING * LAYER;
  static constexpr int HXN = 2 * TY * N * N * 2;  // [side][jy][y][z][v|g]
  static constexpr int HYN = 2 * TX * N * N * 2;  // [side][jx][x][z][v|g]
  static constexpr int OFF_HX = OFF_R + LAYER;    // two parities
  static constexpr int OFF_HY = OFF_HX + 2 * HXN;
  static constexpr int CCS = 15;                  // per-cell column constants (odd stride)
  static constexpr int OFF_CC = OFF_HY + 2 * HYN;
  static constexpr int LCMAX = 64;                // z-chunk length limit
  static constexpr int OFF_ZD = OFF_CC + NCT * CCS;  // [layer - z0 + 1][h, 1/h, tau part, 0]
  static constexpr int OFF_ZERO = OFF_ZD + 4 * (LCMAX + 2);  // zero block (boundary sides)
  static constexpr int OFF_BAR = OFF_ZERO + 2 * N * N;
  static constexpr int NDBL = OFF_BAR + NRING;
  static constexpr size_t SMEM = sizeof(double) * (size_t)NDBL;
  static constexpr int HITEMS = 2 * N * (TX + TY);  // halo stage-1 items per layer
  static constexpr int HROWS = 2 * TX * N * 2;      // halo stage-2 rows per layer
  static_assert(HITEMS <= THREADS, "one halo item per thread");
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// SIP coefficients of one side: cv = A (v - vn) + B g + D gn, cd = B (v - vn)
struct Side7 {
  double A, B, D;
};

// kind: 0 neighbour inside the tile / the z ring, 1 halo, kBndNone, kBndNeumann;
// tmax = tau of max(tau_e, tau_n) (interior) ; taue = tau_e (Neumann)
__device__ __forceinline__ Side7 side7(int kind, double tmax, double taue, double sfac,
                                       double hid, double hin, double sg, double ts) {
  Side7 r{0.0, 0.0, 0.0};
  if (kind <= 1) {
    r.A = ts * (tmax * sfac);
    r.B = sg * sfac * hid;
    r.D = sg * sfac * hin;
  } else if (kind == kBndNeumann) {
    r.A = ts * (2.0 * taue * sfac);
    r.B = 2.0 * sg * sfac * hid;
  }
  return r;
}

// kind of the x / y neighbour of global cell index i (axis extent n, tile
// range [lo, lo + ext)) across side S; lane offset of the in-tile neighbour
template <int S>
__device__ __forceinline__ int kind7(const Geo &g, int d, int i, int n, int lo, int ext, int &nl) {
  int nc = i + (S ? 1 : -1);
  if (nc < 0 || nc >= n) {
    const int m = g.mode[2 * d + S];
    if (m == kWrap) nc = S ? 0 : n - 1;
    else if (m == kGhost) return 1;
    else return m;
  }
  if (nc >= lo && nc < lo + ext) {
    nl = nc - lo;
    return 0;
  }
  return 1;
}

template <int N>
__device__ __forceinline__ void l7_ends(const LapTab<N> &T, const double *e, const double *o,
                                        double &g0, double &g1) {
  constexpr int H = N / 2, NE = (N + 1) / 2;
  double ge = 0.0, go = 0.0;
#pragma unroll
  for (int j = 0; j < NE; ++j) ge += T.dLe[j] * e[j];
#pragma unroll
  for (int j = 0; j < H; ++j) go += T.dLo[j] * o[j];
  g0 = ge + go;  // dL . v
  g1 = go - ge;  // dR . v
}

// SIP face lifts of one line into its even/odd accumulators
template <int N>
__device__ __forceinline__ void l7_lift(const LapTab<N> &T, const Side7 &s0, const Side7 &s1,
                                        double v0, double g0, double vn0, double gn0, double v1,
                                        double g1, double vn1, double gn1, double *E, double *O) {
  constexpr int H = N / 2, NE = (N + 1) / 2;
  const double j0 = v0 - vn0, j1 = v1 - vn1;
  const double cv0 = s0.A * j0 + s0.B * g0 + s0.D * gn0, cd0 = s0.B * j0;
  const double cv1 = s1.A * j1 + s1.B * g1 + s1.D * gn1, cd1 = s1.B * j1;
  E[0] += 0.5 * (cv0 + cv1);
  if (H > 0) O[0] += 0.5 * (cv0 - cv1);
  const double dm = cd0 - cd1, dp = cd0 + cd1;
#pragma unroll
  for (int i = 0; i < NE; ++i) E[i] += T.dLe[i] * dm;
#pragma unroll
  for (int i = 0; i < H; ++i) O[i] += T.dLo[i] * dp;
}

template <int N>
__device__ __forceinline__ void l7_mass(const LapTab<N> &T, const double *v, double *y) {
  constexpr int H = N / 2, NE = (N + 1) / 2;
  double e[NE], o[H > 0 ? H : 1], E[NE], O[H > 0 ? H : 1];
  eo_split<N>(v, e, o);
  eo_apply<N, false>(T.Me, T.Mo, e, o, 1.0, E, O);
  eo_merge<N>(E, O, y);
}

// neighbour functional: in-tile by shuffle, else from shared memory (the halo
// block, or a zero block on boundary sides) -- one select, no branch
__device__ __forceinline__ double l7_pick(int kind, double shfl, double smem_val) {
  return kind == 0 ? shfl : smem_val;
}

// EPI = kEpiCheb: instead of storing out, each finished layer runs the fused
// Chebyshev step on its points (laplace.cuh epi_store arithmetic): rc -= out,
// dnew = a u + b rc / diag, x += dnew; the layer's operands are prefetched
// into L2 during its z phase and loaded four points per thread at a time.
// With several CTAs per SM one CTA's epilogue overlaps the others' sweeps.
template <int N, int TX, int TY, int NRING, int MINB, bool STAGE, int EPI = kEpiStore, int HSPL = 0>
__global__ void __launch_bounds__(Lap7Cfg<N, TX, TY, NRING>::THREADS, MINB)
laplace7_kernel(const double *__restrict__ u, double *__restrict__ out, const Geo g,
                const __grid_constant__ LapTab<N> T, const double ts, const int part,
                const int zlo, const int zhi, const int lc, const int ntx, const int nty,
                const EpiArgs ea = EpiArgs{}) {
  static_assert(EPI == kEpiStore || EPI == kEpiCheb, "laplace7: store or Chebyshev epilogue");
  using C = Lap7Cfg<N, TX, TY, NRING>;
  constexpr int NCT = C::NCT, NP = C::NP, CSTR = C::CSTR, H = N / 2, NE = (N + 1) / 2;
  constexpr int HO = H > 0 ? H : 1;
  constexpr int N2 = N * N;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double smem[];
  double *const ring = smem;
  double *const rbuf = smem + C::OFF_R;
  double *const hxb = smem + C::OFF_HX;
  double *const hyb = smem + C::OFF_HY;
  double *const cc = smem + C::OFF_CC;
  uint64_t *const bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
  const double *const zero = smem + C::OFF_ZERO;

  // ---- unit: tile (tx, ty) x z-chunk -------------------------------------
  int unit = blockIdx.x;
  const int tix = unit % ntx;
  unit /= ntx;
  const int tiy = unit % nty;
  const int chunk = unit / nty;
  const int x0 = tix * TX, y0 = tiy * TY;
  const int ex = min(TX, g.nx - x0), ey = min(TY, g.ny - y0);
  const int z0 = zlo + chunk * lc, z1 = min(zhi, z0 + lc);
  if (z0 >= z1) return;
  if (part != 0) {
    const bool touches = (g.mode[0] == kGhost && x0 == 0) || (g.mode[1] == kGhost && x0 + ex == g.nx);
    if ((part == 1 && touches) || (part == 2 && !touches)) return;
  }
  const int nlay = z1 - z0;
  const size_t nxy = (size_t)g.nx * g.ny;

  const int tid = threadIdx.x;
  const int c = tid % NCT, sraw = tid / NCT;
  const bool live = sraw < N;
  const int s = live ? sraw : N - 1;
  const int cs = live ? c : NCT;  // shared-memory cell slot (idle groups: scratch)
  const int jx = c % TX, jy = c / TX;
  const int ix = x0 + min(jx, ex - 1), iy = y0 + min(jy, ey - 1);  // clamped (inactive lanes)

  // ---- per-column constants and neighbour kinds --------------------------
  int kx0, kx1, ky0, ky1, lx0 = 0, lx1 = 0, ly0 = 0, ly1 = 0;
  {
    int nl = 0;
    kx0 = kind7<0>(g, 0, ix, g.nx, x0, ex, nl);
    lx0 = nl + TX * jy;
    kx1 = kind7<1>(g, 0, ix, g.nx, x0, ex, nl);
    lx1 = nl + TX * jy;
    ky0 = kind7<0>(g, 1, iy, g.ny, y0, ey, nl);
    ly0 = jx + TX * nl;
    ky1 = kind7<1>(g, 1, iy, g.ny, y0, ey, nl);
    ly1 = jx + TX * nl;
    if (kx0 != 0) lx0 = c;
    if (kx1 != 0) lx1 = c;
    if (ky0 != 0) ly0 = c;
    if (ky1 != 0) ly1 = c;
  }
  if (tid < NCT) {
    const double *ax = g.ax[0] + 4 * ix, *ay = g.ax[1] + 4 * iy;
    const double hx = ax[0], hxi = ax[1], tx = ax[2];
    const double hy = ay[0], hyi = ay[1], ty = ay[2];
    double *q = cc + c * C::CCS;
    q[0] = 0.25 * hx * hy;                 // z-face scale
    q[1] = 0.5 * hx * hy;                  // kz / (1/hz)
    q[2] = tx + ty;                        // tau_e - tau_z
    q[3] = hy;
    q[4] = hxi;
    q[5] = fmax(tx, ax[-4 + 2]) + ty;      // x side 0: max(tau) - tau_z
    q[6] = fmax(tx, ax[4 + 2]) + ty;       // x side 1
    q[7] = ax[-4 + 1];                     // 1/h of the x neighbours
    q[8] = ax[4 + 1];
    q[9] = hx;
    q[10] = hyi;
    q[11] = tx + fmax(ty, ay[-4 + 2]);     // y sides
    q[12] = tx + fmax(ty, ay[4 + 2]);
    q[13] = ay[-4 + 1];
    q[14] = ay[4 + 1];
  }
  for (int i = tid; i < 2 * N * N; i += C::THREADS) smem[C::OFF_ZERO + i] = 0.0;
  double *const zd = smem + C::OFF_ZD;  // z data of layers z0 - 1 .. z1
  for (int i = tid; i < 4 * (nlay + 2); i += C::THREADS) zd[i] = g.ax[2][4 * (z0 - 1) + i];

  // ---- ring ----------------------------------------------------------------
  // ring position r: 0 = the layer below the column, 1..nlay = the column,
  // nlay + 1 = the layer above; slot r % NRING, mbarrier use r / NRING
  auto layer_of = [&](int r) -> int {
    const int z = z0 + r - 1;
    if (z < 0) return g.mode[4] == kWrap ? g.nz - 1 : -1;
    if (z >= g.nz) return g.mode[5] == kWrap ? 0 : -1;
    return z;
  };
  // odd N: one bulk copy per tile row (contiguous cells); even N: one per cell
  const bool rows_ok = (N & 1) ? (!(g.nx & 1) && !(ex & 1)) : true;
  const bool tma = rows_ok && !(reinterpret_cast<uintptr_t>(u) & 15) &&
                   !(reinterpret_cast<uintptr_t>(out) & 15);
  if (tid == 0)
    for (int i = 0; i < NRING; ++i) mbar_init(&bar[i], 1);
  __syncthreads();
  // all threads call issue(); thread 0 issues TMA, or all threads copy
  auto issue = [&](int r) {
    if (tma && tid >= 32) return;  // TMA: warp 0 alone (no per-warp layer arithmetic)
    if (r > nlay + 1) return;
    const int lay = layer_of(r);
    uint64_t *b = &bar[r % NRING];
    if (lay < 0) {  // complete the phase anyway: later parities stay aligned
      if (tma && tid == 0) mbar_arrive(b);
      return;
    }
    double *dst = ring + (r % NRING) * C::LAYER;
    if (tma) {
      // warp 0: lane 0 arms the barrier, then one bulk copy per lane (a tile
      // row for odd N, a cell for even N)
      if (tid >= 32) return;
      if (tid == 0) mbar_expect_tx(b, (uint32_t)(ex * ey * NP * sizeof(double)));
      __syncwarp();
      const int nitem = (N & 1) ? ey : ex * ey;
      for (int i = tid; i < nitem; i += 32) {
        const int xx = (N & 1) ? 0 : i % ex, yy = (N & 1) ? i : i / ex;
        const size_t e0 = (size_t)x0 + xx + (size_t)g.nx * (y0 + yy) + nxy * lay;
        bulk_g2s(dst + (xx + TX * yy) * CSTR, u + e0 * NP,
                 (uint32_t)(((N & 1) ? ex : 1) * NP * sizeof(double)), b);
      }
    } else {  // unaligned rows: plain copies (visible after the next CTA barrier)
      for (int i = tid; i < ex * ey * NP; i += C::THREADS) {
        const int cl = i / NP, w = i - cl * NP;
        const int xx = cl % ex, yy = cl / ex;
        dst[(xx + TX * yy) * CSTR + w] =
            u[((size_t)x0 + xx + (size_t)g.nx * (y0 + yy) + nxy * lay) * NP + w];
      }
    }
  };
  auto wait_slot = [&](int r) {
    if (tma && layer_of(r) >= 0) mbar_wait(&bar[r % NRING], (r / NRING) & 1);
  };

  // ---- halo --------------------------------------------------------------------
  // stage 1, item < 2 TY N: x halo (side, row jy, y): the ZX plane y of the
  //   neighbour -> facing-end value / derivative along x, then M_z (final);
  // else y halo (side, column jx, x): the ZY plane x -> facing end along y,
  //   then M_z; stage 2 (next layer's z phase) applies M_x along x.
  const int hit = tid;
  const bool hx_item = hit < 2 * TY * N;
  int hside = 0, hrow = 0, hpos = 0;
  if (hit < C::HITEMS) {
    const int it = hx_item ? hit : hit - 2 * TY * N;
    const int per = hx_item ? TY * N : TX * N;
    hside = it / per;
    const int rem = it - hside * per;
    hrow = rem / N;
    hpos = rem - hrow * N;
  }
  int htrace = 0;
  auto halo_src = [&](int lay) -> const double * {
    htrace = 0;
    if (hit >= C::HITEMS || lay < 0) return nullptr;
    if (hx_item) {
      if (hrow >= ey) return nullptr;
      const int yy = y0 + hrow;
      int nc = hside ? x0 + ex : x0 - 1;
      if (nc < 0 || nc >= g.nx) {
        const int m = g.mode[hside];
        if (m == kWrap) nc = hside ? 0 : g.nx - 1;
        else if (m == kGhost) {  // remote neighbour: its face traces (or whole cells)
          htrace = g.ghost_traces;
          return g.ghost[hside] + ((size_t)yy + (size_t)g.ny * lay) * (htrace ? 2 * N2 : NP);
        }
        else return nullptr;
      }
      if (nc >= x0 && nc < x0 + ex) return nullptr;  // wraps onto the tile itself
      return u + ((size_t)nc + (size_t)g.nx * yy + nxy * lay) * NP;
    }
    if (hrow >= ex) return nullptr;
    const int xx = x0 + hrow;
    int nc = hside ? y0 + ey : y0 - 1;
    if (nc < 0 || nc >= g.ny) {
      const int m = g.mode[2 + hside];
      if (m == kWrap) nc = hside ? 0 : g.ny - 1;
      else return nullptr;
    }
    if (nc >= y0 && nc < y0 + ey) return nullptr;
    return u + ((size_t)xx + (size_t)g.nx * nc + nxy * lay) * NP;
  };
  // HSPL: the halo item's N z-rows are loaded in HSPL + 1 parts of NH rows
  // (part j + 1 issued part-way through the z lines, once part j is reduced
  // to its facing-end value / derivative): NH rows of registers instead of N
  constexpr int NPART = HSPL + 1;
  constexpr int NH = (N + NPART - 1) / NPART;
  double hreg[NH][N];
  double v[N], gg[N];  // facing-end value / derivative per z row
  const double *hsrc = nullptr;
  auto halo_load = [&](int lay, int hf) {
    if (hf == 0) hsrc = halo_src(lay);
    if (!hsrc) return;
    const int zb = hf * NH, ze = min(N, zb + NH);
    if (htrace) {  // [z][y][v|g] of the facing end, raw (M_z below)
#pragma unroll
      for (int z = zb; z < ze; ++z) {
        hreg[z - zb][0] = __ldg(hsrc + (z * N + hpos) * 2);
        hreg[z - zb][1] = __ldg(hsrc + (z * N + hpos) * 2 + 1);
      }
      return;
    }
#pragma unroll
    for (int z = zb; z < ze; ++z)
#pragma unroll
      for (int q = 0; q < N; ++q)
        // x halo: [z][x] of plane y = hpos ; y halo: [z][y] of plane x = hpos
        hreg[z - zb][q] = __ldg(hsrc + z * N2 + (hx_item ? hpos * N + q : q * N + hpos));
  };
  auto halo_reduce = [&](int hf) {  // rows of part hf (all rows without HSPL)
    if (!hsrc) return;
    const int zb = hf * NH, ze = min(N, zb + NH);
#pragma unroll
    for (int z = zb; z < ze; ++z) {
      double e[NE], o[HO], g0, g1;
      eo_split<N>(hreg[z - zb], e, o);
      l7_ends<N>(T, e, o, g0, g1);
      // lower side (hside 0): the neighbour's upper end faces the tile
      v[z] = htrace ? hreg[z - zb][0] : (hside ? hreg[z - zb][0] : hreg[z - zb][N - 1]);
      gg[z] = htrace ? hreg[z - zb][1] : (hside ? g0 : g1);
    }
  };
  auto halo_stage1 = [&](int par) {
    if (!hsrc) return;
    halo_reduce(NPART - 1);
    double mv[N], mg[N];
    l7_mass<N>(T, v, mv);
    l7_mass<N>(T, gg, mg);
    double *hp = hx_item ? hxb + par * C::HXN + ((hside * TY + hrow) * N + hpos) * N * 2
                         : hyb + par * C::HYN + ((hside * TX + hrow) * N + hpos) * N * 2;
#pragma unroll
    for (int z = 0; z < N; ++z) {
      hp[2 * z] = mv[z];
      hp[2 * z + 1] = mg[z];
    }
  };
  // one stage-2 row per thread (the Q3 / Q5 tiles): its offset resolved once
  int s2off = -1;
  if (C::HROWS <= C::THREADS && tid < C::HROWS) {
    const int vg = tid & 1, rz = tid >> 1, z = rz % N, sj = rz / N;
    if ((sj % TX) < ex) s2off = sj * N * N * 2 + z * 2 + vg;
  }
  auto halo_stage2 = [&](int par) {  // y halo: M_x along x, rows (side, jx, z, v|g)
    if (C::HROWS <= C::THREADS) {
      if (s2off < 0) return;
      double *row = hyb + par * C::HYN + s2off;
      double v[N], y[N];
#pragma unroll
      for (int x = 0; x < N; ++x) v[x] = row[x * N * 2];
      l7_mass<N>(T, v, y);
#pragma unroll
      for (int x = 0; x < N; ++x) row[x * N * 2] = y[x];
      return;
    }
    for (int i = tid; i < C::HROWS; i += C::THREADS) {
      const int vg = i & 1, rz = i >> 1;
      const int z = rz % N, sj = rz / N;  // sj = side * TX + jx
      if ((sj % TX) >= ex) continue;
      double *row = hyb + par * C::HYN + sj * N * N * 2 + z * 2 + vg;
      double v[N], y[N];
#pragma unroll
      for (int x = 0; x < N; ++x) v[x] = row[x * N * 2];
      l7_mass<N>(T, v, y);
#pragma unroll
      for (int x = 0; x < N; ++x) row[x * N * 2] = y[x];
    }
  };

  // ---- prologue ------------------------------------------------------------------
  for (int r = 0; r < NRING; ++r) issue(r);
  double ztv[N], ztg[N];  // raw top functionals of the layer below (z-line x of plane y = s)
#pragma unroll
  for (int x = 0; x < N; ++x) {
    ztv[x] = 0.0;
    ztg[x] = 0.0;
  }
  halo_load(layer_of(1), 0);
#pragma unroll
  for (int j = 1; j < NPART; ++j) {
    halo_reduce(j - 1);
    halo_load(layer_of(1), j);
  }
  if (!tma) __syncthreads();
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
  halo_stage1(0);
  __syncthreads();  // slot 0 consumed, halo stage 1 of the first layer, cc

  // ---- march ---------------------------------------------------------------------------
  for (int p = 0; p < nlay; ++p) {
    const int r = p + 1;  // ring position of this layer
    const int iz = z0 + p;
    const int par = p & 1;
    double *const slot = ring + (r % NRING) * C::LAYER;
    const double *az = zd + 4 * (p + 1);
    const double hz = az[0], hzi = az[1], tz = az[2];

    // ================= z phase: W = M_z u (in place), R = A_z u =================
    // the ring slot of layer p - 1 gets ring position r + NRING - 1 once the
    // out rows of layer p - 1 have left it: NRING 2 here (it is this layer's
    // look-ahead), NRING 3 in the middle of the z lines, NRING 4 after them
    auto refill = [&]() {
      if (tid < 32 && tma) bulk_wait_read();
      issue(r + NRING - 1);
    };
    if (NRING == 2) {
      refill();
      if (!tma) __syncthreads();  // plain copies of the look-ahead layer
    }
    wait_slot(r);
    const int lay_up = layer_of(r + 1);
    wait_slot(r + 1);
    const bool more = p + 1 < nlay;
    halo_load(more ? iz + 1 : -1, 0);
    halo_stage2(par);
    if (EPI == kEpiCheb) {  // this layer's epilogue operands -> L2 (128 B lines)
      const int npts = ex * ey * NP;
      for (int i = tid * 16; i < 4 * npts; i += 16 * C::THREADS) {
        const int v = i / npts, j = i - v * npts, cl = j / NP, w = j - cl * NP;
        const size_t gi = ((size_t)x0 + cl % ex + (size_t)g.nx * (y0 + cl / ex) + nxy * iz) * NP + w;
        const double *pp = v == 0 ? ea.rc : (v == 1 ? ea.diag : (v == 2 ? ea.x : u));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pp + gi));
      }
    }
    {
      const double *q = cc + c * C::CCS;
      const double sfz = q[0], kz = q[1] * hzi, txy = q[2];
      const double taue = txy + tz;
      const int kz0 = iz == 0 ? (g.mode[4] == kWrap ? 0 : g.mode[4]) : 0;
      const int kz1 = iz == g.nz - 1 ? (g.mode[5] == kWrap ? 0 : g.mode[5]) : 0;
      // z-face tau = max of the two cells' z parts (plain compare, no fmax NaN fix-up)
      const double tzl = az[-4 + 2], tzu = az[4 + 2];
      const Side7 s0 = side7(kz0, txy + (tz > tzl ? tz : tzl), taue, sfz, hzi, az[-4 + 1], 1.0, ts);
      const Side7 s1 = side7(kz1, txy + (tz > tzu ? tz : tzu), taue, sfz, hzi, az[4 + 1], -1.0, ts);
      double *up = slot + cs * CSTR + s * N;
      double *rp = rbuf + cs * CSTR + s * N;
      const double *lp = ring + ((r + 1) % NRING) * C::LAYER + cs * CSTR + s * N;
      const bool la_ok = lay_up >= 0;
#pragma unroll
      for (int x = 0; x < N; ++x) {
        double w[N], e[NE], o[HO], E[NE], O[HO], g0, g1;
#pragma unroll
        for (int z = 0; z < N; ++z) w[z] = up[z * N2 + x];
        // the layer above: bottom value and dL derivative (stale slot data when
        // there is none: selected away)
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
        if (NRING == 3 && x == N / 2) refill();
#pragma unroll
        for (int j = 1; j < NPART; ++j)
          if (x == (j * N) / NPART - 1) {
            halo_reduce(j - 1);
            halo_load(more ? iz + 1 : -1, j);
          }
      }
    }
    if (NRING == 4) refill();
    halo_stage1(par ^ 1);
    __syncthreads();  // B_a: W, R complete; halo of this layer complete

    // ================= xy phase: T = A_x W + M_x R, V = M_x W; out = M_y T + A_y V =========
    {
      const double *q = cc + c * C::CCS;
      const double hy = q[3], hxi = q[4], hx = q[9], hyi = q[10];
      const double taue = q[2] + tz;
      // T, V rows: registers, or (STAGE) written over this thread's W / R rows
      double Tp[STAGE ? 1 : N][N], Vp[STAGE ? 1 : N][N];
      {
        const double sfx = 0.25 * hy * hz, kx = 0.5 * hy * hz * hxi;
        const Side7 s0 = side7(kx0, q[5] + tz, taue, sfx, hxi, q[7], 1.0, ts);
        const Side7 s1 = side7(kx1, q[6] + tz, taue, sfx, hxi, q[8], -1.0, ts);
        const double *wp = slot + cs * CSTR + s * N2;
        const double *rp = rbuf + cs * CSTR + s * N2;
        double *tsp = slot + cs * CSTR + s * N2, *rsp = rbuf + cs * CSTR + s * N2;
        const double *h0 = kx0 == 1 ? hxb + par * C::HXN + (jy * N) * N * 2 + 2 * s : zero;
        const double *h1 = kx1 == 1 ? hxb + par * C::HXN + ((TY + jy) * N) * N * 2 + 2 * s : zero;
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
          const double vn0 = l7_pick(kx0, __shfl_sync(FULL, v1, lx0, NCT), h0[y * N * 2]);
          const double gn0 = l7_pick(kx0, __shfl_sync(FULL, g1, lx0, NCT), h0[y * N * 2 + 1]);
          const double vn1 = l7_pick(kx1, __shfl_sync(FULL, v0, lx1, NCT), h1[y * N * 2]);
          const double gn1 = l7_pick(kx1, __shfl_sync(FULL, g0, lx1, NCT), h1[y * N * 2 + 1]);
          eo_apply<N, false>(T.Ke, T.Ko, e, o, kx, E, O);
          eo_apply<N, true>(T.Me, T.Mo, re, ro, 1.0, E, O);
          l7_lift<N>(T, s0, s1, v0, g0, vn0, gn0, v1, g1, vn1, gn1, E, O);
          eo_merge<N>(E, O, Tp[STAGE ? 0 : y]);
          eo_apply<N, false>(T.Me, T.Mo, e, o, 1.0, E, O);
          eo_merge<N>(E, O, Vp[STAGE ? 0 : y]);
          if (STAGE) {  // this thread's own rows: no synchronisation needed
#pragma unroll
            for (int x = 0; x < N; ++x) {
              tsp[y * N + x] = Tp[0][x];
              rsp[y * N + x] = Vp[0][x];
            }
          }
        }
      }
      {
        const double sfy = 0.25 * hx * hz, ky = 0.5 * hx * hz * hyi;
        const Side7 s0 = side7(ky0, q[11] + tz, taue, sfy, hyi, q[13], 1.0, ts);
        const Side7 s1 = side7(ky1, q[12] + tz, taue, sfy, hyi, q[14], -1.0, ts);
        const double *h0 = ky0 == 1 ? hyb + par * C::HYN + (jx * N) * N * 2 + 2 * s : zero;
        const double *h1 = ky1 == 1 ? hyb + par * C::HYN + ((TX + jx) * N) * N * 2 + 2 * s : zero;
        double *op = slot + cs * CSTR + s * N2;
        const double *vsp = rbuf + cs * CSTR + s * N2;
#pragma unroll
        for (int x = 0; x < N; ++x) {
          double vc[N], tc[N], e[NE], o[HO], te[NE], to[HO], E[NE], O[HO], g0, g1;
#pragma unroll
          for (int y = 0; y < N; ++y) {
            vc[y] = STAGE ? vsp[y * N + x] : Vp[y][x];
            tc[y] = STAGE ? op[y * N + x] : Tp[y][x];
          }
          eo_split<N>(vc, e, o);
          eo_split<N>(tc, te, to);
          l7_ends<N>(T, e, o, g0, g1);
          const double v0 = vc[0], v1 = vc[N - 1];
          const double vn0 = l7_pick(ky0, __shfl_sync(FULL, v1, ly0, NCT), h0[x * N * 2]);
          const double gn0 = l7_pick(ky0, __shfl_sync(FULL, g1, ly0, NCT), h0[x * N * 2 + 1]);
          const double vn1 = l7_pick(ky1, __shfl_sync(FULL, v0, ly1, NCT), h1[x * N * 2]);
          const double gn1 = l7_pick(ky1, __shfl_sync(FULL, g0, ly1, NCT), h1[x * N * 2 + 1]);
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
    if (tma && EPI == kEpiStore) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // B_b: out complete in the slot
    if (EPI == kEpiCheb) {
      // cell-major points of the layer: a round of THREADS consecutive points
      // per load batch, coalesced in global memory
      constexpr int U = 4;
      const int npts = ex * ey * NP;
      for (int j0 = tid; j0 < npts; j0 += U * C::THREADS) {
        double yv[U], rc[U], dg[U], xv[U], uv[U];
        size_t gi[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int j = j0 + q * C::THREADS;
          if (j < npts) {
            const int cl = j / NP, w = j - cl * NP;
            const int xx = cl % ex, yy = cl / ex;
            gi[q] = ((size_t)x0 + xx + (size_t)g.nx * (y0 + yy) + nxy * iz) * NP + w;
            yv[q] = slot[(xx + TX * yy) * CSTR + w];
            rc[q] = ea.rc[gi[q]];
            dg[q] = ea.diag[gi[q]];
            xv[q] = ea.x[gi[q]];
            uv[q] = u[gi[q]];
          }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int j = j0 + q * C::THREADS;
          if (j < npts) {
            const double r = __dsub_rn(rc[q], yv[q]);
            const double dn = __dadd_rn(__dmul_rn(ea.a, uv[q]), __dmul_rn(ea.b, __ddiv_rn(r, dg[q])));
            ea.rc[gi[q]] = r;
            ea.dnew[gi[q]] = dn;
            ea.x[gi[q]] = __dadd_rn(xv[q], dn);
          }
        }
      }
      if (tma) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();  // the slot is reloaded in a later z phase
    } else if (tma) {
      if (tid < 32) {  // one bulk store per lane of warp 0 (row / cell)
        const int nitem = (N & 1) ? ey : ex * ey;
        for (int i = tid; i < nitem; i += 32) {
          const int xx = (N & 1) ? 0 : i % ex, yy = (N & 1) ? i : i / ex;
          const size_t e0 = (size_t)x0 + xx + (size_t)g.nx * (y0 + yy) + nxy * iz;
          bulk_s2g(out + e0 * NP, slot + (xx + TX * yy) * CSTR,
                   (uint32_t)(((N & 1) ? ex : 1) * NP * sizeof(double)));
        }
      }
    } else {
      for (int i = tid; i < ex * ey * NP; i += C::THREADS) {
        const int cl = i / NP, w = i - cl * NP;
        const int xx = cl % ex, yy = cl / ex;
        out[((size_t)x0 + xx + (size_t)g.nx * (y0 + yy) + nxy * iz) * NP + w] =
            slot[(xx + TX * yy) * CSTR + w];
      }
      __syncthreads();  // the slot is reloaded in the next z phase
    }
  }
  if (tid < 32 && tma && EPI == kEpiStore) bulk_wait_read();
}

}  // namespace dg
