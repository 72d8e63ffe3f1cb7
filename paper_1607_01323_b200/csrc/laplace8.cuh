// SIP Laplace vmult, 3D Cartesian cells: z-marching column kernel with
// half-plane threads (sm_100a, fp64).  Same operator, factorisation, column
// decomposition, TMA ring, halo pipeline and face coefficients as
// laplace7.cuh (reference operators.py:187-238), but every plane of a cell is
// shared by TWO threads, each running about half of the plane's lines:
//   z phase  (ZX plane y = s): z-lines of the columns x in its half,
//   x phase  (XY plane z = s): x-lines of the rows y in its half -> T, V rows
//            written over the W / R rows just read,
//   pair sync (the two halves of plane s),
//   y phase  (XY plane z = s): y-lines of the columns x in its half -> out.
// Twice the threads for the same shared memory and about half the registers
// per thread: the column kernel is latency bound, so occupancy is what pays.
// Layout of the halves:
// * NCT = 16 cells: one warp per plane, lanes 0-15 / 16-31 are the halves
//   (pair sync = __syncwarp); meant for even N (equal halves).
// * NCT = 32 cells: one warp per (plane, half), 2N warps; the role table
//   below places the (N+1)/2-line and N/2-line warps so that the four SM
//   sub-partitions (warp % 4) carry about equal line counts (odd N);
//   pair sync = named barrier 1 + s over the plane's two warps.
#pragma once
#include "laplace7.cuh"

namespace dg {

template <int N, int TX, int TY, int NRING, int HSM = 0>
struct Lap8Cfg : Lap7Cfg<N, TX, TY, NRING> {
  using B = Lap7Cfg<N, TX, TY, NRING>;
  static constexpr int NCT = TX * TY;
  static constexpr int THREADS = (NCT == 16 ? 32 : 64) * N;
  static constexpr int LMAX = (N + 1) / 2;
  static_assert(B::HITEMS <= THREADS, "one halo item per thread");
  // HSM: halo cells staged by cp.async in shared memory ([item][N*N], odd
  // stride) instead of N*N registers per item thread
  static constexpr int OFF_HST = ((B::NDBL + 1) / 2) * 2;
  static constexpr int HSTR = N * N + ((N & 1) ? 0 : 1);
  // HSM = 2: the halo CELLS (2 (TX + TY) per layer) copied whole by the
  // stage-1 warps, lanes on consecutive doubles (coalesced, one address per
  // cell), into [cell][HCS]; per-cell source table [cell]{p0, layer stride, n}
  static constexpr int HCELLS = 2 * (TX + TY);
  static constexpr int HCS = N * N * N + ((N & 1) ? 2 : 1);
  static constexpr int OFF_HTAB = OFF_HST + HCELLS * HCS;
  // per-cell x / y side coefficients for FSD (A = PA hz (tA + tz), B = PB hz,
  // D = PD hz per side, kind folded in; plus the stiffness scales / hz)
  static constexpr int CC2 = 21;
  static constexpr int OFF_CC2 = HSM == 2 ? OFF_HTAB + 3 * HCELLS
                                          : (HSM ? OFF_HST + B::HITEMS * HSTR : B::NDBL);
  // FSD: per-layer z-side data [layer][a0, t0, b0, d0, a1, t1, b1, d1]:
  // A = (ts sf_z) a (txy + t), B = sf_z b, D = sf_z d (kinds folded in)
  static constexpr int OFF_ZS = OFF_CC2 + NCT * CC2;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(OFF_ZS + 8 * B::LCMAX);
  // kEpiDotS: copy of the layer's u ([cell][CSTR] as a ring slot) and the
  // products wint[z] wint[x] of the dual weights
  static constexpr int OFF_UB = ((OFF_ZS + 8 * B::LCMAX + 1) / 2) * 2;
  static constexpr int OFF_WT = OFF_UB + B::LAYER;
  static constexpr size_t SMEM_DOTS = sizeof(double) * (size_t)(OFF_WT + N * N);
  // lane halves run the same lines in lockstep (shuffles inside the line loops)
  static_assert(NCT == 32 || N % 2 == 0, "NCT = 16 halves need even N");
};

// 8-byte asynchronous global -> shared copy
__device__ __forceinline__ void l8_cp_async8(double *dst, const double *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// HMAP (N = 5, NCT = 32): halo stage-1 items / stage-2 rows in 32-wide chunks
// on chosen warps, so that each SM sub-partition (warp % 4) carries about
// the same z-interval work (lines + halo); -1 = none
__device__ __forceinline__ int l8_s1_chunk(int w) {
  constexpr int tab[10] = {-1, 1, -1, -1, -1, -1, 2, 3, 0, -1};
  return tab[w];
}

// NCT = 32: warp -> plane * 2 + half.  Odd N: h = 0 warps (N+1)/2 lines;
// warps {0, 2, 3, 6, 7, ...} take them so that warp % 4 loads stay within one
// line of each other (N = 5: 7 / 6 / 6 / 6).
template <int N>
__device__ __forceinline__ int l8_role(int w) {
  if (N == 5) {
    constexpr int tab[10] = {0, 1, 2, 4, 3, 5, 6, 8, 7, 9};  // warp -> s * 2 + h
    return tab[w];
  }
  return w;
}

// EPI: kEpiStore (out by TMA bulk stores) or a CG / Chebyshev epilogue
// (laplace.cuh epi_store) applied cooperatively to each finished layer of
// the tile; kEpiDot leaves one partial-sum triple per CTA in ea.partials.
template <int N, int TX, int TY, int NRING, int MINB, int EPI = kEpiStore, int HSM = 0, int HMAP = 0,
          int FSD = 0, int UBC = 0>
__global__ void __launch_bounds__(Lap8Cfg<N, TX, TY, NRING>::THREADS, MINB)
laplace8_kernel(const double *__restrict__ u, double *__restrict__ out, const Geo g,
                const __grid_constant__ LapTab<N> T, const double ts, const int part,
                const int zlo, const int zhi, const int lc, const int ntx, const int nty,
                const EpiArgs ea = EpiArgs{}) {
  using C = Lap8Cfg<N, TX, TY, NRING, HSM>;
  static_assert(HMAP == 0 || (N == 5 && TX * TY == 32), "HMAP tables are for N = 5, 32-cell tiles");
  constexpr int NCT = C::NCT, NP = C::NP, CSTR = C::CSTR, H = N / 2, NE = (N + 1) / 2;
  constexpr int HO = H > 0 ? H : 1;
  constexpr int N2 = N * N;
  constexpr int LMAX = C::LMAX;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double smem[];
  double *const ring = smem;
  double *const rbuf = smem + C::OFF_R;
  double *const hxb = smem + C::OFF_HX;
  double *const hyb = smem + C::OFF_HY;
  double *const cc = smem + C::OFF_CC;
  uint64_t *const bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
  const double *const zero = smem + C::OFF_ZERO;
  unsigned long long *const htab = reinterpret_cast<unsigned long long *>(smem + C::OFF_HTAB);

  // ---- unit: tile (tx, ty) x z-chunk -------------------------------------
  int unit = blockIdx.x;
  const int tix = unit % ntx;
  unit /= ntx;
  const int tiy = unit % nty;
  const int chunk = unit / nty;
  const int x0 = tix * TX, y0 = tiy * TY;
  const int ex = min(TX, g.nx - x0), ey = min(TY, g.ny - y0);
  const int z0 = zlo + chunk * lc, z1 = min(zhi, z0 + lc);
  bool skip = z0 >= z1;
  if (part != 0) {
    const bool touches = (g.mode[0] == kGhost && x0 == 0) || (g.mode[1] == kGhost && x0 + ex == g.nx);
    if ((part == 1 && touches) || (part == 2 && !touches)) skip = true;
  }
  if (skip) {
    if ((EPI == kEpiDot || EPI == kEpiDotS) && threadIdx.x < 3) ea.partials[(size_t)blockIdx.x * 4 + threadIdx.x] = 0.0;
    return;
  }
  double eacc[3] = {0.0, 0.0, 0.0};  // kEpiDot partial sums of this CTA
  const int nlay = z1 - z0;
  const size_t nxy = (size_t)g.nx * g.ny;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int c, s, h;
  if (NCT == 16) {
    c = lane & 15;
    h = lane >> 4;
    s = warp;
  } else {
    const int role = l8_role<N>(warp);
    c = lane;
    s = role >> 1;
    h = role & 1;
  }
  const int l0 = h ? NE : 0;       // first line of this half
  const int nl = h ? N - NE : NE;  // lines of this half (warp-uniform for NCT = 32)
  const int jx = c % TX, jy = c / TX;
  const int ix = x0 + min(jx, ex - 1), iy = y0 + min(jy, ey - 1);  // clamped (inactive lanes)
  // pair sync of the two halves of plane s
  auto pair_sync = [&]() {
    if (NCT == 16) __syncwarp();
    else asm volatile("bar.sync %0, 64;" ::"r"(1 + s) : "memory");
  };

  // ---- per-column constants and neighbour kinds --------------------------
  int kx0, kx1, ky0, ky1, lx0 = 0, lx1 = 0, ly0 = 0, ly1 = 0;
  {
    int nb = 0;
    kx0 = kind7<0>(g, 0, ix, g.nx, x0, ex, nb);
    lx0 = nb + TX * jy;
    kx1 = kind7<1>(g, 0, ix, g.nx, x0, ex, nb);
    lx1 = nb + TX * jy;
    ky0 = kind7<0>(g, 1, iy, g.ny, y0, ey, nb);
    ly0 = jx + TX * nb;
    ky1 = kind7<1>(g, 1, iy, g.ny, y0, ey, nb);
    ly1 = jx + TX * nb;
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
    if (FSD) {  // side coefficients of this cell with its kinds folded in
      double *f = smem + C::OFF_CC2 + c * C::CC2;
      f[0] = 0.5 * hy * hxi;  // kx / hz
      f[1] = 0.5 * hx * hyi;  // ky / hz
      auto put = [&](double *o, int kind, double tmx, double sf, double hid, double hin, double sg) {
        o[0] = o[1] = o[2] = o[3] = 0.0;
        if (kind <= 1) {
          o[0] = ts * sf;
          o[1] = tmx;
          o[2] = sg * sf * hid;
          o[3] = sg * sf * hin;
        } else if (kind == kBndNeumann) {
          o[0] = ts * 2.0 * sf;
          o[1] = tx + ty;
          o[2] = 2.0 * sg * sf * hid;
        }
      };
      put(f + 2, kx0, q[5], 0.25 * hy, hxi, q[7], 1.0);
      put(f + 6, kx1, q[6], 0.25 * hy, hxi, q[8], -1.0);
      put(f + 10, ky0, q[11], 0.25 * hx, hyi, q[13], 1.0);
      put(f + 14, ky1, q[12], 0.25 * hx, hyi, q[14], -1.0);
    }
  }
  for (int i = tid; i < 2 * N * N; i += C::THREADS) smem[C::OFF_ZERO + i] = 0.0;
  double *const ubuf = smem + C::OFF_UB;
  if (EPI == kEpiDotS && tid == 0) {
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) smem[C::OFF_WT + a * N + b] = ea.wint[a] * ea.wint[b];
  }
  const bool act = jx < ex && jy < ey;  // kEpiDotS: lanes of cells outside the mesh add nothing
  double *const zd = smem + C::OFF_ZD;
  for (int i = tid; i < 4 * (nlay + 2); i += C::THREADS) zd[i] = g.ax[2][4 * (z0 - 1) + i];
  double *const zs = smem + C::OFF_ZS;
  if (FSD)
    for (int L = tid; L < nlay; L += C::THREADS) {  // z sides of layer z0 + L
      const int iz = z0 + L;
      const double *a = g.ax[2] + 4 * iz;
      const double tz = a[2], hzi = a[1];
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) {
        const double *an = a + (sd ? 4 : -4);
        const bool edge = sd ? iz == g.nz - 1 : iz == 0;
        const int m = g.mode[4 + sd];
        const int kind = edge ? (m == kWrap ? 0 : m) : 0;
        const double sg = sd ? -1.0 : 1.0;
        double *o = zs + 8 * L + 4 * sd;
        o[0] = o[1] = o[2] = o[3] = 0.0;
        if (kind <= 1) {
          o[0] = 1.0;
          o[1] = tz > an[2] ? tz : an[2];
          o[2] = sg * hzi;
          o[3] = sg * an[1];
        } else if (kind == kBndNeumann) {
          o[0] = 2.0;
          o[1] = tz;
          o[2] = 2.0 * sg * hzi;
        }
      }
    }

  // ---- ring ----------------------------------------------------------------
  auto layer_of = [&](int r) -> int {
    const int z = z0 + r - 1;
    if (z < 0) return g.mode[4] == kWrap ? g.nz - 1 : -1;
    if (z >= g.nz) return g.mode[5] == kWrap ? 0 : -1;
    return z;
  };
  const bool rows_ok = (N & 1) ? (!(g.nx & 1) && !(ex & 1)) : true;
  const bool tma = rows_ok && !(reinterpret_cast<uintptr_t>(u) & 15) &&
                   !(reinterpret_cast<uintptr_t>(out) & 15);
  if (tid == 0)
    for (int i = 0; i < NRING; ++i) mbar_init(&bar[i], 1);
  if (HSM == 2 && tid < C::HCELLS) {  // halo cell sources of this tile (layer 0 + layer stride)
    const double *p0 = nullptr;
    size_t lst = 0;
    int n = 0;
    if (tid < 2 * TY) {  // x neighbours (side, row)
      const int side = tid / TY, row = tid % TY, yy = y0 + row;
      int nc = side ? x0 + ex : x0 - 1;
      bool ok = row < ey;
      if (ok && (nc < 0 || nc >= g.nx)) {
        const int m = g.mode[side];
        if (m == kWrap) nc = side ? 0 : g.nx - 1;
        else if (m == kGhost) {
          const int cs = g.ghost_traces ? 2 * N2 : NP;
          p0 = g.ghost[side] + (size_t)yy * cs;
          lst = (size_t)g.ny * cs;
          n = cs;
          ok = false;
        } else ok = false;
      }
      if (ok && !(nc >= x0 && nc < x0 + ex)) {
        p0 = u + ((size_t)nc + (size_t)g.nx * yy) * NP;
        lst = nxy * NP;
        n = NP;
      }
    } else {  // y neighbours (side, column)
      const int c8 = tid - 2 * TY, side = c8 / TX, col = c8 % TX, xx = x0 + col;
      int nc = side ? y0 + ey : y0 - 1;
      bool ok = col < ex;
      if (ok && (nc < 0 || nc >= g.ny)) {
        if (g.mode[2 + side] == kWrap) nc = side ? 0 : g.ny - 1;
        else ok = false;
      }
      if (ok && !(nc >= y0 && nc < y0 + ey)) {
        p0 = u + ((size_t)xx + (size_t)g.nx * nc) * NP;
        lst = nxy * NP;
        n = NP;
      }
    }
    htab[3 * tid] = reinterpret_cast<unsigned long long>(p0);
    htab[3 * tid + 1] = lst;
    htab[3 * tid + 2] = n;
  }
  __syncthreads();
  auto issue = [&](int r) {
    if (HSM == 2 && tma && tid >= 32) return;  // only warp 0 takes part with TMA
    if (r > nlay + 1) return;
    const int lay = layer_of(r);
    uint64_t *b = &bar[r % NRING];
    if (lay < 0) {
      if (tma && tid == 0) mbar_arrive(b);
      return;
    }
    double *dst = ring + (r % NRING) * C::LAYER;
    if (tma) {
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
    } else {
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

  // ---- halo (as laplace7.cuh) ------------------------------------------------
  static_assert(HSM != 2 || (HMAP && N == 5 && TX * TY == 32), "HSM 2: 6 cells of 5 items per warp");
  const int hch = HMAP ? l8_s1_chunk(warp) : -1;  // stage-1 chunk of this warp
  int hit = tid;
  if (HMAP) hit = hch < 0 ? C::THREADS : (HSM == 2 ? (lane < 30 ? hch * 30 + lane : C::THREADS)
                                                    : hch * 32 + lane);
  double *const hcell = smem + C::OFF_HST;  // HSM 2: staged halo cells
  double *const hst = smem + C::OFF_HST + (size_t)min(hit, C::HITEMS - 1) * C::HSTR;
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
      if (nc >= x0 && nc < x0 + ex) return nullptr;
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
  constexpr int HR = HSM ? 1 : N;
  double hreg[HR][N];
  const double *hsrc = nullptr;
  const int hmy = hit < C::HITEMS ? hit / N : 0;  // HSM 2: this item's cell
  auto halo_load = [&](int lay) {
    if (HSM == 2) {
      hsrc = nullptr;
      if (hch < 0 || lay < 0) return;
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const int cid = hch * 6 + j;
        if (cid >= C::HCELLS) break;
        const int n = (int)htab[3 * cid + 2];
        if (n == 0) continue;
        const double *src = reinterpret_cast<const double *>(htab[3 * cid]) + (size_t)lay * htab[3 * cid + 1];
        double *dst = hcell + cid * C::HCS;
#pragma unroll
        for (int m = 0; m < (NP + 31) / 32; ++m)
          if (lane + 32 * m < n) l8_cp_async8(dst + lane + 32 * m, src + lane + 32 * m);
      }
      if (hit < C::HITEMS && htab[3 * hmy + 2] != 0) {
        hsrc = hcell + hmy * C::HCS;  // flag + staged cell
        htrace = htab[3 * hmy + 2] == (unsigned long long)(2 * N2);
      }
      return;
    }
    hsrc = halo_src(lay);
    if (!hsrc) return;
    if (htrace) {  // [z][y][v|g] of the facing end, raw (M_z below)
#pragma unroll
      for (int z = 0; z < N; ++z) {
        if (HSM) {
          l8_cp_async8(hst + 2 * z, hsrc + (z * N + hpos) * 2);
          l8_cp_async8(hst + 2 * z + 1, hsrc + (z * N + hpos) * 2 + 1);
        } else {
          hreg[z % HR][0] = __ldg(hsrc + (z * N + hpos) * 2);
          hreg[z % HR][1] = __ldg(hsrc + (z * N + hpos) * 2 + 1);
        }
      }
      return;
    }
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const double *src = hsrc + z * N2 + (hx_item ? hpos * N + q : q * N + hpos);
        if (HSM) l8_cp_async8(hst + z * N + q, src);
        else hreg[z % HR][q] = __ldg(src);
      }
  };
  auto halo_stage1 = [&](int par) {
    if (HSM == 2 && hch >= 0) {  // the warp's cells, copied by all its lanes
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncwarp();
    }
    if (!hsrc) return;
    if (HSM == 1) asm volatile("cp.async.wait_all;" ::: "memory");
    double v[N], gg[N], mv[N], mg[N];
#pragma unroll
    for (int z = 0; z < N; ++z) {
      double e[NE], o[HO], g0, g1, hr[N];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        if (HSM == 2)
          hr[q] = (htrace && q >= 2) ? 0.0
                  : hcell[hmy * C::HCS +
                          (htrace ? (z * N + hpos) * 2 + q : z * N2 + (hx_item ? hpos * N + q : q * N + hpos))];
        else if (HSM) hr[q] = (htrace && q >= 2) ? 0.0 : hst[htrace ? 2 * z + q : z * N + q];
        else hr[q] = hreg[z % HR][q];
      }
      eo_split<N>(hr, e, o);
      l7_ends<N>(T, e, o, g0, g1);
      v[z] = htrace ? hr[0] : (hside ? hr[0] : hr[N - 1]);
      gg[z] = htrace ? hr[1] : (hside ? g0 : g1);
    }
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
  // HMAP: stage-2 row chunks on warps 5, 9, 2, 3, 2 (see l8_s1_chunk)
  // HSM 2: this thread's stage-2 rows (at most 2 with HMAP) resolved once
  int s2off[2] = {-1, -1};
  if (HSM == 2) {
    const int a = warp == 5 ? 0 : warp == 9 ? 1 : warp == 2 ? 2 : warp == 3 ? 3 : -1;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int i = a < 0 ? C::HROWS : a * 32 + lane + 64 * rr;
      if (i < C::HROWS && (rr == 0 || warp == 2)) {
        const int vg = i & 1, rz = i >> 1;
        const int z = rz % N, sj = rz / N;
        if ((sj % TX) < ex) s2off[rr] = sj * N * N * 2 + z * 2 + vg;
      }
    }
  }
  auto halo_stage2 = [&](int par) {
    if (HSM == 2) {
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        if (s2off[rr] < 0) continue;
        double *row = hyb + par * C::HYN + s2off[rr];
        double v[N], y[N];
#pragma unroll
        for (int x = 0; x < N; ++x) v[x] = row[x * N * 2];
        l7_mass<N>(T, v, y);
#pragma unroll
        for (int x = 0; x < N; ++x) row[x * N * 2] = y[x];
      }
      return;
    }
    int i0 = tid, i1 = C::HROWS, di = C::THREADS;
    if (HMAP) {
      const int a = warp == 5 ? 0 : warp == 9 ? 1 : warp == 2 ? 2 : warp == 3 ? 3 : -1;
      i0 = a < 0 ? C::HROWS : a * 32 + lane;
      di = 64;  // warp 2 also takes chunk 4
      if (warp != 2) i1 = min(i1, i0 + 1);
    }
    for (int i = i0; i < i1; i += di) {
      const int vg = i & 1, rz = i >> 1;
      const int z = rz % N, sj = rz / N;
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
  double ztv[LMAX], ztg[LMAX];  // raw top functionals of the layer below, own columns
#pragma unroll
  for (int k = 0; k < LMAX; ++k) {
    ztv[k] = 0.0;
    ztg[k] = 0.0;
  }
  halo_load(layer_of(1));
  if (!tma) __syncthreads();
  if (layer_of(0) >= 0) {
    wait_slot(0);
    const double *p = ring + c * CSTR + s * N + l0;
#pragma unroll
    for (int k = 0; k < LMAX; ++k) {
      if (k < nl) {
        double w[N], e[NE], o[HO], g0, g1;
#pragma unroll
        for (int z = 0; z < N; ++z) w[z] = p[z * N2 + k];
        eo_split<N>(w, e, o);
        l7_ends<N>(T, e, o, g0, g1);
        ztv[k] = w[N - 1];
        ztg[k] = g1;
      }
    }
  }
  halo_stage1(0);
  __syncthreads();

  // ---- march ---------------------------------------------------------------------------
  for (int p = 0; p < nlay; ++p) {
    const int r = p + 1;
    const int iz = z0 + p;
    const int par = p & 1;
    double *const slot = ring + (r % NRING) * C::LAYER;
    const double *az = zd + 4 * (p + 1);
    const double hz = az[0], hzi = az[1], tz = az[2];

    auto refill = [&]() {
      if (tid < 32 && tma) bulk_wait_read();
      issue(r + NRING - 1);
    };
    if (NRING == 2) {
      refill();
      if (!tma) __syncthreads();
    }
    wait_slot(r);
    const int lay_up = layer_of(r + 1);
    wait_slot(r + 1);
    const bool more = p + 1 < nlay;
    halo_load(more ? iz + 1 : -1);
    halo_stage2(par);
    if (EPI == kEpiCheb && (N & 1)) {  // this layer's epilogue operands -> L2
      const int R = ex * NP;
      for (int i = tid * 16; i < (UBC ? 3 : 4) * ey * R; i += 16 * C::THREADS) {  // 128 B lines
        const int v = i / (ey * R), rem = i - v * (ey * R), yy = rem / R, j = rem - yy * R;
        const size_t gi = ((size_t)x0 + (size_t)g.nx * (y0 + yy) + nxy * iz) * NP + j;
        const double *p = v == 0 ? ea.rc : (v == 1 ? ea.diag : (v == 2 ? ea.x : u));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p + gi));
      }
    }
    // ================= z phase: columns x in this half of plane y = s =================
    {
      const double *q = cc + c * C::CCS;
      const double sfz = q[0], kz = q[1] * hzi, txy = q[2];
      const double taue = txy + tz;
      const int kz0 = iz == 0 ? (g.mode[4] == kWrap ? 0 : g.mode[4]) : 0;
      const int kz1 = iz == g.nz - 1 ? (g.mode[5] == kWrap ? 0 : g.mode[5]) : 0;
      // tau of the z faces: max of the two cells' z parts (plain compare: no NaN
      // fix-up sequence as in fmax)
      const double tzl = az[-4 + 2], tzu = az[4 + 2];
      const double *zq = zs + 8 * p;
      const double tsf = ts * sfz;
      const Side7 s0 = FSD ? Side7{tsf * zq[0] * (txy + zq[1]), sfz * zq[2], sfz * zq[3]}
                           : side7(kz0, txy + (tz > tzl ? tz : tzl), taue, sfz, hzi, az[-4 + 1], 1.0, ts);
      const Side7 s1 = FSD ? Side7{tsf * zq[4] * (txy + zq[5]), sfz * zq[6], sfz * zq[7]}
                           : side7(kz1, txy + (tz > tzu ? tz : tzu), taue, sfz, hzi, az[4 + 1], -1.0, ts);
      double *up = slot + c * CSTR + s * N + l0;
      double *rp = rbuf + c * CSTR + s * N + l0;
      const double *lp = ring + ((r + 1) % NRING) * C::LAYER + c * CSTR + s * N + l0;
      const bool la_ok = lay_up >= 0;
#pragma unroll
      for (int k = 0; k < LMAX; ++k) {
        if (k < nl) {
          double w[N], e[NE], o[HO], E[NE], O[HO], g0, g1;
#pragma unroll
          for (int z = 0; z < N; ++z) w[z] = up[z * N2 + k];
          if (EPI == kEpiDotS || (EPI == kEpiCheb && UBC)) {  // u of this layer stays readable
            double *ub = ubuf + c * CSTR + s * N + l0;
#pragma unroll
            for (int z = 0; z < N; ++z) ub[z * N2 + k] = w[z];
          }
          double la0 = lp[k], lg = T.dL[0] * la0;
#pragma unroll
          for (int z = 1; z < N; ++z) lg += T.dL[z] * lp[z * N2 + k];
          const double vn1 = la_ok ? la0 : 0.0, gn1 = la_ok ? lg : 0.0;
          eo_split<N>(w, e, o);
          l7_ends<N>(T, e, o, g0, g1);
          const double vn0 = ztv[k], gn0 = ztg[k];
          ztv[k] = w[N - 1];
          ztg[k] = g1;
          eo_apply<N, false>(T.Ke, T.Ko, e, o, kz, E, O);
          l7_lift<N>(T, s0, s1, w[0], g0, vn0, gn0, w[N - 1], g1, vn1, gn1, E, O);
          double y[N];
          eo_merge<N>(E, O, y);
#pragma unroll
          for (int z = 0; z < N; ++z) rp[z * N2 + k] = y[z];
          eo_apply<N, false>(T.Me, T.Mo, e, o, 1.0, E, O);
          eo_merge<N>(E, O, y);
#pragma unroll
          for (int z = 0; z < N; ++z) up[z * N2 + k] = y[z];
        }
      }
    }
    if (NRING >= 3) refill();
    halo_stage1(par ^ 1);
    __syncthreads();  // B_a: W, R complete; halo of this layer complete

    // ================= x phase: rows y in this half of plane z = s =================
    const double *q = cc + c * C::CCS;
    const double hy = q[3], hxi = q[4], hx = q[9], hyi = q[10];
    const double taue = q[2] + tz;
    double *const wp = slot + c * CSTR + s * N2;  // W rows -> T rows -> out
    double *const rp = rbuf + c * CSTR + s * N2;  // R rows -> V rows
    {
      const double *f = smem + C::OFF_CC2 + c * C::CC2;
      const double sfx = 0.25 * hy * hz;
      const double kx = FSD ? f[0] * hz : 0.5 * hy * hz * hxi;
      const Side7 s0 = FSD ? Side7{f[2] * hz * (f[3] + tz), f[4] * hz, f[5] * hz}
                           : side7(kx0, q[5] + tz, taue, sfx, hxi, q[7], 1.0, ts);
      const Side7 s1 = FSD ? Side7{f[6] * hz * (f[7] + tz), f[8] * hz, f[9] * hz}
                           : side7(kx1, q[6] + tz, taue, sfx, hxi, q[8], -1.0, ts);
      const double *h0 = kx0 == 1 ? hxb + par * C::HXN + (jy * N) * N * 2 + 2 * s : zero;
      const double *h1 = kx1 == 1 ? hxb + par * C::HXN + ((TY + jy) * N) * N * 2 + 2 * s : zero;
#pragma unroll
      for (int k = 0; k < LMAX; ++k) {
        if (k < nl) {
          const int y = l0 + k;
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
          double yt[N];
          eo_merge<N>(E, O, yt);
          eo_apply<N, false>(T.Me, T.Mo, e, o, 1.0, E, O);
          double yv[N];
          eo_merge<N>(E, O, yv);
#pragma unroll
          for (int x = 0; x < N; ++x) {
            wp[y * N + x] = yt[x];
            rp[y * N + x] = yv[x];
          }
        }
      }
    }
    pair_sync();
    // ================= y phase: columns x in this half of plane z = s =================
    {
      const double *f = smem + C::OFF_CC2 + c * C::CC2;
      const double sfy = 0.25 * hx * hz;
      const double ky = FSD ? f[1] * hz : 0.5 * hx * hz * hyi;
      const Side7 s0 = FSD ? Side7{f[10] * hz * (f[11] + tz), f[12] * hz, f[13] * hz}
                           : side7(ky0, q[11] + tz, taue, sfy, hyi, q[13], 1.0, ts);
      const Side7 s1 = FSD ? Side7{f[14] * hz * (f[15] + tz), f[16] * hz, f[17] * hz}
                           : side7(ky1, q[12] + tz, taue, sfy, hyi, q[14], -1.0, ts);
      const double *h0 = ky0 == 1 ? hyb + par * C::HYN + (jx * N) * N * 2 + 2 * s : zero;
      const double *h1 = ky1 == 1 ? hyb + par * C::HYN + ((TX + jx) * N) * N * 2 + 2 * s : zero;
#pragma unroll
      for (int k = 0; k < LMAX; ++k) {
        if (k < nl) {
          const int x = l0 + k;
          double vc[N], tc[N], e[NE], o[HO], te[NE], to[HO], E[NE], O[HO], g0, g1;
#pragma unroll
          for (int y = 0; y < N; ++y) {
            vc[y] = rp[y * N + x];
            tc[y] = wp[y * N + x];
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
          for (int yy = 0; yy < N; ++yy) wp[yy * N + x] = yv[yy];
          if (EPI == kEpiDotS) {  // u.Lu, sum(Lu), u.w of this line
            const double *ub = ubuf + c * CSTR + s * N2 + x;
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
            for (int yy = 0; yy < N; ++yy) {
              const double pu = ub[yy * N];
              t0 += pu * yv[yy];
              t1 += yv[yy];
              t2 += pu * ea.wint[yy];
            }
            if (act) {
              eacc[0] += t0;
              eacc[1] += t1;
              eacc[2] += t2 * (smem[C::OFF_WT + s * N + x] * (0.5 * q[0] * hz));
            }
          }
        }
      }
    }
    if (tma && (EPI == kEpiStore || EPI == kEpiDotS)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // B_b: out complete in the slot
    if (EPI == kEpiCheb && (N & 1)) {
      // Chebyshev epilogue, odd N (a tile row of cells is one contiguous run
      // in global and shared memory): per row, each thread loads the operands
      // of up to 4 points (prefetched into L2 during the z phase) before any
      // arithmetic or store, so the row's loads are in flight together
      constexpr int U = 4;
      const int R = ex * NP;
      for (int yy = 0; yy < ey; ++yy) {
        const size_t rb = ((size_t)x0 + (size_t)g.nx * (y0 + yy) + nxy * iz) * NP;
        const double *sl = slot + TX * yy * CSTR;
        const double *ul = ubuf + TX * yy * CSTR;  // UBC: d of this layer from shared memory
        for (int j0 = tid; j0 < R; j0 += U * C::THREADS) {
          double yv[U], rc[U], dg[U], xv[U], uv[U];
#pragma unroll
          for (int q = 0; q < U; ++q) {
            const int j = j0 + q * C::THREADS;
            if (j < R) {
              yv[q] = sl[j];
              rc[q] = ea.rc[rb + j];
              dg[q] = ea.diag[rb + j];
              xv[q] = ea.x[rb + j];
              uv[q] = UBC ? ul[j] : u[rb + j];
            }
          }
#pragma unroll
          for (int q = 0; q < U; ++q) {
            const int j = j0 + q * C::THREADS;
            if (j < R) {
              const double r = __dsub_rn(rc[q], yv[q]);
              const double dn = __dadd_rn(__dmul_rn(ea.a, uv[q]), __dmul_rn(ea.b, __ddiv_rn(r, dg[q])));
              ea.rc[rb + j] = r;
              ea.dnew[rb + j] = dn;
              ea.x[rb + j] = __dadd_rn(xv[q], dn);
            }
          }
        }
      }
      __syncthreads();  // the slot is refilled by a later z phase
    } else if (EPI != kEpiStore && EPI != kEpiDotS) {
      // epilogue on this layer's cells: out / Chebyshev vectors / partial sums
      const double hzl = hz;
      for (int i = tid; i < ex * ey * NP; i += C::THREADS) {
        const int cl = i / NP, w = i - cl * NP;
        const int xx = cl % ex, yy = cl / ex;
        const size_t gi = ((size_t)x0 + xx + (size_t)g.nx * (y0 + yy) + nxy * iz) * NP + w;
        double wq = 0.0;
        if (EPI == kEpiDot) {
          const int qx = w % N, qy = (w / N) % N, qz = w / N2;
          wq = 0.5 * g.ax[0][4 * (x0 + xx)] * ea.wint[qx] * 0.5 * g.ax[1][4 * (y0 + yy)] *
               ea.wint[qy] * 0.5 * hzl * ea.wint[qz];
        }
        epi_store<EPI, 3, N>(u, out, ea, gi, slot[(xx + TX * yy) * CSTR + w], wq, eacc);
      }
      __syncthreads();  // the slot is refilled by a later z phase
    } else if (tma) {
      if (tid < 32) {
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
      __syncthreads();
    }
  }
  if (EPI == kEpiDot || EPI == kEpiDotS) epi_reduce(eacc, rbuf, ea, blockIdx.x);
  if (tid < 32 && tma && (EPI == kEpiStore || EPI == kEpiDotS)) bulk_wait_read();
}

}  // namespace dg
