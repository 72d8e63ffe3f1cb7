// Persistent, software-pipelined form of the Cartesian convective kernel
// (same algebra, rule and phase order as vconv.cuh; reference
// operators.py:533-604).  Differences, all measured on C3 (32^3 Q5):
// * one CTA per SM slot loops over cells (e = blockIdx.x + k gridDim.x) and
//   over the history levels of each cell; the own-cell nodal values of the
//   NEXT (cell, level) item are fetched by TMA bulk copies into the second of
//   two buffers while the current item is computed, and the neighbours' end
//   layers of the next item by cp.async into a second shared buffer -- the
//   one-CTA-per-cell kernel stalled on exactly these loads at the start of
//   every cell;
// * lines that one thread writes (reads) contiguously and its neighbours
//   read (write) across use an odd pitch NQ + 1, so the line-per-thread
//   phases are free of the 8-way shared-memory bank conflicts of pitch NQ;
// * the 1D operators in even-odd form (vconv.cuh EoTab).
#pragma once
#include "tma.cuh"
#include "vconv.cuh"

namespace dg {

template <int N, int NQ, int TV = 0, int MB = 0>
struct Cv2Cfg {
  static constexpr int NP = N * N * N, QP = NQ * NQ * NQ, FQ = NQ * NQ, FN = N * N;
  static constexpr int T = TV ? TV : (QP <= 64 ? 64 : 128);
  static constexpr int MINB = MB ? MB : (N >= 5 ? 3 : 4);
  static constexpr int P1 = NQ + 1;  // odd pitch of NQ-long lines
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  static constexpr int WR = (NQ + 1) & ~1;        // Gauss weights (keeps the TMA buffers 16 B aligned)
  static constexpr int SU0 = WR, SU1 = SU0 + 3 * NP;  // own nodal cell, two buffers
  static constexpr int OUT = SU1 + 3 * NP;        // accumulator
  static constexpr int NB = OUT + 3 * NP;         // neighbour end layers [2][side][c][sl][fa]
  static constexpr int RA = NB + 36 * FN;
  // RA: x1 (3 N N P1) | u_q (3 QP) | A, B (6 N N P1) | traces (36 FQ) |
  //     lift 1 (18 NQ N) | body force (3 N N P1)
  static constexpr int SZA = mx(mx(3 * QP, 6 * N * N * P1), 36 * FQ);
  static constexpr int RB = RA + SZA;
  // RB: x2 (3 N NQ NQ) | Z (9 N NQ NQ) | fast sweep (36 N P1) | LF values
  //     (18 NQ P1) | body force (3 N NQ NQ)
  static constexpr int SZB = mx(9 * N * FQ, mx(36 * N * P1, 18 * NQ * P1));
  static constexpr int NDBL = RB + SZB;
  static constexpr size_t SMEM = sizeof(double) * NDBL;
  static_assert((SU0 % 2) == 0 && (NP % 2) == 0, "TMA destinations 16 B aligned");
};

// side kind (0 interior / periodic, kBndNone, kBndNeumann) and the neighbour
// cell across it, from the cell coordinates
__device__ __forceinline__ int cv2_side(const Geo &g, int ix, int iy, int iz, int side,
                                        int64_t &nbr) {
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
  nbr = cx + (int64_t)g.nx * (cy + (int64_t)g.ny * cz);
  return k;
}

// 8-byte asynchronous global -> shared copy (zero fill when !valid)
__device__ __forceinline__ void cp_async8(double *dst, const double *src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}

// TMA bulk store of a shared-memory block (16-byte aligned, size a multiple
// of 16) and the wait until the engine has read it
__device__ __forceinline__ void cv2_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cv2_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <int V>
struct Cv2Job {  // compile-time job index of the G_ab phase
  static constexpr int value = V;
};

__device__ __forceinline__ void cv2_xyz(const Geo &g, int64_t e, int &ix, int &iy, int &iz) {
  const unsigned ei = (unsigned)e, nx = (unsigned)g.nx, ny = (unsigned)g.ny;
  const unsigned q = ei / nx;
  ix = (int)(ei - q * nx);
  iz = (int)(q / ny);
  iy = (int)(q - (unsigned)iz * ny);
}

template <int N, int NQ, int TV = 0, int MB = 0>
__global__ void __launch_bounds__(Cv2Cfg<N, NQ, TV, MB>::T, Cv2Cfg<N, NQ, TV, MB>::MINB)
vconv2_kernel(double *__restrict__ out, const Geo g, const __grid_constant__ QuadTab<N, NQ> tab,
              const __grid_constant__ CvEo<N, NQ> eo, const VecParams prm, const int64_t ncells) {
  using C = Cv2Cfg<N, NQ, TV, MB>;
  constexpr int NP = C::NP, QP = C::QP, FQ = C::FQ, FN = C::FN, T = C::T, P1 = C::P1;
  constexpr int NQ2 = NQ * NQ;
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ const double *p_hist[kMaxHist], *p_gh[kMaxHist][6];
  __shared__ double p_beta[kMaxHist];
  // side kinds / neighbour cells of the items two apart share a slot: slot
  // (w & 1) holds item w's, written by threads 0-5 during item w - 2 (w >= 2)
  __shared__ int skind[2][6];
  __shared__ int64_t snbr[2][6];
  double *W = sm;
  double *so = sm + C::OUT, *ra = sm + C::RA, *rb = sm + C::RB;
  const int tid = threadIdx.x;
  const int nh = prm.n_hist;
  const int64_t ncta = (ncells - blockIdx.x + gridDim.x - 1) / gridDim.x;  // cells of this CTA
  const int64_t nitems = ncta * nh;
  if (nitems <= 0) return;

  for (int i = tid; i < NQ; i += T) W[i] = tab.w[i];
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < kMaxHist; ++j) {
      p_hist[j] = prm.hist[j];
      p_beta[j] = prm.beta[j];
#pragma unroll
      for (int q = 0; q < 6; ++q) p_gh[j][q] = prm.gh[j][q];
    }
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  __syncthreads();

  // item w = k nh + lev: cell blockIdx.x + k gridDim.x, history level lev
  // items per CTA fit 32 bits: 32-bit division by nh (a 64-bit one cost ~100
  // instructions of warp 0 per item)
  auto item_cell = [&](int64_t w) {
    return (int64_t)blockIdx.x + (int64_t)((unsigned)w / (unsigned)nh) * gridDim.x;
  };
  auto side_info = [&](int64_t w) {  // threads 0-5
    if (tid < 6) {
      int ix, iy, iz;
      cv2_xyz(g, item_cell(w), ix, iy, iz);
      int64_t nb;
      skind[w & 1][tid] = cv2_side(g, ix, iy, iz, tid, nb);
      snbr[w & 1][tid] = nb * NP;  // element offset of the neighbour cell
    }
  };
  // TMA of item w's own cell into buffer w & 1 (one thread)
  auto issue_own = [&](int64_t w) {
    const int64_t e = item_cell(w);
    const double *src = p_hist[(int)((unsigned)w % (unsigned)nh)];  // one thread, once per item
    double *dst = sm + ((w & 1) ? C::SU1 : C::SU0);
    uint64_t *bar = &bars[w & 1];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, (uint32_t)(3 * NP * sizeof(double)));
#pragma unroll
    for (int c = 0; c < 3; ++c)
      bulk_g2s(dst + c * NP, src + ((int64_t)c * ncells + e) * NP, (uint32_t)(NP * sizeof(double)), bar);
  };
  // neighbour end layers of item w -> snb buffer w & 1, by cp.async (this
  // thread's copies; waited for before the barrier that ends item w - 1)
  auto load_nbr = [&](int64_t w, int lv) {
    const double *src = p_hist[lv];
    const int sl = (int)(w & 1);
    double *snb = sm + C::NB + sl * 18 * FN;
    if (3 * FN <= T) {  // thread -> (component, face node); one side per pass
      const int nc_f = tid % FN, nc_c = tid / FN, nc_fs = nc_f / N, nc_fa = nc_f % N;
      if (nc_c < 3) {
        const double *srcc = src + (int64_t)nc_c * ncells * NP;  // this thread's component
#pragma unroll
        for (int side = 0; side < 6; ++side) {
          const bool in = skind[sl][side] == 0;
          const double *p = in ? srcc + snbr[sl][side] + cv_end_node<N>(side >> 1, (side & 1) ^ 1, nc_fs, nc_fa)
                               : src;
          cp_async8(snb + (side * 3 + nc_c) * FN + nc_f, p, in);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      return;
    }
    for (int i = tid; i < 18 * FN; i += T) {
      const int side = i / (3 * FN), c = (i / FN) % 3, f = i % FN;
      const bool in = skind[sl][side] == 0;
      const double *p = in ? src + (int64_t)c * ncells * NP + snbr[sl][side] +
                                 cv_end_node<N>(side >> 1, (side & 1) ^ 1, f / N, f % N)
                           : src;
      cp_async8(snb + i, p, in);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // prologue: item 0 (own cell, neighbour layers), side info of items 0, 1
  if (tid == 0) issue_own(0);
  side_info(0);
  if (nitems > 1) side_info(1);
  __syncthreads();
  load_nbr(0, 0);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();

  int64_t e = blockIdx.x;
  int lev = 0;
  for (int64_t w = 0; w < nitems; ++w) {
    const double beta = p_beta[lev];
    const bool has_next = w + 1 < nitems;
    const int lev_next = lev + 1 == nh ? 0 : lev + 1;
    if (has_next && tid == 0) issue_own(w + 1);
    if (has_next) load_nbr(w + 1, lev_next);
    const double *snb = sm + C::NB + (w & 1) * 18 * FN;
    int ix, iy, iz;
    cv2_xyz(g, e, ix, iy, iz);  // 32-bit divisions, once per item
    const double h[3] = {g.hx[ix], g.hy[iy], g.hz[iz]};
    const double sc[3] = {2.0 * g.hxi[ix], 2.0 * g.hyi[iy], 2.0 * g.hzi[iz]};
    const double det = 0.125 * h[0] * h[1] * h[2];
    mbar_wait(&bars[w & 1], (int)((w >> 1) & 1));
    const double *su = sm + ((w & 1) ? C::SU1 : C::SU0);

    // ---- volume: nodes -> Gauss points --------------------------------------
    double *x1 = ra, *x2 = rb, *uq = ra;
    for (int l = tid; l < 3 * N * N; l += T) {  // x lines: x1[c z y][qx] (pitch P1)
      double xi[N], yo[NQ];
      cv_load<N>(su + l * N, 1, xi);
      eo_line<NQ, N, 1>(eo.S, xi, yo);
      cv_store<NQ>(x1 + l * P1, 1, yo);
    }
    __syncthreads();
    for (int l = tid; l < 3 * N * NQ; l += T) {  // y lines: x2[c][z][qy][qx]
      const int cz = l / NQ, qx = l % NQ;
      double xi[N], yo[NQ];
      cv_load<N>(x1 + cz * N * P1 + qx, P1, xi);
      eo_line<NQ, N, 1>(eo.S, xi, yo);
      cv_store<NQ>(x2 + cz * NQ2 + qx, NQ, yo);
    }
    __syncthreads();
    for (int l = tid; l < 3 * NQ2; l += T) {  // z lines: uq[c][qz][qy][qx]
      const int c = l / NQ2, qxy = l % NQ2;
      double xi[N], yo[NQ];
      cv_load<N>(x2 + c * N * NQ2 + qxy, NQ2, xi);
      eo_line<NQ, N, 1>(eo.S, xi, yo);
      cv_store<NQ>(uq + c * QP + qxy, NQ2, yo);
    }
    __syncthreads();
    // G_ab = beta u_a u_b JxW and its z test contraction (vconv.cuh jobs)
    auto gjob = [&](const int job, const int qxy, const double wxy) {
      const int a = job == 1 ? 1 : (job == 2 ? 2 : (job >= 6 ? 1 : 0));
      const int b = job == 0 ? 0 : (job == 1 || job == 3 ? 1 : 2);
      const bool dz = job == 2 || job == 4 || job == 6;
      double ua[NQ], ub[NQ], gz[NQ], zo[N];
      cv_load<NQ>(uq + a * QP + qxy, NQ2, ua);
      cv_load<NQ>(uq + b * QP + qxy, NQ2, ub);
#pragma unroll
      for (int q = 0; q < NQ; ++q) gz[q] = ua[q] * ub[q] * (wxy * tab.w[q]);
      if (dz) eo_line<N, NQ, -1>(eo.Dt, gz, zo);
      else eo_line<N, NQ, 1>(eo.St, gz, zo);
      const int r = dz ? a : (job == 5 || job == 7 ? 2 : a);
      const int t = dz ? 2 : (job == 5 ? 0 : (job == 7 ? 1 : b));
      const double st = cv_sel3(sc, t);
      double *zd = rb + (r * 3 + t) * N * NQ2 + qxy;
#pragma unroll
      for (int z = 0; z < N; ++z) zd[z * NQ2] = st * zo[z];
      if (job == 3) {
        double *z2 = rb + (1 * 3 + 0) * N * NQ2 + qxy;
#pragma unroll
        for (int z = 0; z < N; ++z) z2[z * NQ2] = sc[0] * zo[z];
      }
        };
    // two jobs per pass (T = 2 NQ2): the warp-uniform job residue picks one of
    // two fully compile-time job sequences; the three component lines at this
    // point are loaded once for its four jobs
    auto gjob_c = [&](auto JC, const double (&uc)[3][NQ], const int qxy, const double wxy) {
      constexpr int job = decltype(JC)::value;
      constexpr int a = job == 1 ? 1 : (job == 2 ? 2 : (job >= 6 ? 1 : 0));
      constexpr int b = job == 0 ? 0 : (job == 1 || job == 3 ? 1 : 2);
      constexpr bool dz = job == 2 || job == 4 || job == 6;
      constexpr int r = dz ? a : (job == 5 || job == 7 ? 2 : a);
      constexpr int t = dz ? 2 : (job == 5 ? 0 : (job == 7 ? 1 : b));
      double gz[NQ], zo[N];
#pragma unroll
      for (int q = 0; q < NQ; ++q) gz[q] = uc[a][q] * uc[b][q] * (wxy * tab.w[q]);
      if (dz) eo_line<N, NQ, -1>(eo.Dt, gz, zo);
      else eo_line<N, NQ, 1>(eo.St, gz, zo);
      const double st = sc[t];
      double *zd = rb + (r * 3 + t) * N * NQ2 + qxy;
#pragma unroll
      for (int z = 0; z < N; ++z) zd[z * NQ2] = st * zo[z];
      if (job == 3) {
        double *z2 = rb + (1 * 3 + 0) * N * NQ2 + qxy;
#pragma unroll
        for (int z = 0; z < N; ++z) z2[z * NQ2] = sc[0] * zo[z];
      }
    };
    if (T == 2 * NQ2) {
      const int jh = tid / NQ2, qxy = tid - jh * NQ2;
      const double wxy = beta * det * W[qxy % NQ] * W[qxy / NQ];
      double uc[3][NQ];
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) cv_load<NQ>(uq + cc * QP + qxy, NQ2, uc[cc]);
      if (jh == 0) {
        gjob_c(Cv2Job<0>{}, uc, qxy, wxy);
        gjob_c(Cv2Job<2>{}, uc, qxy, wxy);
        gjob_c(Cv2Job<4>{}, uc, qxy, wxy);
        gjob_c(Cv2Job<6>{}, uc, qxy, wxy);
      } else {
        gjob_c(Cv2Job<1>{}, uc, qxy, wxy);
        gjob_c(Cv2Job<3>{}, uc, qxy, wxy);
        gjob_c(Cv2Job<5>{}, uc, qxy, wxy);
        gjob_c(Cv2Job<7>{}, uc, qxy, wxy);
      }
    } else if (T % NQ2 == 0 && (8 * NQ2) % T == 0) {
      // T / NQ2 jobs per pass: this thread's point and its job residue are
      // fixed, the job index is a compile-time offset (no select chains)
      constexpr int JP = T % NQ2 == 0 ? T / NQ2 : 1;
      const int jh = tid / NQ2, qxy = tid - jh * NQ2;
      const double wxy = beta * det * W[qxy % NQ] * W[qxy / NQ];
#pragma unroll
      for (int jp = 0; jp < 8 / JP; ++jp) gjob(jp * JP + jh, qxy, wxy);
    } else {
      for (int l = tid; l < 8 * NQ2; l += T) {
        const int job = l / NQ2, qxy = l % NQ2;
        gjob(job, qxy, beta * det * W[qxy % NQ] * W[qxy / NQ]);
      }
    }
    __syncthreads();
    // y lines: A_a = S^T Z_a2 + D^T Z_a1, B_a = S^T Z_a0 -> ra[a][A|B][z][y][qx] (pitch P1)
    for (int l = tid; l < 3 * N * NQ; l += T) {
      const int a = l / (N * NQ), z = (l / NQ) % N, qx = l % NQ;
      double z0[NQ], z1[NQ], z2[NQ], ya[N], yb[N], yd[N];
      const double *zb = rb + (a * 3 * N + z) * NQ2 + qx;
      cv_load<NQ>(zb, NQ, z0);
      cv_load<NQ>(zb + N * NQ2, NQ, z1);
      cv_load<NQ>(zb + 2 * N * NQ2, NQ, z2);
      eo_line<N, NQ, 1>(eo.St, z2, ya);
      eo_line<N, NQ, -1>(eo.Dt, z1, yd);
      eo_line<N, NQ, 1>(eo.St, z0, yb);
#pragma unroll
      for (int y = 0; y < N; ++y) ya[y] += yd[y];
      cv_store<N>(ra + (((a * 2 + 0) * N + z) * N) * P1 + qx, P1, ya);
      cv_store<N>(ra + (((a * 2 + 1) * N + z) * N) * P1 + qx, P1, yb);
    }
    if (tid == 0) cv2_wait_read();  // the previous cell's bulk store has read so
    __syncthreads();
    // x lines: out_a (=, first level; += later) S^T A_a + D^T B_a, and (same
    // phase, independent) the fast tangential sweep of the own / neighbour end
    // layers -> rb[o side c sl][qfa] (pitch P1; Z is dead)
    for (int l = tid; l < 3 * N * N + 36 * N; l += T) {
      if (l < 3 * N * N) {
        const int a = l / (N * N), zy = l % (N * N);
        double xa[NQ], xb[NQ], oa[N], ob[N];
        cv_load<NQ>(ra + ((a * 2 + 0) * N * N + zy) * P1, 1, xa);
        cv_load<NQ>(ra + ((a * 2 + 1) * N * N + zy) * P1, 1, xb);
        eo_line<N, NQ, 1>(eo.St, xa, oa);
        eo_line<N, NQ, -1>(eo.Dt, xb, ob);
        double *o = so + a * NP + zy * N;
        if (lev == 0) {
#pragma unroll
          for (int x = 0; x < N; ++x) o[x] = oa[x] + ob[x];
        } else {
#pragma unroll
          for (int x = 0; x < N; ++x) o[x] += oa[x] + ob[x];
        }
      } else {
        const int m = l - 3 * N * N;
        const int o = m / (18 * N), side = (m / (3 * N)) % 6, c = (m / N) % 3, sl = m % N;
        const int d = side >> 1;
        double xi[N], yo[NQ];
        if (o == 0) cv_load<N>(su + c * NP + cv_end_node<N>(d, side & 1, sl, 0), d == 0 ? N : 1, xi);
        else cv_load<N>(snb + (side * 3 + c) * FN + sl * N, 1, xi);
        eo_line<NQ, N, 1>(eo.S, xi, yo);
        cv_store<NQ>(rb + m * P1, 1, yo);
      }
    }
    __syncthreads();
    // ---- faces ----------------------------------------------------------------
    // slow sweep: traces ra[o][side][c][qsl][qfa]
    double *tr = ra;
    for (int l = tid; l < 36 * NQ; l += T) {
      const int osc = l / NQ, qfa = l % NQ;
      double xi[N], yo[NQ];
      cv_load<N>(rb + osc * N * P1 + qfa, P1, xi);
      eo_line<NQ, N, 1>(eo.S, xi, yo);
      cv_store<NQ>(tr + osc * FQ + qfa, NQ, yo);
    }
    __syncthreads();
    // Lax-Friedrichs flux at the face Gauss points -> vf[side a qsl][qfa] (rb, pitch P1)
    double *vf = rb;
    for (int i = tid; i < 6 * FQ; i += T) {
      const int side = i / FQ, f = i % FQ, d = side >> 1, s = side & 1;
      const int k = skind[w & 1][side];
      const double nsgn = s ? 1.0 : -1.0;
      const double fdet = d == 0 ? 0.25 * h[1] * h[2] : (d == 1 ? 0.25 * h[0] * h[2] : 0.25 * h[0] * h[1]);
      const double sj = fdet * W[f % NQ] * W[f / NQ];
      double uo[3], up[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        uo[c] = tr[(side * 3 + c) * FQ + f];
        up[c] = tr[(18 + side * 3 + c) * FQ + f];
      }
      if (k != 0) {  // mirror state 2 g - u with the level's Dirichlet data
        const double *gd = p_gh[lev][side];
        const int64_t it = d == 0 ? (int64_t)iz * g.ny + iy
                                  : (d == 1 ? (int64_t)iz * g.nx + ix : (int64_t)iy * g.nx + ix);
#pragma unroll
        for (int c = 0; c < 3; ++c) up[c] = (gd ? 2.0 * gd[(it * 3 + c) * FQ + f] : 0.0) - uo[c];
      }
      const double unm = cv_sel3(uo, d) * nsgn, unp = cv_sel3(up, d) * nsgn;
      const int fo = (f / NQ) * P1 + f % NQ;
      if (k == kBndNeumann) {
#pragma unroll
        for (int a = 0; a < 3; ++a) vf[(side * 3 + a) * NQ * P1 + fo] = -beta * uo[a] * unm * sj;
      } else {
        const double lam = 2.0 * fmax(fabs(unm), fabs(unp));
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double Fl = 0.5 * (uo[a] * unm + up[a] * unp) + 0.5 * lam * (uo[a] - up[a]);
          vf[(side * 3 + a) * NQ * P1 + fo] = -beta * Fl * sj;
        }
      }
    }
    __syncthreads();
    // lift, fast: ra[side a qsl][fa] = S^T along the fast face axis
    for (int l = tid; l < 18 * NQ; l += T) {
      double xi[NQ], yo[N];
      cv_load<NQ>(vf + l * P1, 1, xi);
      eo_line<N, NQ, 1>(eo.St, xi, yo);
      cv_store<N>(ra + l * N, 1, yo);
    }
    __syncthreads();
    // lift, slow, added straight onto the end nodes one axis at a time (the
    // two sides of an axis touch disjoint nodes; edges / corners get one side
    // per phase)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      for (int l = tid; l < 6 * N; l += T) {  // [s][a][fa]
        const int sa = 6 * d + l / N, fa = l % N, s = (sa / 3) & 1, a = sa % 3;
        double xi[NQ], yo[N];
        cv_load<NQ>(ra + sa * NQ * N + fa, N, xi);
        eo_line<N, NQ, 1>(eo.St, xi, yo);
#pragma unroll
        for (int sl = 0; sl < N; ++sl) so[a * NP + cv_end_node<N>(d, s, sl, fa)] += yo[sl];
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // so -> bulk store
      __syncthreads();
    }

    if (lev == nh - 1) {
      if (prm.vol_data != nullptr) {
        // (v, f) with the body force at the quadrature points, z, y, x
        for (int l = tid; l < 3 * NQ2; l += T) {  // rb[a][z][qy][qx]
          const int a = l / NQ2, qxy = l % NQ2;
          const double wxy = det * W[qxy % NQ] * W[qxy / NQ];
          const double *fd = prm.vol_data + ((int64_t)a * ncells + e) * QP + qxy;
          double xi[NQ], yo[N];
#pragma unroll
          for (int q = 0; q < NQ; ++q) xi[q] = fd[q * NQ2] * (wxy * tab.w[q]);
          eo_line<N, NQ, 1>(eo.St, xi, yo);
          cv_store<N>(rb + a * N * NQ2 + qxy, NQ2, yo);
        }
        __syncthreads();
        for (int l = tid; l < 3 * N * NQ; l += T) {  // ra[a z y][qx] (pitch P1)
          const int az = l / NQ, qx = l % NQ;
          double xi[NQ], yo[N];
          cv_load<NQ>(rb + az * NQ2 + qx, NQ, xi);
          eo_line<N, NQ, 1>(eo.St, xi, yo);
          cv_store<N>(ra + az * N * P1 + qx, P1, yo);
        }
        __syncthreads();
        for (int l = tid; l < 3 * N * N; l += T) {
          double xi[NQ], yo[N];
          cv_load<NQ>(ra + l * P1, 1, xi);
          eo_line<N, NQ, 1>(eo.St, xi, yo);
          double *o = so + l * N;
#pragma unroll
          for (int x = 0; x < N; ++x) o[x] += yo[x];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
      }
      if ((NP * sizeof(double)) % 16 == 0 && (smem_u32(so) & 15) == 0 &&
          (reinterpret_cast<uintptr_t>(out) & 15) == 0) {  // 3 TMA bulk stores
        if (tid == 0) {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            cv2_s2g(out + ((int64_t)c * ncells + e) * NP, so + c * NP, (uint32_t)(NP * sizeof(double)));
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      } else {
        for (int i = tid; i < 3 * NP; i += T) {
          const int c = i / NP, o = i % NP;
          out[((int64_t)c * ncells + e) * NP + o] = so[i];
        }
      }
    }
    // side info of item w + 2 into this item's slot (read by the LF phase
    // above and by the prefetch at the start of this item: both done)
    if (w + 2 < nitems) side_info(w + 2);
    asm volatile("cp.async.wait_all;" ::: "memory");  // the next item's neighbour layers
    __syncthreads();  // so / skind are rewritten by the next items
    if (++lev == nh) {
      lev = 0;
      e += gridDim.x;
    }
  }
  if (tid == 0) cv2_wait_read();  // the last bulk store has read so
}

}  // namespace dg
