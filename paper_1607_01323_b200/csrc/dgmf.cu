// C-ABI implementation of the B200 matrix-free DG library (include/dgmf.h).
#include <cmath>
#include <initializer_list>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <algorithm>
#include <map>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "laplace.cuh"
#include "laplace6.cuh"
#include "laplace7.cuh"
#include "laplace8.cuh"
#include "laplace9.cuh"
#include "mg.cuh"
#include "tables.h"
#include "tensor.cuh"
#include "tensor_fast.cuh"
#include "vector.cuh"

namespace dg {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char *where) {
  g_err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
  return DG_ECUDA;
}

int inval(const std::string &m) {
  g_err = m;
  return DG_EINVAL;
}

}  // namespace dg

using namespace dg;

// tau_e of GLOBAL cell (gx, gy, gz), Eq. 18 (geometry.py:90-108): every
// boundary face counts in A_bnd (also walls without a pressure term),
// periodic faces count as interior.  On Cartesian cells A/V separates per
// axis, tau_e = (k+1)^2 sum_d (w_lo + w_hi) / h_d with w = 1 on a boundary
// side and 1/2 otherwise; the sum is taken in the fixed order (x + y) + z,
// the order in which the Laplace column kernel (laplace7.cuh) forms it from
// the per-axis terms, so tau is bitwise the same everywhere.
static double tau_axis(const dg_ctx *c, int d, int gi) {
  const double h = c->gvert[d][gi + 1] - c->gvert[d][gi];
  double w = 0.0;
  for (int s = 0; s < 2; ++s) {
    const bool edge = s ? (gi == c->gcounts[d] - 1) : (gi == 0);
    w += (edge && !c->periodic[d]) ? 1.0 : 0.5;
  }
  const double kp = (double)(c->k + 1);
  return kp * kp * w / h;
}

static double tau_global(const dg_ctx *c, int gx, int gy, int gz) {
  double t = tau_axis(c, 0, gx) + tau_axis(c, 1, gy);
  if (c->dim == 3) t += tau_axis(c, 2, gz);
  return t;
}

// per-axis cell data of the owned index range extended by one cell per side
// (the periodic wrap or x-slab ghost neighbour; a copy of the end cell on a
// boundary): [i + 1][h, 1/h, tau_axis, 0] for local i in [-1, n_d]
static std::vector<double> axis_table(const dg_ctx *c, int d) {
  const int n = c->counts[d], off = d == 0 ? c->slab_begin : 0, gn = c->gcounts[d];
  std::vector<double> t(4 * (size_t)(n + 2), 0.0);
  for (int i = -1; i <= n; ++i) {
    int gi = off + i;
    if (gi < 0) gi = c->periodic[d] ? gn - 1 : 0;
    if (gi >= gn) gi = c->periodic[d] ? 0 : gn - 1;
    double *e = &t[4 * (size_t)(i + 1)];
    e[0] = c->gvert[d][gi + 1] - c->gvert[d][gi];
    e[1] = 1.0 / e[0];
    e[2] = d < c->dim ? tau_axis(c, d, gi) : 0.0;
  }
  return t;
}

template <typename T>
static int upload(T **dst, const std::vector<T> &src) {
  DG_CUDA_CHECK(cudaMalloc((void **)dst, sizeof(T) * (src.empty() ? 1 : src.size())));
  if (!src.empty())
    DG_CUDA_CHECK(cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice));
  return 0;
}

extern "C" {

const char *dg_last_error(void) { return g_err.c_str(); }

int dg_basis_tables(int k, int n_q, double *S, double *D, double *nodes, double *points,
                    double *weights, double *left_deriv, double *right_deriv) {
  if (k < 1 || k > 7) return inval("polynomial degree must be in 1..7");
  if (n_q < 1) return inval("need at least one quadrature point");
  Basis1D b;
  basis_tables(k, n_q, b);
  if (S) std::memcpy(S, b.S.data(), sizeof(double) * b.S.size());
  if (D) std::memcpy(D, b.D.data(), sizeof(double) * b.D.size());
  if (nodes) std::memcpy(nodes, b.nodes.data(), sizeof(double) * b.nodes.size());
  if (points) std::memcpy(points, b.pts.data(), sizeof(double) * b.pts.size());
  if (weights) std::memcpy(weights, b.wts.data(), sizeof(double) * b.wts.size());
  if (left_deriv) std::memcpy(left_deriv, b.ld.data(), sizeof(double) * b.ld.size());
  if (right_deriv) std::memcpy(right_deriv, b.rd.data(), sizeof(double) * b.rd.size());
  return DG_OK;
}

static int ensure_cell_table(dg_ctx *c, cudaStream_t st);

int dg_ctx_create(const dg_mesh_desc *desc, dg_ctx **out) {
  if (!desc || !out) return inval("null argument");
  *out = nullptr;
  if (desc->dim != 2 && desc->dim != 3) return inval("dim must be 2 or 3");
  if (desc->k < 1 || desc->k > 7)
    return inval("polynomial degree must be in 1..7 (got " + std::to_string(desc->k) + ")");
  dg_ctx *c = new dg_ctx();
  c->dim = desc->dim;
  c->k = desc->k;
  c->n = desc->k + 1;
  c->nq_over = desc->n_q_over > 0 ? desc->n_q_over : (3 * desc->k) / 2 + 1;
  for (int d = 0; d < 3; ++d) {
    c->gcounts[d] = (d < c->dim) ? desc->counts[d] : 1;
    c->periodic[d] = (d < c->dim) ? desc->periodic[d] : 0;
    if (c->gcounts[d] < 1) {
      delete c;
      return inval("counts must be >= 1 per axis");
    }
  }
  for (int d = 0; d < c->dim; ++d) {
    if (!desc->vertices[d]) {
      delete c;
      return inval("missing vertex coordinates");
    }
    c->gvert[d].assign(desc->vertices[d], desc->vertices[d] + c->gcounts[d] + 1);
    for (int i = 0; i < c->gcounts[d]; ++i)
      if (!(c->gvert[d][i + 1] > c->gvert[d][i])) {
        delete c;
        return inval("non-positive mapping Jacobian (vertex coordinates must increase)");
      }
  }
  if (c->dim == 2) c->gvert[2] = {0.0, 2.0};  // unit-free dummy z extent
  for (int t = 0; t < 6; ++t) c->bc[t] = (t < 2 * c->dim) ? desc->bc_kind[t] : 0;
  for (int d = 0; d < c->dim; ++d)
    for (int s = 0; s < 2; ++s) {
      const int kind = c->bc[2 * d + s];
      if (!c->periodic[d] && kind != DG_BC_VELOCITY_DIRICHLET && kind != DG_BC_VELOCITY_NEUMANN) {
        delete c;
        static const char *names[6] = {"xmin", "xmax", "ymin", "ymax", "zmin", "zmax"};
        return inval(std::string("boundary tags without a condition: {'") + names[2 * d + s] + "'}");
      }
    }
  c->slab_begin = desc->slab_begin;
  c->slab_end = desc->slab_end > 0 ? desc->slab_end : c->gcounts[0];
  if (c->slab_begin < 0 || c->slab_end > c->gcounts[0] || c->slab_begin >= c->slab_end) {
    delete c;
    return inval("invalid slab range");
  }
  c->counts[0] = c->slab_end - c->slab_begin;
  c->counts[1] = c->gcounts[1];
  c->counts[2] = c->gcounts[2];
  const bool whole_x = (c->slab_begin == 0 && c->slab_end == c->gcounts[0]);
  auto bnd_mode = [&](int t) { return c->bc[t] == DG_BC_VELOCITY_NEUMANN ? kBndNeumann : kBndNone; };
  // x sides
  if (c->slab_begin > 0) c->mode[0] = kGhost;
  else if (c->periodic[0]) c->mode[0] = whole_x ? kWrap : kGhost;
  else c->mode[0] = bnd_mode(0);
  if (c->slab_end < c->gcounts[0]) c->mode[1] = kGhost;
  else if (c->periodic[0]) c->mode[1] = whole_x ? kWrap : kGhost;
  else c->mode[1] = bnd_mode(1);
  for (int d = 1; d < 3; ++d)
    for (int s = 0; s < 2; ++s)
      c->mode[2 * d + s] = (d >= c->dim || c->periodic[d]) ? kWrap : bnd_mode(2 * d + s);

  basis_tables(c->k, c->n, c->basis);
  basis_tables(c->k, c->nq_over, c->over);
  c->np = 1;
  for (int d = 0; d < c->dim; ++d) c->np *= c->n;
  c->n_cells = (int64_t)c->counts[0] * c->counts[1] * c->counts[2];
  c->n_dofs = c->n_cells * c->np;

  c->hx.resize(c->counts[0]);
  for (int i = 0; i < c->counts[0]; ++i)
    c->hx[i] = c->gvert[0][c->slab_begin + i + 1] - c->gvert[0][c->slab_begin + i];
  c->hy.resize(c->counts[1]);
  for (int i = 0; i < c->counts[1]; ++i) c->hy[i] = c->gvert[1][i + 1] - c->gvert[1][i];
  c->hz.resize(c->counts[2]);
  for (int i = 0; i < c->counts[2]; ++i) c->hz[i] = c->gvert[2][i + 1] - c->gvert[2][i];
  c->tau.resize(c->n_cells);
  for (int iz = 0; iz < c->counts[2]; ++iz)
    for (int iy = 0; iy < c->counts[1]; ++iy)
      for (int ix = 0; ix < c->counts[0]; ++ix)
        c->tau[ix + (size_t)c->counts[0] * (iy + (size_t)c->counts[1] * iz)] =
            tau_global(c, c->slab_begin + ix, iy, iz);
  c->volume = 1.0;
  for (int d = 0; d < c->dim; ++d) c->volume *= (c->gvert[d].back() - c->gvert[d].front());
  // ghost layers
  const int64_t layer = (int64_t)c->counts[1] * c->counts[2];
  // 3D Q3-Q5 run the column kernel, whose halo consumes face traces
  c->halo_traces = (c->dim == 3 && c->n >= 4 && c->n <= 6) ? 1 : 0;
  c->halo_count = layer * (c->halo_traces ? 2 * c->n * c->n : c->np);
  int rc = 0;
  for (int s = 0; s < 2; ++s) {
    int gx;
    if (s == 0) gx = c->slab_begin > 0 ? c->slab_begin - 1 : c->gcounts[0] - 1;
    else gx = c->slab_end < c->gcounts[0] ? c->slab_end : 0;
    c->ghost_h[s] = c->gvert[0][gx + 1] - c->gvert[0][gx];
    c->ghost_tau_h[s].resize(layer);
    for (int iz = 0; iz < c->counts[2]; ++iz)
      for (int iy = 0; iy < c->counts[1]; ++iy)
        c->ghost_tau_h[s][iy + (size_t)c->counts[1] * iz] = tau_global(c, gx, iy, iz);
    if (c->mode[2 * 0 + s] == kGhost) {
      if ((rc = upload(&c->d_ghost_tau[s], c->ghost_tau_h[s]))) goto fail;
    }
  }
  if ((rc = upload(&c->d_hx, c->hx))) goto fail;
  if ((rc = upload(&c->d_hy, c->hy))) goto fail;
  if ((rc = upload(&c->d_hz, c->hz))) goto fail;
  {
    std::vector<double> hinv;
    for (double h : c->hx) hinv.push_back(1.0 / h);
    for (double h : c->hy) hinv.push_back(1.0 / h);
    for (double h : c->hz) hinv.push_back(1.0 / h);
    if ((rc = upload(&c->d_hinv, hinv))) goto fail;
  }
  if ((rc = upload(&c->d_tau, c->tau))) goto fail;
  {
    std::vector<double> ax;
    for (int d = 0; d < 3; ++d) {
      c->axis_off[d] = (int64_t)ax.size() + 4;  // entry of local index 0
      const std::vector<double> t = axis_table(c, d);
      ax.insert(ax.end(), t.begin(), t.end());
    }
    if ((rc = upload(&c->d_axis, ax))) goto fail;
  }
  if (cudaMalloc((void **)&c->d_red, sizeof(double) * (kRedBlocks + 64)) != cudaSuccess) goto cfail;
  if (cudaMalloc((void **)&c->d_scal, sizeof(double) * 32) != cudaSuccess) goto cfail;
  if (cudaMemset(c->d_scal, 0, sizeof(double) * 32) != cudaSuccess) goto cfail;
  if (cudaMallocHost((void **)&c->h_scal, sizeof(double) * 32) != cudaSuccess) goto cfail;
  // the Laplace cell table, built here (not lazily: vmults may run under
  // CUDA-graph capture, where allocation is not allowed)
  if (c->dim == 3) {
    if ((rc = ensure_cell_table(c, 0))) goto fail;
    if (cudaDeviceSynchronize() != cudaSuccess) goto cfail;
  }
  *out = c;
  return DG_OK;
cfail:
  rc = cuda_fail(cudaGetLastError(), "dg_ctx_create allocation");
fail:
  dg_ctx_destroy(c);
  return rc ? rc : DG_ECUDA;
}

int dg_ctx_destroy(dg_ctx *c) {
  if (!c) return DG_OK;
  cudaFree(c->d_hx);
  cudaFree(c->d_hy);
  cudaFree(c->d_hz);
  cudaFree(c->d_hinv);
  cudaFree(c->d_hin);
  cudaFree(c->d_hout);
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  cudaFree(c->d_tau);
  cudaFree(c->d_axis);
  cudaFree(c->d_red3);
  cudaFree(c->d_hcell);
  cudaFree(c->d_counter);
  for (int s = 0; s < 2; ++s) {
    cudaFree(c->d_ghost_tau[s]);
  }
  cudaFree(c->d_red);
  cudaFree(c->d_scal);
  if (c->h_scal) cudaFreeHost(c->h_scal);
  for (double *w : c->work) cudaFree(w);
  cudaFree(c->d_partials);
  cudaFree(c->d_trc);
  cudaFree(c->d_ctab);
  for (double *w : c->vwork) cudaFree(w);
  cudaFree(c->d_vpart);
  cudaFree(c->d_apdot);
  cudaFree(c->d_zero_ghost);
  delete c;
  return DG_OK;
}

int dg_ctx_sizes(const dg_ctx *c, int64_t *n_cells, int64_t *n_dofs) {
  if (!c) return inval("null context");
  if (n_cells) *n_cells = c->n_cells;
  if (n_dofs) *n_dofs = c->n_dofs;
  return DG_OK;
}

int dg_ctx_tau(const dg_ctx *c, double *tau_e_host) {
  if (!c || !tau_e_host) return inval("null argument");
  std::memcpy(tau_e_host, c->tau.data(), sizeof(double) * c->tau.size());
  return DG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Laplace vmult dispatch

template <int N>
static LapTab<N> lap_tab(const Basis1D &b) {
  LapTab<N> t;
  for (int i = 0; i < N * N; ++i) {
    t.M[i] = b.M[i];
    t.K[i] = b.K[i];
  }
  for (int i = 0; i < N; ++i) {
    t.dL[i] = b.ld[i];
    t.dR[i] = b.rd[i];
  }
  // even-odd splits of the centro-symmetric M, K (A[i][j] = A[N-1-i][N-1-j])
  // and of the antisymmetric endpoint derivative rows (dR_j = -dL_{N-1-j})
  constexpr int H = N / 2, NE = (N + 1) / 2;
  for (int i = 0; i < NE; ++i)
    for (int j = 0; j < NE; ++j) {
      const bool mid = (j == H);  // only for odd N
      t.Me[i * NE + j] = mid ? b.M[i * N + j] : 0.5 * (b.M[i * N + j] + b.M[i * N + N - 1 - j]);
      t.Ke[i * NE + j] = mid ? b.K[i * N + j] : 0.5 * (b.K[i * N + j] + b.K[i * N + N - 1 - j]);
    }
  for (int i = 0; i < H; ++i)
    for (int j = 0; j < H; ++j) {
      t.Mo[i * H + j] = 0.5 * (b.M[i * N + j] - b.M[i * N + N - 1 - j]);
      t.Ko[i * H + j] = 0.5 * (b.K[i * N + j] - b.K[i * N + N - 1 - j]);
    }
  for (int j = 0; j < NE; ++j)
    t.dLe[j] = (j == H) ? b.ld[j] : 0.5 * (b.ld[j] + b.ld[N - 1 - j]);
  for (int j = 0; j < H; ++j) t.dLo[j] = 0.5 * (b.ld[j] - b.ld[N - 1 - j]);
  return t;
}

// dg_laplace_kernel_name: when set, the launchers below record the kernel
// they would launch ("name<template args>") instead of launching it
static thread_local std::string *t_kname = nullptr;
static std::string kname(const char *base, std::initializer_list<int> args) {
  std::string s = std::string(base) + "<";
  bool first = true;
  for (int a : args) {
    if (!first) s += ",";
    s += std::to_string(a);
    first = false;
  }
  return s + ">";
}

// z-range of cell layers [z0, z1) of the vmult being launched by this host
// thread (the pipelined host-buffer path; z1 <= 0: whole mesh).  Thread-local,
// so concurrent calls on other threads are unaffected.
struct ZChunk {
  int z0 = 0, z1 = 0;
};
static thread_local ZChunk t_chunk;

// z-bricks of a launch: the current chunk (z0 a multiple of 4 >= BZ), else all
static unsigned chunk_bricks_z(const dg_ctx *c, int BZ, Geo &g) {
  (void)c;
  if (t_chunk.z1 > 0) {
    g.bz0 = t_chunk.z0 / BZ;
    return (unsigned)((t_chunk.z1 - t_chunk.z0 + BZ - 1) / BZ);
  }
  g.bz0 = 0;
  return (unsigned)((g.nz + BZ - 1) / BZ);
}

// the context's Laplace cell table (3D): per-(cell, side) SIP coefficients and
// stiffness scales, built once on the stream of the first vmult
static int ensure_cell_table(dg_ctx *c, cudaStream_t st) {
  if (c->d_ctab) return DG_OK;
  double *tab = nullptr;
  DG_CUDA_CHECK(cudaMalloc(&tab, sizeof(double) * kCellTab * (size_t)c->n_cells));
  const Geo g0 = c->geo();
  const int64_t items = 7 * c->n_cells;
  lap6_cell_table_kernel<<<(unsigned)((items + 255) / 256), 256, 0, st>>>(g0, tab);
  DG_LAUNCH_CHECK("lap6_cell_table_kernel");
  c->d_ctab = tab;
  return DG_OK;
}

template <int DIM, int N, int BX, int BY, int BZ, int EPI = kEpiStore>
static int launch_laplace(dg_ctx *c, const double *src, double *dst, double tau_scale, int part,
                          cudaStream_t st, const EpiArgs &ea = EpiArgs{}) {
  if (t_kname) {
    *t_kname = kname("laplace_vmult_kernel", {DIM, N, BX, BY, BZ, EPI});
    return DG_OK;
  }
  using C = LapCfg<DIM, N, BX, BY, BZ>;
  auto kern = laplace_vmult_kernel<DIM, N, BX, BY, BZ, EPI>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr = true;
  }
  if (c->dim == 3 && ensure_cell_table(c, st) != DG_OK) return DG_ECUDA;
  Geo g = c->geo();
  const dim3 grid((g.nx + BX - 1) / BX, (g.ny + BY - 1) / BY, chunk_bricks_z(c, BZ, g));
  kern<<<grid, C::THREADS, C::SMEM, st>>>(src, dst, g, lap_tab<N>(c->basis), tau_scale, part, ea);
  DG_LAUNCH_CHECK("laplace_vmult_kernel");
  return DG_OK;
}

// ---- fp32 Laplace (the fp32 V-cycle): the same v4 kernel
// instantiated in single precision, 1D tables rounded once from the fp64 ones
template <int N>
static LapTab<N, float> lap_tab_f(const Basis1D &b) {
  const LapTab<N> d = lap_tab<N>(b);
  LapTab<N, float> t;
  const double *src = reinterpret_cast<const double *>(&d);
  float *dst = reinterpret_cast<float *>(&t);
  static_assert(sizeof(LapTab<N>) == 2 * sizeof(LapTab<N, float>), "table layouts");
  for (size_t i = 0; i < sizeof(LapTab<N>) / sizeof(double); ++i) dst[i] = (float)src[i];
  return t;
}

template <int DIM, int N, int BX, int BY, int BZ, int EPI>
static int launch_laplace_f(dg_ctx *c, const float *src, float *dst, double tau_scale,
                            cudaStream_t st, const EpiArgsT<float> &ea) {
  using C = LapCfg<DIM, N, BX, BY, BZ, float>;
  auto kern = laplace_vmult_kernel<DIM, N, BX, BY, BZ, EPI, float>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr = true;
  }
  if (DIM == 3 && ensure_cell_table(c, st) != DG_OK) return DG_ECUDA;
  Geo g = c->geo();
  g.bz0 = 0;
  const dim3 grid((g.nx + BX - 1) / BX, (g.ny + BY - 1) / BY, (g.nz + BZ - 1) / BZ);
  kern<<<grid, C::THREADS, C::SMEM, st>>>(src, dst, g, lap_tab_f<N>(c->basis), tau_scale, 0, ea);
  DG_LAUNCH_CHECK("laplace_vmult_kernel<float>");
  return DG_OK;
}

// out = L src (epi = kEpiStore) or the fused Chebyshev step (kEpiCheb), fp32,
// 3D whole-mesh contexts
static int laplace_dispatch_f(dg_ctx *c, const float *src, float *dst, double tau_scale, int epi,
                              const EpiArgsT<float> &ea, cudaStream_t st) {
  if (c->dim != 3 || c->mode[0] == kGhost || c->mode[1] == kGhost)
    return inval("fp32 Laplace: 3D whole-mesh contexts");
#define DG_F(NN, X, Y, Z)                                                                   \
  case NN:                                                                                  \
    return epi == kEpiCheb                                                                  \
               ? launch_laplace_f<3, NN, X, Y, Z, kEpiCheb>(c, src, dst, tau_scale, st, ea) \
               : launch_laplace_f<3, NN, X, Y, Z, kEpiStore>(c, src, dst, tau_scale, st, ea);
  // fp32 halves the shared memory per cell: larger bricks than fp64 at
  // k = 3, 4 (measured on the config-4 / config-2 V-cycles: 4x4x4 1.24 vs
  // 4x4x2 1.31 ms; 8x2x2 1.70 vs 4x2x2 1.85 ms)
  switch (c->n) {
    DG_F(2, 8, 4, 4) DG_F(3, 4, 4, 4) DG_F(4, 4, 4, 4) DG_F(5, 8, 2, 2) DG_F(6, 2, 2, 1)
    DG_F(7, 2, 1, 1) DG_F(8, 2, 1, 1)
  }
#undef DG_F
  return inval("unsupported degree");
}

// number of CTAs (bricks) of the default Laplace configuration: the size of
// the kEpiDot partial-sum array
// below kSmallMesh cells (multigrid coarse levels) the v4 bricks replace the
// column kernel
constexpr int64_t kSmallMesh = 16384;

// Q3 meshes of at most 2048 cells run the v4 kernel with one cell per CTA:
// graph-replayed vmults at 4x2x2 / 8x4x4 / 16x8x8 cells take 4.6 / 4.7 / 5.1 us
// against 5.6 / 6.9 / 6.9 us with 4x4x2 bricks (profiles/r02/small_ab.py)
static bool tiny_q3(const dg_ctx *c) { return c->dim == 3 && c->n == 4 && c->n_cells <= 2048; }

static int64_t laplace_bricks(const dg_ctx *c) {
  if (tiny_q3(c)) return c->n_cells;
  int bx = 0, by = 0, bz = 1;
  if (c->dim == 3) {
    static const int B[9][3] = {{0, 0, 0}, {0, 0, 0}, {8, 4, 4}, {4, 4, 4}, {4, 4, 2},
                                {4, 2, 2}, {2, 2, 1}, {2, 1, 1}, {2, 1, 1}};
    bx = B[c->n][0]; by = B[c->n][1]; bz = B[c->n][2];
  } else {
    static const int B[9][2] = {{0, 0}, {0, 0}, {16, 16}, {16, 8}, {16, 8}, {8, 8}, {8, 8}, {8, 8}, {8, 8}};
    bx = B[c->n][0]; by = B[c->n][1];
  }
  return (int64_t)((c->counts[0] + bx - 1) / bx) * ((c->counts[1] + by - 1) / by) *
         ((c->counts[2] + bz - 1) / bz);
}

template <int N, int BX, int BY, int BZ, int EPI = kEpiStore>
static int launch_laplace6(dg_ctx *c, const double *src, double *dst, double tau_scale, int part,
                           cudaStream_t st, const EpiArgs &ea = EpiArgs{});

// fused-epilogue vmults for the CG / Chebyshev loop (default bricks, k = 2..5)
template <int N, int TX, int TY, int NRING, int MINB, int EPI = kEpiStore, int HSM = 0, int HMAP = 0, int FSD = 0, int UBC = 0>
static int launch_laplace8(dg_ctx *c, const double *src, double *dst, double tau_scale, int part,
                           cudaStream_t st, const EpiArgs &ea = EpiArgs{});

template <int N, int TX, int TY, int NRING, int MINB, bool STAGE = false, int EPI = kEpiStore, int HSPL = 0>
static int launch_laplace7(dg_ctx *c, const double *src, double *dst, double tau_scale, int part,
                           cudaStream_t st, const EpiArgs &ea = EpiArgs{});

static int laplace_dispatch_epi(dg_ctx *c, const double *src, double *dst, double tau_scale,
                                int epi, const EpiArgs &ea, cudaStream_t st) {
  c->epi_nparts = laplace_bricks(c);
  // Column-kernel cooperative epilogues (DG_EPI_COL: unset = Q4 only, 1 = also
  // Q3, 0 = never).  Q4: laplace8 with the halo in shared memory (HSM) beats
  // the v4 bricks: C2 Chebyshev-Jacobi PCG 0.537 vs 0.571 ms per iteration
  // (before HSM 0.62 vs 0.57, profiles/r02/cheb_time.py)
  static const int col = getenv("DG_EPI_COL") ? atoi(getenv("DG_EPI_COL")) : -1;
  if (col != 0 && c->dim == 3 && c->n == 5 && c->n_cells >= 16384 && c->mode[0] != kGhost &&
      c->mode[1] != kGhost) {
    // (HSM 1 here: C2 0.535 / 0.537 ms per iteration vs 0.549 with HSM 2)
    const char *ec = getenv("DG_EPI_CFG");  // read per call: A/B
    const int ecfg = ec ? atoi(ec) : 0;
    if (ecfg == 1) {
      if (epi == kEpiCheb) return launch_laplace8<5, 4, 8, 3, 1, kEpiCheb, 1, 1>(c, src, dst, tau_scale, 0, st, ea);
      if (epi == kEpiDot) return launch_laplace8<5, 4, 8, 3, 1, kEpiDot, 1, 1>(c, src, dst, tau_scale, 0, st, ea);
    }
    if (ecfg == 2) {
      if (epi == kEpiCheb) return launch_laplace8<5, 4, 8, 3, 1, kEpiCheb, 2, 1>(c, src, dst, tau_scale, 0, st, ea);
      if (epi == kEpiDot) return launch_laplace8<5, 4, 8, 3, 1, kEpiDot, 2, 1>(c, src, dst, tau_scale, 0, st, ea);
    }
    // Chebyshev epilogue with d from the shared-memory copy (UBC); DG_EPI_CFG=4: re-read
    if (epi == kEpiCheb && ecfg == 5)
      return launch_laplace8<5, 4, 8, 3, 1, kEpiCheb, 2, 1, 1, 1>(c, src, dst, tau_scale, 0, st, ea);
    // (C2 PCG, ms per iteration: 8x4 ring 3 + UBC 0.479, ring 3 0.494, ring 4 0.501,
    // 4x8 ring 3 HSM 2 + UBC 0.540; profiles/r02/cmd_s6e.sh)
    if (epi == kEpiCheb && ecfg == 7)
      return launch_laplace8<5, 8, 4, 3, 1, kEpiCheb, 1, 1>(c, src, dst, tau_scale, 0, st, ea);
    if (epi == kEpiCheb && ecfg == 6)
      return launch_laplace8<5, 8, 4, 3, 1, kEpiCheb, 1, 1, 0, 1>(c, src, dst, tau_scale, 0, st, ea);
    // default: + per-cell / per-layer side coefficients (FSD): 0.479 -> 0.475 (cmd_s6p.sh)
    if (epi == kEpiCheb && ecfg != 4)
      return launch_laplace8<5, 8, 4, 3, 1, kEpiCheb, 1, 1, 1, 1>(c, src, dst, tau_scale, 0, st, ea);
    if (epi == kEpiCheb) return launch_laplace8<5, 8, 4, 4, 1, kEpiCheb, 1, 1>(c, src, dst, tau_scale, 0, st, ea);
    // the dot epilogue from the shared-memory copy of u (kEpiDotS: out by TMA
    // stores, no global re-read of u); DG_EPI_CFG=3: the cooperative one
    if (epi == kEpiDot && ecfg != 3)
      return launch_laplace8<5, 4, 8, 3, 1, kEpiDotS, 2, 1, 1>(c, src, dst, tau_scale, 0, st, ea);
    if (epi == kEpiDot) return launch_laplace8<5, 8, 4, 4, 1, kEpiDot, 1, 1>(c, src, dst, tau_scale, 0, st, ea);
  }
#define DG_E(D, NN, X, Y, Z)                                                                     \
  if (c->dim == D && c->n == NN) {                                                               \
    if (epi == kEpiCheb) return launch_laplace<D, NN, X, Y, Z, kEpiCheb>(c, src, dst, tau_scale, 0, st, ea); \
    if (epi == kEpiDot) return launch_laplace<D, NN, X, Y, Z, kEpiDot>(c, src, dst, tau_scale, 0, st, ea);   \
  }
  // v4 bricks here also for k = 4: its 416-thread CTAs stream the CG vectors of
  // the epilogue faster than the 96-thread register-plane CTAs
  if (tiny_q3(c)) {
    if (epi == kEpiCheb) return launch_laplace<3, 4, 1, 1, 1, kEpiCheb>(c, src, dst, tau_scale, 0, st, ea);
    if (epi == kEpiDot) return launch_laplace<3, 4, 1, 1, 1, kEpiDot>(c, src, dst, tau_scale, 0, st, ea);
  }
  // DG_EPI_COL=1 at Q3: the column kernel's Chebyshev epilogue (laplace7, 4
  // CTAs/SM): 92.4 vs 88.5 us per step of the v4 bricks on the C4 fine level
  // (112.5 vs 106.2 with the split halo) -- the CTAs' sweep and epilogue
  // phases stay aligned, little overlap
  if (col == 1 && epi == kEpiCheb && c->dim == 3 && c->n == 4 && c->n_cells >= kSmallMesh &&
      c->mode[0] != kGhost && c->mode[1] != kGhost)
    return launch_laplace7<4, 4, 4, 4, 4, false, kEpiCheb, 1>(c, src, dst, tau_scale, 0, st, ea);
  DG_E(3, 3, 4, 4, 4) DG_E(3, 4, 4, 4, 2) DG_E(3, 5, 4, 2, 2) DG_E(3, 6, 2, 2, 1)
  DG_E(2, 3, 16, 8, 1) DG_E(2, 4, 16, 8, 1) DG_E(2, 5, 8, 8, 1) DG_E(2, 6, 8, 8, 1)
#undef DG_E
  return DG_ENOTSUP;
}

template <int N, int BX, int BY, int BZ, int EPI>
static int launch_laplace6(dg_ctx *c, const double *src, double *dst, double tau_scale, int part,
                           cudaStream_t st, const EpiArgs &ea) {
  if (t_kname) {
    *t_kname = kname("laplace6_kernel", {N, BX, BY, BZ, EPI});
    return DG_OK;
  }
  using C = Lap6Cfg<N, BX, BY, BZ>;
  auto kern = laplace6_kernel<N, BX, BY, BZ, EPI>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr = true;
  }
  if (c->dim == 3 && ensure_cell_table(c, st) != DG_OK) return DG_ECUDA;
  Geo g = c->geo();
  const dim3 grid((g.nx + BX - 1) / BX, (g.ny + BY - 1) / BY, chunk_bricks_z(c, BZ, g));
  kern<<<grid, C::THREADS, C::SMEM, st>>>(src, dst, g, lap_tab<N>(c->basis), tau_scale, part, ea);
  DG_LAUNCH_CHECK("laplace6_kernel");
  return DG_OK;
}

// shortest z-chunk of the column kernels: each chunk re-reads the layers
// below and above it, so short chunks only pay on meshes too small to fill
// the GPU otherwise (DG_L7_LCMIN: experiments)
static int l7_lcmin(int dflt) {
  const char *e = getenv("DG_L7_LCMIN");
  return e ? std::max(1, atoi(e)) : dflt;
}

// z-chunk length of the column kernels: the lc in [lcmin, lcmax] with the
// smallest makespan of a list-scheduling model of the launch (below; ties:
// longer chunks).  History: the first rule was about 4 waves, lc = nz /
// ceil(4 slots / cols) (DG_CHUNK_OLD=1, per call, for A/B) -- at one CTA per
// SM it left a part-filled last wave on the x-slab sizes (64x128x128 Q4: 768
// CTAs = 5.2 waves); then a wave model, waves x (lc + 2) (DG_CHUNK_MODEL=0;
// 1.24 -> 1.10 ms there, profiles/r02/chunk_ab.py), which at several CTAs
// per SM measured worse than the rule (64^3 Q3 0.163 -> 0.180 ms: few long
// chunks); with several CTAs per SM the 4-wave length is therefore the upper
// bound of the search.
static int chunk_len(int nz, int cols, int slots, int occ, int lcmin, int lcmax) {
  lcmax = std::max(1, std::min(nz, lcmax));
  lcmin = std::max(1, std::min(lcmin, lcmax));
  const char *cm = getenv("DG_CHUNK_MODEL");  // 0: the wave model (A/B, read per call)
  if (occ > 1 || getenv("DG_CHUNK_OLD")) {
    const int want = (4 * slots + cols - 1) / cols;
    const int lc4 = std::min(std::max(lcmin, (nz + want - 1) / want), lcmax);
    // several CTAs per SM: the list model below with chunks no longer than
    // the 4-wave rule's (never slower; 128^3 Q3 +7.1 %, 64^3 Q5 +6.0 %, 96^3
    // Q5 +2.0 %, profiles/r02/chunk_occ_ab.py); DG_CHUNK_MODEL=0: the rule
    if ((cm && atoi(cm) == 0) || getenv("DG_CHUNK_OLD")) return lc4;
    lcmax = lc4;
  }
  if (cm && atoi(cm) == 0) {
    int best = lcmax;
    double best_t = 1e300;
    for (int lc = lcmax; lc >= lcmin; --lc) {
      const int64_t nch = (nz + lc - 1) / lc;
      const int64_t waves = ((int64_t)cols * nch + slots - 1) / slots;
      const double t = (double)waves * (lc + 2.0);
      if (t < best_t - 1e-9) {
        best_t = t;
        best = lc;
      }
    }
    return best;
  }
  // List-scheduling model: the CTAs start in blockIdx order (chunk-major: all
  // columns of chunk 0, of chunk 1, ...; the LAST chunk of a column is the
  // short one, nz - (nch - 1) lc layers), each on the slot that frees first,
  // and take their layer count + 2.  The makespan of that schedule, not the
  // wave count, is what the launch costs: a short last chunk fills the slots
  // the long chunks leave idle (x-slab of P = 8, 64 columns x 128 layers on
  // 148 SMs: lc = 58 -> 128 CTAs of 58 layers + 64 of 12 layers, makespan 60
  // instead of 66 for 2 x 64).  Cached per argument tuple.
  struct Key {
    int nz, cols, slots, lcmin, lcmax;
    bool operator<(const Key &o) const {
      return std::tie(nz, cols, slots, lcmin, lcmax) < std::tie(o.nz, o.cols, o.slots, o.lcmin, o.lcmax);
    }
  };
  static std::map<Key, int> cache;
  static std::mutex mu;
  const Key key{nz, cols, slots, lcmin, lcmax};
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int best = lcmax;
  double best_t = 1e300;
  std::vector<double> heap;
  for (int lc = lcmax; lc >= lcmin; --lc) {
    const int nch = (nz + lc - 1) / lc;
    const int last = nz - (nch - 1) * lc;
    double t;
    if ((int64_t)cols * nch <= slots) {
      t = lc + 2.0;
    } else {
      heap.assign((size_t)slots, 0.0);  // min-heap of slot free times
      auto cmp = [](double a, double b) { return a > b; };
      double end = 0.0;
      for (int ch = 0; ch < nch; ++ch) {
        const double d = (ch == nch - 1 ? last : lc) + 2.0;
        for (int j = 0; j < cols; ++j) {
          std::pop_heap(heap.begin(), heap.end(), cmp);
          const double f = heap.back() + d;
          heap.back() = f;
          std::push_heap(heap.begin(), heap.end(), cmp);
          if (f > end) end = f;
        }
      }
      t = end;
    }
    if (t < best_t - 1e-9) {
      best_t = t;
      best = lc;
    }
  }
  cache[key] = best;
  return best;
}

// z-marching column kernel (laplace7.cuh): units = TX x TY tiles x z-chunks,
// the chunk length chosen so that ~4 waves of CTAs fill the GPU
template <int N, int TX, int TY, int NRING, int MINB, bool STAGE, int EPI, int HSPL>
static int launch_laplace7(dg_ctx *c, const double *src, double *dst, double tau_scale, int part,
                           cudaStream_t st, const EpiArgs &ea) {
  if (t_kname) {
    *t_kname = HSPL ? kname("laplace7_kernel", {N, TX, TY, NRING, MINB, (int)STAGE, EPI, HSPL})
                    : kname("laplace7_kernel", {N, TX, TY, NRING, MINB, (int)STAGE, EPI});
    return DG_OK;
  }
  using C = Lap7Cfg<N, TX, TY, NRING>;
  auto kern = laplace7_kernel<N, TX, TY, NRING, MINB, STAGE, EPI, HSPL>;
  static int nsm = 0, occ = 1;
  if (!nsm) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    int dev = 0;
    DG_CUDA_CHECK(cudaGetDevice(&dev));
    DG_CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    DG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM));
    if (occ < 1) occ = 1;
  }
  const Geo g = c->geo();
  int zlo = 0, zhi = g.nz;
  if (t_chunk.z1 > 0) {
    zlo = t_chunk.z0;
    zhi = t_chunk.z1;
  }
  const int ntx = (g.nx + TX - 1) / TX, nty = (g.ny + TY - 1) / TY;
  const int cols = ntx * nty, nz = zhi - zlo;
  // chunks >= 4 layers (measured: 32^3 Q3 54 -> 78 GDoF/s)
  const int lc = chunk_len(nz, cols, nsm * occ, occ, l7_lcmin(4), C::LCMAX);
  const int nch = (nz + lc - 1) / lc;
  kern<<<(unsigned)(cols * nch), C::THREADS, C::SMEM, st>>>(src, dst, g, lap_tab<N>(c->basis),
                                                            tau_scale, part, zlo, zhi, lc, ntx, nty,
                                                            ea);
  DG_LAUNCH_CHECK("laplace7_kernel");
  return DG_OK;
}

// half-plane column kernel (laplace8.cuh)
template <int N, int TX, int TY, int NRING, int MINB, int EPI, int HSM, int HMAP, int FSD, int UBC>
static int launch_laplace8(dg_ctx *c, const double *src, double *dst, double tau_scale, int part,
                           cudaStream_t st, const EpiArgs &ea) {
  if (t_kname) {
    // (FSD / UBC builds: all ten arguments, as ncu prints the instantiation)
    *t_kname = (UBC || FSD) ? kname("laplace8_kernel", {N, TX, TY, NRING, MINB, EPI, HSM, HMAP, FSD, UBC})
               : (HSM || HMAP) ? kname("laplace8_kernel", {N, TX, TY, NRING, MINB, EPI, HSM, HMAP})
                             : kname("laplace8_kernel", {N, TX, TY, NRING, MINB, EPI});
    return DG_OK;
  }
  using C = Lap8Cfg<N, TX, TY, NRING, HSM>;
  auto kern = laplace8_kernel<N, TX, TY, NRING, MINB, EPI, HSM, HMAP, FSD, UBC>;
  constexpr size_t kSmem = (EPI == kEpiDotS || UBC) ? C::SMEM_DOTS : C::SMEM;
  static_assert(kSmem <= 232448, "laplace8: more than 227 KB of shared memory");
  static int nsm = 0, occ = 1;
  if (!nsm) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    int dev = 0;
    DG_CUDA_CHECK(cudaGetDevice(&dev));
    DG_CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    DG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, kSmem));
    if (occ < 1) occ = 1;
  }
  const Geo g = c->geo();
  int zlo = 0, zhi = g.nz;
  if (t_chunk.z1 > 0) {
    zlo = t_chunk.z0;
    zhi = t_chunk.z1;
  }
  const int ntx = (g.nx + TX - 1) / TX, nty = (g.ny + TY - 1) / TY;
  const int cols = ntx * nty, nz = zhi - zlo;
  const int lc = chunk_len(nz, cols, nsm * occ, occ, l7_lcmin(8), C::LCMAX);
  const int nch = (nz + lc - 1) / lc;
  if (EPI == kEpiDot || EPI == kEpiDotS) {
    if (4 * (int64_t)cols * nch > c->partials_n) return inval("laplace8 epilogue: partials buffer");
    c->epi_nparts = (int64_t)cols * nch;
  }
  kern<<<(unsigned)(cols * nch), C::THREADS, kSmem, st>>>(src, dst, g, lap_tab<N>(c->basis),
                                                            tau_scale, part, zlo, zhi, lc, ntx, nty,
                                                            ea);
  DG_LAUNCH_CHECK("laplace8_kernel");
  return DG_OK;
}

// warp-column kernel (laplace9.cuh): persistent CTAs, warps pull units
// (tile x z-chunk) from a counter reset before the launch
template <int N, int TX, int TY, int NRING, int WPB>
static int launch_laplace9(dg_ctx *c, const double *src, double *dst, double tau_scale, int part,
                           cudaStream_t st) {
  if (t_kname) {
    *t_kname = kname("laplace9_kernel", {N, TX, TY, NRING, WPB});
    return DG_OK;
  }
  using C = Lap9Cfg<N, TX, TY, NRING, WPB>;
  auto kern = laplace9_kernel<N, TX, TY, NRING, WPB>;
  static int nsm = 0, occ = 1;
  if (!nsm) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    int dev = 0;
    DG_CUDA_CHECK(cudaGetDevice(&dev));
    DG_CUDA_CHECK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    DG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM));
    if (occ < 1) occ = 1;
  }
  if (!c->d_counter) DG_CUDA_CHECK(cudaMalloc((void **)&c->d_counter, 64));
  const Geo g = c->geo();
  int zlo = 0, zhi = g.nz;
  if (t_chunk.z1 > 0) {
    zlo = t_chunk.z0;
    zhi = t_chunk.z1;
  }
  const int ntx = (g.nx + TX - 1) / TX, nty = (g.ny + TY - 1) / TY;
  const int cols = ntx * nty, nz = zhi - zlo;
  const int warps = nsm * occ * WPB;
  const int want = (4 * warps + cols - 1) / cols;  // ~4 units per warp
  int lc = std::max(4, (nz + want - 1) / want);
  lc = std::min(std::min(lc, nz), C::LCMAX);
  const int nch = (nz + lc - 1) / lc;
  const int nunits = cols * nch;
  const int grid = std::min(nsm * occ, (nunits + WPB - 1) / WPB);
  DG_CUDA_CHECK(cudaMemsetAsync(c->d_counter, 0, sizeof(unsigned), st));
  kern<<<(unsigned)grid, C::THREADS, C::SMEM, st>>>(src, dst, g, lap_tab<N>(c->basis), tau_scale,
                                                    part, zlo, zhi, lc, ntx, nty, nunits,
                                                    c->d_counter);
  DG_LAUNCH_CHECK("laplace9_kernel");
  return DG_OK;
}

// tile / ring configuration of the column kernel (DG_L7CFG: experiments)
static int l7_cfg() {
  const char *e = getenv("DG_L7CFG");  // read per call: A/B within one process
  return e ? atoi(e) : 0;
}

static int laplace_dispatch(dg_ctx *c, const double *src, double *dst, double tau_scale, int part,
                            cudaStream_t st) {
  // DG_LAP_VARIANT (read per call, A/B experiments): 4 = v4 bricks, 6 = the
  // round-1 register-plane bricks, 7 = column kernel with tile config DG_L7CFG
  const char *vv = getenv("DG_LAP_VARIANT");
  int variant = vv ? atoi(vv) : 0;
  // ghost layers in the trace format are read by the column kernels only
  if (c->halo_traces && (c->mode[0] == kGhost || c->mode[1] == kGhost) && variant != 7 && variant != 8 &&
      variant != 9)
    variant = 0;
  if (c->dim == 3 && variant == 9) {
    const int cfg = l7_cfg();
    if (c->n == 4) {
      if (cfg == 1) return launch_laplace9<4, 2, 4, 3, 6>(c, src, dst, tau_scale, part, st);
      return launch_laplace9<4, 2, 4, 2, 8>(c, src, dst, tau_scale, part, st);
    }
    if (c->n == 5) {
      if (cfg == 1) return launch_laplace9<5, 2, 3, 3, 6>(c, src, dst, tau_scale, part, st);
      return launch_laplace9<5, 2, 3, 2, 8>(c, src, dst, tau_scale, part, st);
    }
  }
  if (c->dim == 3 && variant == 8) {
    const int cfg = l7_cfg();
    if (c->n == 4) {
      if (cfg == 1) return launch_laplace8<4, 4, 4, 4, 3>(c, src, dst, tau_scale, part, st);
      if (cfg == 2) return launch_laplace8<4, 8, 4, 3, 2>(c, src, dst, tau_scale, part, st);
      return launch_laplace8<4, 4, 4, 4, 4>(c, src, dst, tau_scale, part, st);
    }
    if (c->n == 5) {
      // round-2 session-3 A/B: 1 = halo in registers, round-robin halo items
      // (session 2), 2 = halo items staged per thread by cp.async, 3 = + HMAP
      if (cfg == 1) return launch_laplace8<5, 8, 4, 4, 1>(c, src, dst, tau_scale, part, st);
      if (cfg == 2) return launch_laplace8<5, 8, 4, 4, 1, kEpiStore, 1, 0>(c, src, dst, tau_scale, part, st);
      if (cfg == 3) return launch_laplace8<5, 8, 4, 4, 1, kEpiStore, 1, 1>(c, src, dst, tau_scale, part, st);
      // 4 / 5 / 6: 8x4 ring 3, 4x8 ring 4, 8x4 ring 4 (session-3 HSM 2 configurations)
      if (cfg == 4) return launch_laplace8<5, 8, 4, 3, 1, kEpiStore, 2, 1>(c, src, dst, tau_scale, part, st);
      if (cfg == 5) return launch_laplace8<5, 4, 8, 4, 1, kEpiStore, 2, 1>(c, src, dst, tau_scale, part, st);
      if (cfg == 6) return launch_laplace8<5, 8, 4, 4, 1, kEpiStore, 2, 1>(c, src, dst, tau_scale, part, st);
      if (cfg == 7) return launch_laplace8<5, 4, 8, 3, 1, kEpiStore, 2, 1, 1>(c, src, dst, tau_scale, part, st);
      if (cfg == 8) return launch_laplace8<5, 4, 8, 3, 1, kEpiStore, 2, 1>(c, src, dst, tau_scale, part, st);
      return launch_laplace8<5, 4, 8, 3, 1, kEpiStore, 2, 1, 1>(c, src, dst, tau_scale, part, st);
    }
    if (c->n == 6) return launch_laplace8<6, 4, 4, 2, 2>(c, src, dst, tau_scale, part, st);
  }
  if (c->dim == 3 && variant == 7) {
    const int cfg = l7_cfg();
    if (c->n == 4) {
      if (cfg == 1) return launch_laplace7<4, 8, 4, 3, 2>(c, src, dst, tau_scale, part, st);
      if (cfg == 2) return launch_laplace7<4, 4, 4, 3, 5>(c, src, dst, tau_scale, part, st);
    }
    if (c->n == 5) {
      if (cfg == 1) return launch_laplace7<5, 8, 4, 4, 1>(c, src, dst, tau_scale, part, st);
      if (cfg == 2) return launch_laplace7<5, 4, 4, 3, 2>(c, src, dst, tau_scale, part, st);
      if (cfg == 3) return launch_laplace7<5, 8, 4, 3, 1>(c, src, dst, tau_scale, part, st);
      if (cfg == 4) return launch_laplace7<5, 4, 4, 4, 2>(c, src, dst, tau_scale, part, st);
    }
    if (c->n == 6 && cfg == 1) return launch_laplace7<6, 4, 4, 3, 1>(c, src, dst, tau_scale, part, st);
    // halo rows in one piece (round-2 sessions 1-2 defaults): Q3 96^3 107.1,
    // Q5 64^3 76.7 GDoF/s vs 109.3 / 86.9 in two halves (3 or 6 parts: Q5 86.8 / 79.4)
    if (c->n == 6 && cfg == 3) return launch_laplace7<6, 4, 4, 2, 2>(c, src, dst, tau_scale, part, st);
    if (c->n == 4 && cfg == 3) return launch_laplace7<4, 4, 4, 4, 4>(c, src, dst, tau_scale, part, st);
    if (c->n == 3) return launch_laplace7<3, 8, 4, 3, 2>(c, src, dst, tau_scale, part, st);
  }
  // default 3D Q3-Q5: the z-marching column kernel (laplace7.cuh); tile, ring
  // depth and CTAs/SM measured per degree (profiles/r02/NOTES.md)
  // small meshes (multigrid coarse levels): the column kernel's z march is a
  // serial chain per CTA (a 16x8x8 level takes ~20 us at any tile), the v4
  // bricks run all bricks at once (~9 us; profiles/r02/NOTES.md)
  const bool traced = c->halo_traces && (c->mode[0] == kGhost || c->mode[1] == kGhost);
  if (c->dim == 3 && variant == 0 && !traced && c->n_cells < kSmallMesh) variant = 4;
  if (c->dim == 3 && variant != 4 && variant != 6) {
    // Q3 / Q5: halo item rows loaded in two halves (HSPL; Q5 spills 288 -> 176 B)
    if (c->n == 4) return launch_laplace7<4, 4, 4, 4, 4, false, kEpiStore, 1>(c, src, dst, tau_scale, part, st);
    // Q4: the half-plane variant (laplace8.cuh, 8x4 tile, 10 warps) -- +3..7 %
    // over laplace7<5,4,4,4,2> from 48^3 to 160^3 (profiles/r02/NOTES.md)
    // (x-slabs too: 4x8 tiles measured slower at every P, profiles/r02/slab_parts.py);
    // halo cells staged in shared memory (HSM: no halo registers, no spills;
    // HSM 2: whole cells copied by coalesced warp-wide cp.async from a per-CTA
    // source table) and halo work placed per SM sub-partition (HMAP); per-layer
    // set-up hoisted: 120.8 -> 133.7 GDoF/s at 128^3; 4x8 tile, ring 3: 136.3
    // (+1.6-1.9 % at 64^3-160^3 and on the x-slabs of P = 1-8; profiles/r02/NOTES.md)
    // x / y side coefficients per cell precomputed with the kinds folded in (FSD): +1 %
    if (c->n == 5) return launch_laplace8<5, 4, 8, 3, 1, kEpiStore, 2, 1, 1>(c, src, dst, tau_scale, part, st);
    if (c->n == 6) return launch_laplace7<6, 4, 4, 2, 2, false, kEpiStore, 1>(c, src, dst, tau_scale, part, st);
  }
  if (c->dim == 3 && variant == 6 && c->n == 4)  // register-plane kernel at k = 3 (experiment)
    return launch_laplace6<4, 4, 2, 2>(c, src, dst, tau_scale, part, st);

  // tiny Q3 meshes (the coarsest multigrid levels): one cell per CTA
  if (tiny_q3(c) && variant == 4) return launch_laplace<3, 4, 1, 1, 1>(c, src, dst, tau_scale, part, st);
  if (c->dim == 3) {
    switch (c->n) {
      case 2: return launch_laplace<3, 2, 8, 4, 4>(c, src, dst, tau_scale, part, st);
      case 3:  // register-plane kernel (64^3 Q2: 69 vs 52 GDoF/s for the v4 bricks;
               // bricks 4x2x2 66, 8x4x2 65, 4x4x4 59)
        if (variant == 4) return launch_laplace<3, 3, 4, 4, 4>(c, src, dst, tau_scale, part, st);
        return launch_laplace6<3, 4, 4, 2>(c, src, dst, tau_scale, part, st);
      case 4: return launch_laplace<3, 4, 4, 4, 2>(c, src, dst, tau_scale, part, st);
      case 5:
        if (variant == 4) return launch_laplace<3, 5, 4, 2, 2>(c, src, dst, tau_scale, part, st);
        return launch_laplace6<5, 4, 2, 2>(c, src, dst, tau_scale, part, st);
      // k >= 5: flatter bricks (measured at 64^3: Q5 2x2x1 69 vs 2x2x2 62 GDoF/s,
      // Q6 2x1x1 62 vs 52, Q7 2x1x1 63 vs 57 at 48^3; profiles/NOTES.md)
      case 6: return launch_laplace<3, 6, 2, 2, 1>(c, src, dst, tau_scale, part, st);
      case 7: return launch_laplace<3, 7, 2, 1, 1>(c, src, dst, tau_scale, part, st);
      case 8: return launch_laplace<3, 8, 2, 1, 1>(c, src, dst, tau_scale, part, st);
    }
  } else {
    switch (c->n) {
      case 2: return launch_laplace<2, 2, 16, 16, 1>(c, src, dst, tau_scale, part, st);
      case 3: return launch_laplace<2, 3, 16, 8, 1>(c, src, dst, tau_scale, part, st);
      case 4: return launch_laplace<2, 4, 16, 8, 1>(c, src, dst, tau_scale, part, st);
      case 5: return launch_laplace<2, 5, 8, 8, 1>(c, src, dst, tau_scale, part, st);
      case 6: return launch_laplace<2, 6, 8, 8, 1>(c, src, dst, tau_scale, part, st);
      case 7: return launch_laplace<2, 7, 8, 8, 1>(c, src, dst, tau_scale, part, st);
      case 8: return launch_laplace<2, 8, 8, 8, 1>(c, src, dst, tau_scale, part, st);
    }
  }
  return inval("unsupported degree");
}

// ---------------------------------------------------------------------------
// element-wise helpers

// w_i = integral of the nodal basis function i: prod_d (h_d/2) wint[i_d]
struct WInt {
  double w[kMaxN];
};

// w: the 1D integrals staged in shared memory by the calling kernel
// (indexing the WInt kernel parameter per lane serialises the constant
// cache); 32-bit index math below 2^32 DoFs
__device__ __forceinline__ double dual_weight(const Geo &g, int dim, int n, const double *w,
                                              int64_t i) {
  int x, y, z, ix, iy, iz;
  if ((uint64_t)i < (1ull << 32)) {
    const unsigned np = (dim == 3) ? (unsigned)(n * n * n) : (unsigned)(n * n);
    const unsigned ui = (unsigned)i, e = ui / np;
    unsigned o = ui - e * np;
    x = (int)(o % (unsigned)n);
    o /= (unsigned)n;
    y = (int)(o % (unsigned)n);
    z = (dim == 3) ? (int)(o / (unsigned)n) : 0;
    const unsigned r = e / (unsigned)g.nx;
    ix = (int)(e - r * (unsigned)g.nx);
    iy = (int)(r % (unsigned)g.ny);
    iz = (int)(r / (unsigned)g.ny);
  } else {
    const int64_t np = (dim == 3) ? (int64_t)n * n * n : (int64_t)n * n;
    const int64_t e = i / np;
    int o = (int)(i % np);
    x = o % n;
    o /= n;
    y = o % n;
    z = (dim == 3) ? o / n : 0;
    ix = (int)(e % g.nx);
    const int64_t r = e / g.nx;
    iy = (int)(r % g.ny);
    iz = (int)(r / g.ny);
  }
  double v = 0.5 * g.hx[ix] * w[x] * 0.5 * g.hy[iy] * w[y];
  if (dim == 3) v *= 0.5 * g.hz[iz] * w[z];
  return v;
}

// stage the WInt parameter in shared memory (all threads; ends with a barrier)
#define DG_STAGE_WINT(sw, wi)                                     \
  __shared__ double sw[kMaxN];                                    \
  if (threadIdx.x < kMaxN) sw[threadIdx.x] = (wi).w[threadIdx.x]; \
  __syncthreads()

// face traces of the first (side 0: value, dL . line) or last (side 1:
// value, dR . line) x-layer: one thread per (cell (iy, iz), y, z), the x-line
// of that cell; out[cell][z][y][v|g] (the ghost layout of laplace7.cuh)
struct HaloTab {
  double dL[kMaxN], dR[kMaxN];
};
__global__ void halo_trace_kernel(const double *__restrict__ src, double *__restrict__ out,
                                  int nx, int n, int64_t items, int side, HaloTab t) {
  const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (it >= items) return;
  const int64_t nn = (int64_t)n * n;
  const int64_t cell = it / nn;  // iy + ny * iz
  const int zy = (int)(it - cell * nn), z = zy / n, y = zy - z * n;
  const int64_t e = (int64_t)(side ? nx - 1 : 0) + (int64_t)nx * cell;
  const double *l = src + e * nn * n + (int64_t)z * nn + (int64_t)y * n;
  double g = 0.0;
  for (int q = 0; q < n; ++q) g += (side ? t.dR[q] : t.dL[q]) * l[q];
  double *o = out + (cell * nn + (int64_t)z * n + y) * 2;
  o[0] = side ? l[n - 1] : l[0];
  o[1] = g;
}

__global__ void wdot_partial_kernel(const double *__restrict__ p, int64_t n, Geo g, int dim,
                                    int nn, WInt wi, double *__restrict__ partial) {
  __shared__ double sh[32];
  DG_STAGE_WINT(sw, wi);
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    acc += p[i] * dual_weight(g, dim, nn, sw, i);
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// b_i -= (s / vol) * w_i   (mode 0, dual projection)   or   p_i -= s / vol (mode 1)
__global__ void zero_mean_apply_kernel(double *__restrict__ b, int64_t n, Geo g, int dim, int nn,
                                       WInt wi, const double *__restrict__ s, double vol,
                                       int mode) {
  DG_STAGE_WINT(sw, wi);
  const double coef = __ddiv_rn(*s, vol);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (mode == 0) b[i] = __dsub_rn(b[i], __dmul_rn(coef, dual_weight(g, dim, nn, sw, i)));
    else b[i] = __dsub_rn(b[i], coef);
  }
}

static WInt wint_of(const dg_ctx *c) {
  WInt w;
  for (int i = 0; i < kMaxN; ++i) w.w[i] = i < c->n ? c->basis.wint[i] : 0.0;
  return w;
}

static int reduce_sum(dg_ctx *c, const double *x, const double *y, int64_t n, double *out,
                      cudaStream_t st) {
  dot_partial_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(x, y, n, c->d_red);
  sum_partials_kernel<<<1, 1024, 0, st>>>(c->d_red, kRedBlocks, out);
  DG_LAUNCH_CHECK("dot");
  return DG_OK;
}

static int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

extern "C" {

int dg_laplace_vmult(dg_ctx *c, const double *src, double *dst, double tau_scale, void *stream) {
  if (!c || !src || !dst) return inval("null argument");
  if ((c->mode[0] == kGhost && !c->d_recv[0]) || (c->mode[1] == kGhost && !c->d_recv[1]))
    return inval("x-slab context: attach ghost layers (dg_halo_attach) first");
  return laplace_dispatch(c, src, dst, tau_scale, 0, (cudaStream_t)stream);
}

// apply_pressure_laplace on HOST buffers (pinned for overlap): the mesh is
// cut into z-chunks of whole x-y layers (contiguous in the element-major
// layout); host->device copies of chunk i+1, the vmult of chunk i and the
// device->host copy of chunk i-1 run on three streams, so the two PCIe
// directions and the kernel overlap.  A chunk's vmult waits for the copies of
// its z-neighbour chunks (its halo).
int dg_laplace_vmult_host(dg_ctx *c, const double *src_host, double *dst_host, double tau_scale,
                          int n_chunks, void *stream) {
  if (!c || !src_host || !dst_host) return inval("null argument");
  if (c->mode[0] == kGhost || c->mode[1] == kGhost)
    return inval("host-buffer vmult runs on whole-mesh contexts");
  std::lock_guard<std::mutex> lock(c->mu);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = c->n_dofs;
  if (!c->d_hin) {
    DG_CUDA_CHECK(cudaMalloc((void **)&c->d_hin, sizeof(double) * (n > 0 ? n : 1)));
    DG_CUDA_CHECK(cudaMalloc((void **)&c->d_hout, sizeof(double) * (n > 0 ? n : 1)));
    DG_CUDA_CHECK(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    DG_CUDA_CHECK(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
  }
  static const bool variant = getenv("DG_LAP_VARIANT") && atoi(getenv("DG_LAP_VARIANT")) != 0;
  const int nz = c->counts[2];
  int nch = (c->dim == 3 && !variant) ? n_chunks : 1;
  if (nch < 1) nch = 1;
  int layers = (nz + nch - 1) / nch;
  layers = ((layers + 3) / 4) * 4;  // chunk boundaries on multiples of 4 (brick heights)
  nch = (nz + layers - 1) / layers;
  const int64_t per_layer = (int64_t)c->counts[0] * c->counts[1] * c->np;
  std::vector<cudaEvent_t> eh(nch), ec(nch);
  for (int i = 0; i < nch; ++i) {
    DG_CUDA_CHECK(cudaEventCreateWithFlags(&eh[i], cudaEventDisableTiming));
    DG_CUDA_CHECK(cudaEventCreateWithFlags(&ec[i], cudaEventDisableTiming));
  }
  cudaEvent_t start, done;
  DG_CUDA_CHECK(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  DG_CUDA_CHECK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  DG_CUDA_CHECK(cudaEventRecord(start, st));  // order after prior work on the caller's stream
  DG_CUDA_CHECK(cudaStreamWaitEvent(c->s_h2d, start, 0));
  int rc = DG_OK;
  for (int i = 0; i < nch; ++i) {
    const int z0 = i * layers, z1 = std::min(nz, z0 + layers);
    const int64_t off = z0 * per_layer, cnt = (int64_t)(z1 - z0) * per_layer;
    DG_CUDA_CHECK(cudaMemcpyAsync(c->d_hin + off, src_host + off, sizeof(double) * cnt,
                                  cudaMemcpyHostToDevice, c->s_h2d));
    DG_CUDA_CHECK(cudaEventRecord(eh[i], c->s_h2d));
  }
  const bool zper = c->mode[4] == kWrap;
  for (int i = 0; i < nch && rc == DG_OK; ++i) {
    DG_CUDA_CHECK(cudaStreamWaitEvent(st, eh[std::min(i + 1, nch - 1)], 0));
    if (zper && i == 0) DG_CUDA_CHECK(cudaStreamWaitEvent(st, eh[nch - 1], 0));
    t_chunk.z0 = i * layers;
    t_chunk.z1 = nch > 1 ? std::min(nz, t_chunk.z0 + layers) : 0;
    rc = laplace_dispatch(c, c->d_hin, c->d_hout, tau_scale, 0, st);
    t_chunk = ZChunk{};
    if (rc) break;
    DG_CUDA_CHECK(cudaEventRecord(ec[i], st));
    DG_CUDA_CHECK(cudaStreamWaitEvent(c->s_d2h, ec[i], 0));
    const int z0 = i * layers, z1 = std::min(nz, z0 + layers);
    const int64_t off = z0 * per_layer, cnt = (int64_t)(z1 - z0) * per_layer;
    DG_CUDA_CHECK(cudaMemcpyAsync(dst_host + off, c->d_hout + off, sizeof(double) * cnt,
                                  cudaMemcpyDeviceToHost, c->s_d2h));
  }
  DG_CUDA_CHECK(cudaEventRecord(done, c->s_d2h));
  DG_CUDA_CHECK(cudaStreamWaitEvent(st, done, 0));  // the caller's stream sees the result
  for (int i = 0; i < nch; ++i) {
    cudaEventDestroy(eh[i]);
    cudaEventDestroy(ec[i]);
  }
  cudaEventDestroy(start);
  cudaEventDestroy(done);
  return rc;
}

int dg_laplace_vmult_part(dg_ctx *c, const double *src, double *dst, double tau_scale, int part,
                          void *stream) {
  if (!c || !src || !dst) return inval("null argument");
  if (part < 0 || part > 2) return inval("part must be 0, 1 or 2");
  if (part != 1 &&
      ((c->mode[0] == kGhost && !c->d_recv[0]) || (c->mode[1] == kGhost && !c->d_recv[1])))
    return inval("x-slab context: attach ghost layers (dg_halo_attach) first");
  return laplace_dispatch(c, src, dst, tau_scale, part, (cudaStream_t)stream);
}

int dg_laplace_kernel_name(dg_ctx *c, char *buf, int len) {
  if (!c || !buf || len < 1) return inval("null argument");
  std::string name;
  t_kname = &name;
  const int rc = laplace_dispatch(c, nullptr, nullptr, 1.0, 0, nullptr);
  t_kname = nullptr;
  if (rc) return rc;
  std::snprintf(buf, (size_t)len, "%s", name.c_str());
  return DG_OK;
}

int dg_dot(dg_ctx *c, const double *x, const double *y, int64_t n, double *out_dev,
           void *stream) {
  if (!c || !x || !out_dev) return inval("null argument");
  return reduce_sum(c, x, y, n, out_dev, (cudaStream_t)stream);
}

int dg_zero_mean_dual(dg_ctx *c, double *b, void *stream) {
  if (!c || !b) return inval("null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = reduce_sum(c, b, nullptr, c->n_dofs, c->d_scal + 8, st);
  if (rc) return rc;
  zero_mean_apply_kernel<<<grid_for(c->n_dofs), 256, 0, st>>>(b, c->n_dofs, c->geo(), c->dim, c->n,
                                                               wint_of(c), c->d_scal + 8, c->volume, 0);
  DG_LAUNCH_CHECK("zero_mean_dual");
  return DG_OK;
}

int dg_zero_mean(dg_ctx *c, double *p, void *stream) {
  if (!c || !p) return inval("null argument");
  cudaStream_t st = (cudaStream_t)stream;
  wdot_partial_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(p, c->n_dofs, c->geo(), c->dim, c->n,
                                                          wint_of(c), c->d_red);
  sum_partials_kernel<<<1, 1024, 0, st>>>(c->d_red, kRedBlocks, c->d_scal + 9);
  zero_mean_apply_kernel<<<grid_for(c->n_dofs), 256, 0, st>>>(p, c->n_dofs, c->geo(), c->dim, c->n,
                                                               wint_of(c), c->d_scal + 9, c->volume, 1);
  DG_LAUNCH_CHECK("zero_mean");
  return DG_OK;
}

int dg_halo_count(const dg_ctx *c, int64_t *count) {
  if (!c || !count) return inval("null argument");
  *count = c->halo_count;
  return DG_OK;
}

}  // extern "C"

// Ghost-face part of the x-slab vmult (dg_laplace_vmult_split phase 2): the
// SIP operator is linear in the ghost traces, so with phase 1 run on ZERO
// traces, out += the terms of the x-lifts of the column kernel
// (laplace8.cuh x phase, l7_lift) that carry the neighbour's data:
//   per face node (y, z): vn = (M z-mass) v_ghost, gn = (M) g_ghost,
//   cv = -A vn + D gn, cd = -B vn  (A, B, D of side7 for a halo side),
//   T[z][y][x] = delta(x, end) cv + dEnd[x] cd,  out += (M y-mass) T.
// One group of N*N threads per (boundary cell, side); both ghost sides in one
// launch (blockIdx.y, side0 + blockIdx.y; one launch instead of two: the
// x-slab rank of P = 8 spends 21 -> 1x us here).
// DOTS: also the partial sums of p . (added terms) and sum(added terms) per
// block -> partials[2 * block + {0, 1}] (dg_laplace_vmult_split_dots).
template <int N, bool DOTS = false>
__global__ void ghost_lift_kernel(const Geo g, const __grid_constant__ LapTab<N> T, double ts,
                                  int side0, double *__restrict__ out,
                                  const double *__restrict__ p = nullptr,
                                  double *__restrict__ partials = nullptr) {
  const int side = side0 + (int)blockIdx.y;
  constexpr int N2 = N * N, G = 128 / N2, NP = N * N2;
  __shared__ double sv[G][N2], sg[G][N2], c1[G][N2], c2[G][N2];
  const int grp = threadIdx.x / N2, t = threadIdx.x - grp * N2;
  const int64_t cell = (int64_t)blockIdx.x * G + grp;  // (iy, iz) of the boundary layer
  const bool ok = grp < G && cell < (int64_t)g.ny * g.nz;
  const int iy = ok ? (int)(cell % g.ny) : 0, iz = ok ? (int)(cell / g.ny) : 0;
  const int ix = side ? g.nx - 1 : 0;
  const double *gh = g.ghost[side];
  // ghost payload [z][y][v|g] per boundary cell
  if (ok) {
    sv[grp][t] = gh[(cell * N2 + t) * 2];
    sg[grp][t] = gh[(cell * N2 + t) * 2 + 1];
  }
  __syncthreads();
  const double *ax = g.ax[0] + 4 * ix, *ay = g.ax[1] + 4 * iy, *az = g.ax[2] + 4 * iz;
  const double hxi = ax[1], tx = ax[2], hy = ay[0], ty = ay[2], hz = az[0], tz = az[2];
  const double *axn = ax + (side ? 4 : -4);  // the ghost cell's entry
  const double sfx = 0.25 * hy * hz;
  const double sgn = side ? -1.0 : 1.0;
  const double A = ts * ((fmax(tx, axn[2]) + ty + tz) * sfx);
  const double B = sgn * sfx * hxi, D = sgn * sfx * axn[1];
  if (ok) {  // thread (z, y): z-mass of the traces, the lift coefficients
    const int z = t / N, y = t - z * N;
    double vn = 0.0, gn = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      vn += T.M[z * N + q] * sv[grp][q * N + y];
      gn += T.M[z * N + q] * sg[grp][q * N + y];
    }
    c1[grp][t] = -A * vn + D * gn;
    c2[grp][t] = -B * vn;
  }
  __syncthreads();
  double a0 = 0.0, a1 = 0.0;
  if (ok) {  // thread (z, x): y-mass, add into the x-line ends / derivative rows
    const int z = t / N, x = t - z * N;
    const int end = side ? N - 1 : 0;
    const double dx = side ? T.dR[x] : T.dL[x];
    const int64_t o0 = ((int64_t)ix + (int64_t)g.nx * (iy + (int64_t)g.ny * iz)) * NP + z * N2 + x;
    double *o = out + o0;
#pragma unroll
    for (int y = 0; y < N; ++y) {
      double m1 = 0.0, m2 = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        m1 += T.M[y * N + q] * c1[grp][z * N + q];
        m2 += T.M[y * N + q] * c2[grp][z * N + q];
      }
      const double add = (x == end ? m1 : 0.0) + dx * m2;
      o[y * N] += add;
      if (DOTS) {
        a0 += p[o0 + y * N] * add;
        a1 += add;
      }
    }
  }
  if (DOTS) {  // fixed-order block sums (128 threads)
    __shared__ double red[2][4];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = a0;
      red[1][threadIdx.x >> 5] = a1;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
      const double *r = red[threadIdx.x];
      const size_t blk = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
      partials[2 * blk + threadIdx.x] = ((r[0] + r[1]) + r[2]) + r[3];
    }
  }
}

// out3[k] += sum_b partials[2 b + k], k < 2, fixed order (one block)
__global__ void add_partials2_kernel(const double *__restrict__ partials, int64_t nb,
                                     double *__restrict__ out3) {
  __shared__ double sh[32];
  for (int k = 0; k < 2; ++k) {
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < nb; i += blockDim.x) acc += partials[2 * i + k];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) out3[k] += acc;
    __syncthreads();
  }
}

extern "C" {

// x-slab vmult in two phases around the ghost exchange: phase 1 = the whole
// slab with ZERO ghost traces (one launch, no dependence on the exchange),
// phase 2 = out += the ghost-trace terms on the boundary x-layers
// (ghost_lift_kernel).  Traced-ghost contexts (3D, Q3-Q5).
static int vmult_split_impl(dg_ctx *c, const double *src, double *dst, double tau_scale, int phase,
                            void *stream, double *out3);

int dg_laplace_vmult_split(dg_ctx *c, const double *src, double *dst, double tau_scale,
                           int phase, void *stream) {
  return vmult_split_impl(c, src, dst, tau_scale, phase, stream, nullptr);
}

}  // extern "C"

// out3 != nullptr (dg_laplace_vmult_split_dots, slabcg.inc): the fused form,
// phase 1 = column kernel with the kEpiDotS sums on zero traces -> out3,
// phase 2 = ghost lifts with their share of p.Lp and sum(Lp) added to out3
static bool split_dots_fused(const dg_ctx *c);
static int split_phase1_dots(dg_ctx *c, const double *src, double *dst, double tau_scale,
                             cudaStream_t st, double *out3);
static int split_partials(dg_ctx *c, int64_t need);

static int vmult_split_impl(dg_ctx *c, const double *src, double *dst, double tau_scale, int phase,
                            void *stream, double *out3) {
  if (!c || !dst) return inval("null argument");
  if (phase != 1 && phase != 2) return inval("phase must be 1 or 2");
  if (!c->halo_traces || c->dim != 3) return inval("dg_laplace_vmult_split: traced-ghost 3D contexts");
  if ((c->mode[0] == kGhost && !c->d_recv[0]) || (c->mode[1] == kGhost && !c->d_recv[1]))
    return inval("x-slab context: attach ghost layers (dg_halo_attach) first");
  cudaStream_t st = (cudaStream_t)stream;
  if (phase == 1) {
    if (!src) return inval("null argument");
    if (!c->d_zero_ghost) {
      DG_CUDA_CHECK(cudaMalloc((void **)&c->d_zero_ghost, sizeof(double) * (size_t)std::max<int64_t>(c->halo_count, 1)));
      DG_CUDA_CHECK(cudaMemset(c->d_zero_ghost, 0, sizeof(double) * (size_t)std::max<int64_t>(c->halo_count, 1)));
    }
    const double *keep[2] = {c->d_recv[0], c->d_recv[1]};
    for (int s = 0; s < 2; ++s)
      if (c->mode[s] == kGhost) c->d_recv[s] = c->d_zero_ghost;
    const int rc = out3 ? split_phase1_dots(c, src, dst, tau_scale, st, out3)
                        : laplace_dispatch(c, src, dst, tau_scale, 0, st);
    c->d_recv[0] = keep[0];
    c->d_recv[1] = keep[1];
    return rc;
  }
  if (c->n_cells == 0) return DG_OK;
  const Geo g = c->geo();
  const bool lo = c->mode[0] == kGhost, hi = c->mode[1] == kGhost;
  if (lo || hi) {
    const int side0 = lo ? 0 : 1, nsides = (lo ? 1 : 0) + (hi ? 1 : 0);
    const int64_t cells = (int64_t)g.ny * g.nz;
    if (out3) {  // n == 5 (split_dots_fused): the lifts with their dot shares
      if (!src) return inval("null argument");
      constexpr int G = 128 / 25;
      const int64_t nb = (cells + G - 1) / G * nsides;
      const int rc = split_partials(c, 2 * nb);
      if (rc) return rc;
      ghost_lift_kernel<5, true><<<dim3((unsigned)((cells + G - 1) / G), (unsigned)nsides), 128, 0, st>>>(
          g, lap_tab<5>(c->basis), tau_scale, side0, dst, src, c->d_partials);
      add_partials2_kernel<<<1, 1024, 0, st>>>(c->d_partials, nb, out3);
      DG_LAUNCH_CHECK("ghost_lift_kernel (dots)");
      return DG_OK;
    }
#define DG_GL(NN)                                                                             \
  if (c->n == NN) {                                                                           \
    constexpr int G = 128 / (NN * NN);                                                        \
    ghost_lift_kernel<NN><<<dim3((unsigned)((cells + G - 1) / G), (unsigned)nsides), 128, 0, st>>>( \
        g, lap_tab<NN>(c->basis), tau_scale, side0, dst);                                     \
  }
    DG_GL(4) DG_GL(5) DG_GL(6)
#undef DG_GL
  }
  DG_LAUNCH_CHECK("ghost_lift_kernel");
  return DG_OK;
}

extern "C" {

int dg_halo_attach(dg_ctx *c, const double *recv_lo, const double *recv_hi) {
  if (!c) return inval("null context");
  if ((c->mode[0] == kGhost && !recv_lo) || (c->mode[1] == kGhost && !recv_hi))
    return inval("a remote side needs a ghost buffer");
  c->d_recv[0] = recv_lo;
  c->d_recv[1] = recv_hi;
  return DG_OK;
}

int dg_halo_pack(dg_ctx *c, const double *src, double *send_lo, double *send_hi, void *stream) {
  if (!c || !src) return inval("null argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (c->halo_traces) {  // owner-computed face traces of the first / last x-layer
    const int64_t items = (int64_t)c->counts[1] * c->counts[2] * c->n * c->n;
    HaloTab t;
    for (int i = 0; i < c->n; ++i) {
      t.dL[i] = c->basis.ld[i];
      t.dR[i] = c->basis.rd[i];
    }
    const unsigned gb = (unsigned)((items + 255) / 256);
    if (send_lo) halo_trace_kernel<<<gb, 256, 0, st>>>(src, send_lo, c->counts[0], c->n, items, 0, t);
    if (send_hi) halo_trace_kernel<<<gb, 256, 0, st>>>(src, send_hi, c->counts[0], c->n, items, 1, t);
    DG_LAUNCH_CHECK("halo_trace_kernel");
    return DG_OK;
  }
  const size_t row = sizeof(double) * c->np;
  const size_t pitch = row * c->counts[0];
  const size_t rows = (size_t)c->counts[1] * c->counts[2];
  if (send_lo)
    DG_CUDA_CHECK(cudaMemcpy2DAsync(send_lo, row, src, pitch, row, rows,
                                    cudaMemcpyDeviceToDevice, st));
  if (send_hi)
    DG_CUDA_CHECK(cudaMemcpy2DAsync(send_hi, row, src + (size_t)(c->counts[0] - 1) * c->np,
                                    pitch, row, rows, cudaMemcpyDeviceToDevice, st));
  return DG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// mass / inverse mass (tensor-product apply), diagonal

template <int DIM, int N>
static int launch_tensor(dg_ctx *c, const double *src, double *dst, int ncomp, bool inverse,
                         cudaStream_t st) {
  TensorTab<N> t;
  const std::vector<double> &A = inverse ? c->basis.Minv : c->basis.M;
  for (int i = 0; i < N * N; ++i) t.A[i] = A[i];
  using TC = TensorCfg<DIM, N>;
  const int64_t cells = c->n_cells * ncomp;
  if constexpr (DIM == 3 && (N & 1)) {
    // runs of contiguous cells: TMA in, even-odd sweeps, TMA out
    constexpr int CPB = N <= 3 ? 32 : (N <= 5 ? 16 : 8);
    EOTab<N> eo;
    constexpr int H = N / 2, NE = (N + 1) / 2;
    for (int i = 0; i < NE; ++i)
      for (int j = 0; j < NE; ++j)
        eo.Ae[i * NE + j] = (j == H) ? A[i * N + j] : 0.5 * (A[i * N + j] + A[i * N + N - 1 - j]);
    for (int i = 0; i < H; ++i)
      for (int j = 0; j < H; ++j) eo.Ao[i * H + j] = 0.5 * (A[i * N + j] - A[i * N + N - 1 - j]);
    const int nb = (int)((cells + CPB - 1) / CPB);
    tensor_fast_kernel<N, CPB><<<nb, ((CPB * N * N + 31) / 32) * 32, 0, st>>>(
        src, dst, c->geo(), eo, cells, inverse ? 1 : 0);
    DG_LAUNCH_CHECK("tensor_fast_kernel");
    return DG_OK;
  }
  const int nb = (int)((cells + TC::NC - 1) / TC::NC);
  tensor_apply_kernel<DIM, N><<<nb, TC::THREADS, TC::SMEM, st>>>(src, dst, c->geo(), t, cells,
                                                                  inverse ? 1 : 0);
  DG_LAUNCH_CHECK("tensor_apply_kernel");
  return DG_OK;
}

static int tensor_dispatch(dg_ctx *c, const double *src, double *dst, int ncomp, bool inverse,
                           cudaStream_t st) {
#define DG_T(D, NN) \
  case NN: return launch_tensor<D, NN>(c, src, dst, ncomp, inverse, st);
  if (c->dim == 3) {
    switch (c->n) { DG_T(3, 2) DG_T(3, 3) DG_T(3, 4) DG_T(3, 5) DG_T(3, 6) DG_T(3, 7) DG_T(3, 8) }
  } else {
    switch (c->n) { DG_T(2, 2) DG_T(2, 3) DG_T(2, 4) DG_T(2, 5) DG_T(2, 6) DG_T(2, 7) DG_T(2, 8) }
  }
#undef DG_T
  return inval("unsupported degree");
}

struct DiagTab {
  double Mdiag[kMaxN], Kdiag[kMaxN];
  double dL0, dRn;
};

// exact diagonal of the element block (operators.py:675-730): volume
// sum_d s_d (2/h_d) K_ii prod M_jj plus the own-side face terms at end nodes
__global__ void laplace_diag_kernel(double *__restrict__ diag, Geo g, int dim, int n, DiagTab t,
                                    double tau_scale, int64_t ndofs) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t np = (dim == 3) ? (int64_t)n * n * n : (int64_t)n * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndofs; i += stride) {
    const int64_t e = i / np;
    int o = (int)(i % np);
    int idx[3];
    idx[0] = o % n;
    o /= n;
    idx[1] = o % n;
    idx[2] = (dim == 3) ? o / n : 0;
    int cc[3];
    cc[0] = (int)(e % g.nx);
    cc[1] = (int)((e / g.nx) % g.ny);
    cc[2] = (int)(e / ((int64_t)g.nx * g.ny));
    const double h[3] = {g.hx[cc[0]], g.hy[cc[1]], dim == 3 ? g.hz[cc[2]] : 2.0};
    const double taue = g.tau[e];
    double acc = 0.0;
    for (int d = 0; d < dim; ++d) {
      double sfac = 1.0, tang = 1.0;
      for (int dd = 0; dd < dim; ++dd)
        if (dd != d) {
          sfac *= 0.5 * h[dd];
          tang *= t.Mdiag[idx[dd]];
        }
      double line = 2.0 / h[d] * t.Kdiag[idx[d]];
      for (int s = 0; s < 2; ++s) {
        if (idx[d] != (s ? n - 1 : 0)) continue;
        // neighbour kind
        const int nmax = d == 0 ? g.nx : d == 1 ? g.ny : g.nz;
        const bool at_edge = s ? (cc[d] == nmax - 1) : (cc[d] == 0);
        int kind = 0;
        double taun = 0.0;
        if (at_edge) {
          const int m = g.mode[2 * d + s];
          if (m == kBndNone || m == kBndNeumann) kind = m;
          else if (m == kGhost) taun = g.ghost_tau[s][cc[1] + (int64_t)g.ny * cc[2]];
          else {
            int c2[3] = {cc[0], cc[1], cc[2]};
            c2[d] = s ? 0 : nmax - 1;
            taun = g.tau[c2[0] + (int64_t)g.nx * (c2[1] + (int64_t)g.ny * c2[2])];
          }
        } else {
          int c2[3] = {cc[0], cc[1], cc[2]};
          c2[d] += s ? 1 : -1;
          taun = g.tau[c2[0] + (int64_t)g.nx * (c2[1] + (int64_t)g.ny * c2[2])];
        }
        const double dend = s ? t.dRn : t.dL0;  // own derivative row at own end node
        const double sg = s ? -1.0 : 1.0;
        if (kind == 0) line += sg * 2.0 * dend / h[d] + tau_scale * fmax(taue, taun);
        else if (kind == kBndNeumann) line += sg * 4.0 * dend / h[d] + 2.0 * tau_scale * taue;
      }
      acc += sfac * tang * line;
    }
    diag[i] = acc;
  }
}

extern "C" {

int dg_mass(dg_ctx *c, const double *src, double *dst, int ncomp, void *stream) {
  if (!c || !src || !dst || ncomp < 1) return inval("invalid argument");
  return tensor_dispatch(c, src, dst, ncomp, false, (cudaStream_t)stream);
}

int dg_inverse_mass(dg_ctx *c, const double *src, double *dst, int ncomp, void *stream) {
  if (!c || !src || !dst || ncomp < 1) return inval("invalid argument");
  return tensor_dispatch(c, src, dst, ncomp, true, (cudaStream_t)stream);
}

int dg_laplace_diagonal(dg_ctx *c, double *diag, double tau_scale, void *stream) {
  if (!c || !diag) return inval("null argument");
  DiagTab t;
  for (int i = 0; i < c->n; ++i) {
    t.Mdiag[i] = c->basis.M[i * c->n + i];
    t.Kdiag[i] = c->basis.K[i * c->n + i];
  }
  t.dL0 = c->basis.ld[0];
  t.dRn = c->basis.rd[c->n - 1];
  laplace_diag_kernel<<<grid_for(c->n_dofs), 256, 0, (cudaStream_t)stream>>>(
      diag, c->geo(), c->dim, c->n, t, tau_scale, c->n_dofs);
  DG_LAUNCH_CHECK("laplace_diag_kernel");
  return DG_OK;
}

}  // extern "C"

#include "pcg.inc"

// per-cell dual-weight factor hx hy hz / 8 (3D), built on first use
__global__ void hcell_kernel(Geo g, double *hc) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)g.nx * g.ny * g.nz) return;
  const int ix = (int)(e % g.nx), iy = (int)((e / g.nx) % g.ny), iz = (int)(e / ((int64_t)g.nx * g.ny));
  hc[e] = 0.125 * g.hx[ix] * g.hy[iy] * g.hz[iz];
}
static int ensure_hcell(dg_ctx *c) {
  if (c->d_hcell) return DG_OK;
  DG_CUDA_CHECK(cudaMalloc((void **)&c->d_hcell, sizeof(double) * (c->n_cells > 0 ? c->n_cells : 1)));
  hcell_kernel<<<(unsigned)((c->n_cells + 255) / 256), 256>>>(c->geo(), c->d_hcell);
  DG_LAUNCH_CHECK("hcell_kernel");
  DG_CUDA_CHECK(cudaDeviceSynchronize());
  return DG_OK;
}

static int ensure_red3(dg_ctx *c) {
  if (c->d_red3) return DG_OK;
  DG_CUDA_CHECK(cudaMalloc((void **)&c->d_red3, sizeof(double) * 3 * kRedBlocks));
  return DG_OK;
}
#include "slabcg.inc"

// The quadrature-point operators (Helmholtz, projection, convective, the
// once-per-step right-hand sides, element-local PCG) are in vecops.cu.

// compute_penalty_parameters (operators.py:736-755): one warp per cell forms
// the cell integrals of the velocity components (sum_i u_i w_i with the
// dual weights), |u_mean| = |integral| / V, tau_D = zd |u_mean| V^(1/dim) dt,
// tau_C,e = zc |u_mean| dt; pass 2 averages tau_C,e onto faces.
__global__ void penalty_cell_kernel(const double *__restrict__ u, Geo g, int dim, int nn, WInt wi,
                                    int64_t ncells, double dt, double zd, double zc,
                                    double *__restrict__ tau_d, double *__restrict__ tau_ce) {
  DG_STAGE_WINT(sw, wi);
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= ncells) return;
  const int64_t np = (dim == 3) ? (int64_t)nn * nn * nn : (int64_t)nn * nn;
  double m[3] = {0.0, 0.0, 0.0};
  for (int c = 0; c < dim; ++c) {
    double acc = 0.0;
    for (int64_t o = lane; o < np; o += 32) {
      const int64_t i = e * np + o;
      acc += u[(int64_t)c * ncells * np + i] * dual_weight(g, dim, nn, sw, i);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    m[c] = acc;
  }
  if (lane != 0) return;
  const int ix = (int)(e % g.nx), iy = (int)((e / g.nx) % g.ny), iz = (int)(e / ((int64_t)g.nx * g.ny));
  double vol = g.hx[ix] * g.hy[iy];
  if (dim == 3) vol *= g.hz[iz];
  const double norm = sqrt(m[0] * m[0] + m[1] * m[1] + m[2] * m[2]) / vol;
  if (tau_d) tau_d[e] = zd * norm * pow(vol, 1.0 / dim) * dt;
  if (tau_ce) tau_ce[e] = zc * norm * dt;
}

// tau_C face layout [d*ncells + e]: face between cell e and its +d neighbour
// (periodic wrap included; 0 where there is no face)
__global__ void penalty_face_kernel(const double *__restrict__ tau_ce, Geo g, int dim,
                                    int64_t ncells, double *__restrict__ tau_c) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dim * ncells) return;
  const int d = (int)(i / ncells);
  const int64_t e = i - (int64_t)d * ncells;
  int idx[3];
  idx[0] = (int)(e % g.nx);
  idx[1] = (int)((e / g.nx) % g.ny);
  idx[2] = (int)(e / ((int64_t)g.nx * g.ny));
  const int nd = d == 0 ? g.nx : (d == 1 ? g.ny : g.nz);
  int nb = idx[d] + 1;
  if (nb >= nd) {
    if (g.mode[2 * d + 1] != kWrap) {
      tau_c[i] = 0.0;
      return;
    }
    nb = 0;
  }
  idx[d] = nb;
  const int64_t en = idx[0] + (int64_t)g.nx * (idx[1] + (int64_t)g.ny * idx[2]);
  tau_c[i] = 0.5 * (tau_ce[e] + tau_ce[en]);
}

extern "C" int dg_penalty_parameters(dg_ctx *c, const double *u, double dt, double cfl, double zeta_d_star,
                          double zeta_c_star, double *tau_d, double *tau_c, void *stream) {
  if (!c || !u) return inval("null argument");
  if (!(cfl > 0.0)) return inval("CFL must be positive, got " + std::to_string(cfl));
  if (c->mode[0] == kGhost || c->mode[1] == kGhost)
    return inval("penalty parameters run on whole-mesh contexts");
  const cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_work(c, 1);
  if (rc) return rc;
  double *tce = tau_c ? c->work[0] : nullptr;  // per-cell tau_C (n_cells <= n_dofs)
  const int64_t nc = c->n_cells;
  if (nc == 0) return DG_OK;
  penalty_cell_kernel<<<(unsigned)((nc * 32 + 255) / 256), 256, 0, st>>>(
      u, c->geo(), c->dim, c->n, wint_of(c), nc, dt, zeta_d_star / cfl, zeta_c_star / cfl, tau_d,
      tce);
  DG_LAUNCH_CHECK("penalty_cell_kernel");
  if (tau_c) {
    penalty_face_kernel<<<(unsigned)((c->dim * nc + 255) / 256), 256, 0, st>>>(tce, c->geo(),
                                                                               c->dim, nc, tau_c);
    DG_LAUNCH_CHECK("penalty_face_kernel");
  }
  return DG_OK;
}

