// Host side of the quadrature-point operators (kernels in vecops.cuh,
// elpcg.cuh): viscous Helmholtz, projection, convective, the once-per-step
// right-hand sides and the element-local PCG.  Own translation unit of
// libdgmf (compiled in parallel with dgmf.cu).
#include <string>

#include "ctx.h"
#include "elpcg.cuh"
#include "vecops_impl.cuh"

using namespace dg;

namespace dg {
// Cartesian fast path of the Helmholtz / projection operators (vcart.cu)
int vcart_apply(dg_ctx *c, int op, const double *src, double *dst, double gamma0_dt, double nu,
                const double *tau_d, const double *tau_c, cudaStream_t st);
}  // namespace dg

// operators on the linear rule (n_q = k+1); CI / CO: 0 = dim components,
// 1 = scalar (instantiated in vec_lin<dim>_<CI><CO>.cu)
template <int CI, int CO>
static int vecop_linear(dg_ctx *c, const double *src, double *dst, const VecParams &prm,
                        cudaStream_t st) {
  if (c->dim == 3) return vecop_linear_dim<3, CI, CO>(c, src, dst, prm, st);
  return vecop_linear_dim<2, CI, CO>(c, src, dst, prm, st);
}

static int vec_slab_check(const dg_ctx *c) {
  if (c->mode[0] == kGhost || c->mode[1] == kGhost)
    return inval("vector operators run on whole-mesh contexts (no x-slab ghosts)");
  return DG_OK;
}

static int form_check(int form, bool strong_ok) {
  if (form == kFormStandard || form == kFormWeak || (strong_ok && form == kFormStrong)) return DG_OK;
  return inval(strong_ok ? "unknown divergence form (0 standard, 1 weak, 2 strong)"
                         : "unknown pressure-gradient form (0 standard, 1 weak)");
}

static void copy_bnd(VecParams &prm, const double *const *bnd) {
  for (int s = 0; s < 6; ++s) prm.bnd[s] = bnd ? bnd[s] : nullptr;
}

extern "C" int dg_helmholtz_vmult(dg_ctx *c, const double *src, double *dst, double gamma0_dt,
                                  double nu, void *stream) {
  if (!c || !src || !dst) return inval("null argument");
  if (int rc = vec_slab_check(c)) return rc;
  VecParams prm{};
  prm.op = kOpHelmholtz;
  prm.gamma0_dt = gamma0_dt;
  prm.nu = nu;
  const int rc = vcart_apply(c, 0, src, dst, gamma0_dt, nu, nullptr, nullptr, (cudaStream_t)stream);
  if (rc != DG_ENOTSUP) return rc;
  return vecop_linear<0, 0>(c, src, dst, prm, (cudaStream_t)stream);
}

extern "C" int dg_projection_vmult(dg_ctx *c, const double *src, double *dst,
                                   const double *tau_d, const double *tau_c, void *stream) {
  if (!c || !src || !dst) return inval("null argument");
  if (int rc = vec_slab_check(c)) return rc;
  VecParams prm{};
  prm.op = kOpProjection;
  prm.tau_d = tau_d;
  prm.tau_c = tau_c;
  const int rc = vcart_apply(c, 1, src, dst, 0.0, 0.0, tau_d, tau_c, (cudaStream_t)stream);
  if (rc != DG_ENOTSUP) return rc;
  return vecop_linear<0, 0>(c, src, dst, prm, (cudaStream_t)stream);
}

extern "C" int dg_convective_rhs_ex(dg_ctx *c, int n_hist, const double *const *hist,
                                    const double *betas, const double *const *g_data,
                                    const double *body, double *dst, void *stream) {
  if (!c || !hist || !betas || !dst) return inval("null argument");
  if (n_hist < 1 || n_hist > kMaxHist) return inval("need 1..4 history levels");
  if (int rc = vec_slab_check(c)) return rc;
  VecParams prm{};
  prm.op = kOpConvective;
  prm.n_hist = n_hist;
  for (int j = 0; j < n_hist; ++j) {
    if (!hist[j]) return inval("null history level");
    prm.hist[j] = hist[j];
    prm.beta[j] = betas[j];
    for (int s = 0; s < 6; ++s) prm.gh[j][s] = g_data ? g_data[j * 6 + s] : nullptr;
  }
  prm.vol_data = body;
  return vecop_over(c, hist[0], dst, prm, (cudaStream_t)stream);
}

extern "C" int dg_convective_rhs(dg_ctx *c, int n_hist, const double *const *hist,
                                 const double *betas, double *dst, void *stream) {
  return dg_convective_rhs_ex(c, n_hist, hist, betas, nullptr, nullptr, dst, stream);
}

extern "C" int dg_divergence_rhs(dg_ctx *c, const double *src, double *dst, double scale,
                                 int form, void *stream) {
  if (!c || !src || !dst) return inval("null argument");
  if (int rc = vec_slab_check(c)) return rc;
  if (int rc = form_check(form, true)) return rc;
  VecParams prm{};
  prm.op = kOpDivergence;
  prm.scale = scale;
  prm.form = form;
  return vecop_linear<0, 1>(c, src, dst, prm, (cudaStream_t)stream);
}

extern "C" int dg_pressure_gradient_rhs(dg_ctx *c, const double *src, double *dst, double scale,
                                        int form, void *stream) {
  if (!c || !src || !dst) return inval("null argument");
  if (int rc = vec_slab_check(c)) return rc;
  if (int rc = form_check(form, false)) return rc;
  VecParams prm{};
  prm.op = kOpGradient;
  prm.scale = scale;
  prm.form = form;
  return vecop_linear<1, 0>(c, src, dst, prm, (cudaStream_t)stream);
}

extern "C" int dg_vorticity(dg_ctx *c, const double *src, double *dst, void *stream) {
  if (!c || !src || !dst) return inval("null argument");
  if (src == dst) return inval("vorticity: src and dst must not alias");
  if (int rc = vec_slab_check(c)) return rc;
  VecParams prm{};
  prm.op = kOpVorticity;
  const cudaStream_t st = (cudaStream_t)stream;
  // (curl u, v) per cell, then the exact inverse mass in place
  int rc = c->dim == 3 ? vecop_linear<0, 0>(c, src, dst, prm, st) : vecop_linear<0, 1>(c, src, dst, prm, st);
  if (rc) return rc;
  return dg_inverse_mass(c, dst, dst, c->dim == 3 ? 3 : 1, stream);
}

extern "C" int dg_pressure_neumann_rhs(dg_ctx *c, int n_hist, const double *const *hist,
                                       const double *const *vort, const double *betas, double nu,
                                       const double *const *bnd, double *dst, void *stream) {
  if (!c || !hist || !vort || !betas || !dst) return inval("null argument");
  if (n_hist < 1 || n_hist > kMaxHist) return inval("need 1..4 history levels");
  if (int rc = vec_slab_check(c)) return rc;
  VecParams prm{};
  prm.op = kOpPressureNeumann;
  prm.n_hist = n_hist;
  prm.nu = nu;
  prm.n_vort = c->dim == 3 ? 3 : 1;
  for (int j = 0; j < n_hist; ++j) {
    if (!hist[j] || !vort[j]) return inval("null history level");
    prm.hist[j] = hist[j];
    prm.vort[j] = vort[j];
    prm.beta[j] = betas[j];
  }
  copy_bnd(prm, bnd);
  return vecop_linear<0, 1>(c, hist[0], dst, prm, (cudaStream_t)stream);
}

extern "C" int dg_gp_dirichlet_rhs(dg_ctx *c, const double *const *bnd, double tau_scale,
                                   double *dst, void *stream) {
  if (!c || !dst) return inval("null argument");
  if (int rc = vec_slab_check(c)) return rc;
  VecParams prm{};
  prm.op = kOpGpDirichlet;
  prm.tau_scale = tau_scale;
  copy_bnd(prm, bnd);
  return vecop_linear<1, 1>(c, dst, dst, prm, (cudaStream_t)stream);
}

extern "C" int dg_viscous_rhs_bc(dg_ctx *c, const double *const *bnd, double nu, double *dst,
                                 void *stream) {
  if (!c || !dst) return inval("null argument");
  if (int rc = vec_slab_check(c)) return rc;
  VecParams prm{};
  prm.op = kOpViscousBc;
  prm.nu = nu;
  copy_bnd(prm, bnd);
  return vecop_linear<1, 0>(c, dst, dst, prm, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// element-local PCG (elpcg.cuh)

template <int DIM, int N>
static int launch_el_pcg(dg_ctx *c, const double *b, double *x, const double *tau_d,
                         double rel_tol, int max_iter, double floor_factor, int *iters, int *conv,
                         cudaStream_t st) {
  constexpr int NP = DIM == 3 ? N * N * N : N * N;
  constexpr size_t SMEM = sizeof(double) * 7 * DIM * NP;
  auto kern = el_pcg_kernel<DIM, N>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    attr = true;
  }
  if (c->n_cells == 0) return DG_OK;
  ElTab<N> t;
  const Basis1D &bs = c->basis;
  for (int i = 0; i < N * N; ++i) {
    t.S[i] = bs.S[i];
    t.D[i] = bs.D[i];
    t.M[i] = bs.M[i];
    t.Minv[i] = bs.Minv[i];
  }
  for (int i = 0; i < N; ++i) t.w[i] = bs.wts[i];
  kern<<<(unsigned)c->n_cells, ElCfg<DIM>::THREADS, SMEM, st>>>(b, x, c->geo(), t, tau_d, rel_tol,
                                                               max_iter, floor_factor, iters, conv,
                                                               c->n_cells);
  DG_LAUNCH_CHECK("el_pcg_kernel");
  return DG_OK;
}

extern "C" int dg_element_local_pcg(dg_ctx *c, const double *b, double *x, const double *tau_d,
                                    double rel_tol, int max_iter, double floor_factor, int *iters,
                                    int *converged, void *stream) {
  if (!c || !b || !x) return inval("null argument");
  if (b == x) return inval("element-local PCG: b and x must not alias");
  if (max_iter < 0) return inval("max_iter must be >= 0");
  if (int rc = vec_slab_check(c)) return rc;
  const cudaStream_t st = (cudaStream_t)stream;
#define DG_E(D, NN) \
  case NN: return launch_el_pcg<D, NN>(c, b, x, tau_d, rel_tol, max_iter, floor_factor, iters, converged, st);
  if (c->dim == 3) {
    switch (c->n) { DG_E(3, 2) DG_E(3, 3) DG_E(3, 4) DG_E(3, 5) DG_E(3, 6) DG_E(3, 7) DG_E(3, 8) }
  } else {
    switch (c->n) { DG_E(2, 2) DG_E(2, 3) DG_E(2, 4) DG_E(2, 5) DG_E(2, 6) DG_E(2, 7) DG_E(2, 8) }
  }
#undef DG_E
  return inval("unsupported degree");
}
