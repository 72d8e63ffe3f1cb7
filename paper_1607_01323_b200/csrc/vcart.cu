// Host side of the Cartesian vector-operator fast path (vcart.cuh): tables,
// the per-context trace buffer, launches.  Own translation unit of libdgmf.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ctx.h"
#include "vcart2.cuh"
#include "vector.cuh"

namespace dg {

template <int N>
static VcTab<N> vc_tab(const Basis1D &b) {
  VcTab<N> t;
  std::vector<double> V, Dv, Ve, De;
  lagrange_tables(b.pts, b.pts, V, Dv);
  lagrange_tables(b.pts, std::vector<double>{-1.0, 1.0}, Ve, De);
  for (int i = 0; i < N * N; ++i) {
    t.S[i] = b.S[i];
    t.Dg[i] = Dv[i];
  }
  for (int m = 0; m < N; ++m) {
    t.w[m] = b.wts[m];
    t.eL[m] = Ve[m];
    t.eR[m] = Ve[N + m];
    t.gL[m] = De[m];
    t.gR[m] = De[N + m];
  }
  return t;
}

static int ensure_trc(dg_ctx *c, int64_t n) {
  if (c->trc_n >= n) return DG_OK;
  cudaFree(c->d_trc);
  c->d_trc = nullptr;
  c->trc_n = 0;
  DG_CUDA_CHECK(cudaMalloc(&c->d_trc, sizeof(double) * (size_t)n));
  c->trc_n = n;
  return DG_OK;
}

// pz != null (the velocity PCG): the trace kernel first updates the direction
// in place, src = pz + beta src, and sets scal[0] = rz_new (vpcg_p_kernel's
// work); *fused = whether it did (no trace kernel without face terms)
template <int N, int OP, int CB = 0>
static int launch_vc(dg_ctx *c, const double *src, double *dst, double gamma0_dt, double nu,
                     const double *tau_d, const double *tau_c, cudaStream_t st,
                     double *pdot = nullptr, const double *pz = nullptr, double beta = 0.0,
                     double *scal = nullptr, double rz_new = 0.0, bool *fused = nullptr) {
  if (fused) *fused = false;
  using C = VlCfg<N, CB>;
  static const VcTab<N> tab = vc_tab<N>(c->basis);  // depends on k only
  auto ktr = vl_trace_kernel<N, OP == kVcHelmholtz, CB>;
  auto kap = vl_apply_kernel<N, OP, CB>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(ktr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    DG_CUDA_CHECK(cudaFuncSetAttribute(kap, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    DG_CUDA_CHECK(cudaFuncSetAttribute(ktr, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    DG_CUDA_CHECK(cudaFuncSetAttribute(kap, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    attr = true;
  }
  if (c->n_cells == 0) return DG_OK;
  const bool faces = OP == kVcHelmholtz ? nu != 0.0 : tau_c != nullptr;
  if (faces) {
    if (int rc = ensure_trc(c, c->n_cells * 36 * N * N)) return rc;
  }
  const unsigned grid = (unsigned)((c->n_cells + C::CPB - 1) / C::CPB);
  const Geo g = c->geo();
  if (faces) {
    ktr<<<grid, C::THREADS, C::SMEM, st>>>(src, c->d_trc, g, tab, c->n_cells, pz, beta, scal,
                                            rz_new);
    DG_LAUNCH_CHECK("vl_trace_kernel");
    if (fused) *fused = pz != nullptr;
  }
  kap<<<grid, C::THREADS, C::SMEM, st>>>(src, c->d_trc, dst, g, tab, gamma0_dt, nu, tau_d, tau_c,
                                          c->n_cells, pdot);
  DG_LAUNCH_CHECK("vl_apply_kernel");
  return DG_OK;
}

// 3D, n_q = k+1 (the linear rule); returns DG_ENOTSUP when the generic
// kernel should run (DG_VEC_GENERIC=1 forces it, for A/B comparisons).
int vcart_apply(dg_ctx *c, int op, const double *src, double *dst, double gamma0_dt, double nu,
                const double *tau_d, const double *tau_c, cudaStream_t st) {
  static const bool generic = [] {
    const char *v = getenv("DG_VEC_GENERIC");
    return v && atoi(v) != 0;
  }();
  if (generic || c->dim != 3 || c->basis.nq != c->n) return DG_ENOTSUP;
  if (src == dst) return inval("vector operator: src and dst must not alias");
#define DG_VC(NN)                                                                                   \
  case NN:                                                                                          \
    return op == kVcHelmholtz                                                                       \
               ? launch_vc<NN, kVcHelmholtz>(c, src, dst, gamma0_dt, nu, tau_d, tau_c, st)         \
               : launch_vc<NN, kVcProjection>(c, src, dst, gamma0_dt, nu, tau_d, tau_c, st);
  switch (c->n) { DG_VC(2) DG_VC(3) DG_VC(4) DG_VC(5) DG_VC(6) DG_VC(7) DG_VC(8) }
#undef DG_VC
  return DG_ENOTSUP;
}

// the fast-path operator with the CG product: dst = A src and, per CTA of the
// apply kernel, pdot[b] = sum of src . dst over its cells (deterministic);
// *nparts = the number of CTAs.  DG_ENOTSUP where vcart_apply has no fast path.
static int vcart_apply_dot(dg_ctx *c, int op, const double *src, double *dst, double gamma0_dt,
                           double nu, const double *tau_d, const double *tau_c, double *pdot,
                           int64_t *nparts, cudaStream_t st, const double *pz = nullptr,
                           double beta = 0.0, double *scal = nullptr, double rz_new = 0.0,
                           bool *fused = nullptr) {
  if (fused) *fused = false;
  static const bool generic = [] {
    const char *v = getenv("DG_VEC_GENERIC");
    return v && atoi(v) != 0;
  }();
  if (generic || c->dim != 3 || c->basis.nq != c->n) return DG_ENOTSUP;
  if (src == dst) return inval("vector operator: src and dst must not alias");
#define DG_VC(NN)                                                                                   \
  case NN:                                                                                          \
    *nparts = (c->n_cells + VlCfg<NN>::CPB - 1) / VlCfg<NN>::CPB;                                  \
    return op == kVcHelmholtz                                                                       \
               ? launch_vc<NN, kVcHelmholtz>(c, src, dst, gamma0_dt, nu, tau_d, tau_c, st, pdot,   \
                                             pz, beta, scal, rz_new, fused)                        \
               : launch_vc<NN, kVcProjection>(c, src, dst, gamma0_dt, nu, tau_d, tau_c, st, pdot,  \
                                              pz, beta, scal, rz_new, fused);
  switch (c->n) { DG_VC(2) DG_VC(3) DG_VC(4) DG_VC(5) DG_VC(6) DG_VC(7) DG_VC(8) }
#undef DG_VC
  return DG_ENOTSUP;
}

}  // namespace dg

// ---------------------------------------------------------------------------
// M^-1-preconditioned CG of the velocity solves (viscous Helmholtz,
// projection), the reference pcg (solvers.py:30-73) with
// prec = inverse_mass_apply, run on the device: the operator is the fast
// path above, the x / r update, the exact inverse mass and the r.z partial
// sums are one kernel (vpcg_update_kernel), reductions are deterministic,
// the host reads two scalars per iteration.

namespace dg {

__global__ void vpcg_sub_kernel(double *__restrict__ r, const double *__restrict__ b,
                                const double *__restrict__ y, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    r[i] = __dsub_rn(b[i], y[i]);
}

// p = z + beta p ; scal[0] = rz_new
__global__ void vpcg_p_kernel(double *__restrict__ p, const double *__restrict__ z, double beta,
                              double rz_new, double *__restrict__ scal, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
  if (blockIdx.x == 0 && threadIdx.x == 0) scal[0] = rz_new;
}

static int vgrid(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

static int ensure_vwork(dg_ctx *c, int nvec, int64_t per) {
  if (c->vwork_n < per) {
    for (double *w : c->vwork) cudaFree(w);
    c->vwork.clear();
    c->vwork_n = per;
  }
  while ((int)c->vwork.size() < nvec) {
    double *p = nullptr;
    DG_CUDA_CHECK(cudaMalloc((void **)&p, sizeof(double) * (size_t)std::max<int64_t>(per, 1)));
    c->vwork.push_back(p);
  }
  return DG_OK;
}

template <int N>
static int launch_vpcg_update(dg_ctx *c, double *x, double *r, const double *p, const double *Ap,
                              double *z, const double *scal, cudaStream_t st, int *nblocks) {
  using C = VcCfg<N>;
  MinvTab<N> mi;
  for (int i = 0; i < N * N; ++i) mi.A[i] = c->basis.Minv[i];
  const int64_t nb = (c->n_cells + C::CPB - 1) / C::CPB;
  if (c->vpart_n < nb) {
    cudaFree(c->d_vpart);
    c->d_vpart = nullptr;
    c->vpart_n = 0;
    DG_CUDA_CHECK(cudaMalloc((void **)&c->d_vpart, sizeof(double) * (size_t)nb));
    c->vpart_n = nb;
  }
  *nblocks = (int)nb;
  if (nb == 0) return DG_OK;
  vpcg_update_kernel<N><<<(unsigned)nb, ((C::THREADS + 31) / 32) * 32, 0, st>>>(
      x, r, p, Ap, z, scal, mi, c->geo(), c->n_cells, c->d_vpart);
  DG_LAUNCH_CHECK("vpcg_update_kernel");
  return DG_OK;
}

// the update kernel's per-CTA partial buffer (allocated outside any capture)
static int vpcg_ensure_part(dg_ctx *c, int *nblocks) {
  int64_t nb = 0;
#define DG_U(NN) \
  case NN: nb = (c->n_cells + VcCfg<NN>::CPB - 1) / VcCfg<NN>::CPB; break;
  switch (c->n) { DG_U(2) DG_U(3) DG_U(4) DG_U(5) DG_U(6) DG_U(7) DG_U(8) default: return inval("unsupported degree"); }
#undef DG_U
  if (c->vpart_n < nb) {
    cudaFree(c->d_vpart);
    c->d_vpart = nullptr;
    c->vpart_n = 0;
    DG_CUDA_CHECK(cudaMalloc((void **)&c->d_vpart, sizeof(double) * (size_t)nb));
    c->vpart_n = nb;
  }
  *nblocks = (int)nb;
  return DG_OK;
}

static int vpcg_update(dg_ctx *c, double *x, double *r, const double *p, const double *Ap, double *z,
                       const double *scal, cudaStream_t st, int *nblocks) {
#define DG_U(NN) \
  case NN: return launch_vpcg_update<NN>(c, x, r, p, Ap, z, scal, st, nblocks);
  switch (c->n) { DG_U(2) DG_U(3) DG_U(4) DG_U(5) DG_U(6) DG_U(7) DG_U(8) }
#undef DG_U
  return inval("unsupported degree");
}

}  // namespace dg

using namespace dg;

extern "C" int dg_vector_pcg(dg_ctx *c, int op, double gamma0_dt, double nu, const double *tau_d,
                             const double *tau_c, const double *b, double *x, double rel_tol,
                             double abs_tol, int max_iter, dg_pcg_stats *stats, double *hist,
                             void *stream) {
  if (!c || !b || !x || !stats) return inval("null argument");
  if (op != 0 && op != 1) return inval("vector PCG: op 0 (viscous Helmholtz) or 1 (projection)");
  if (c->dim != 3) return inval("vector PCG: 3D contexts");
  if (c->mode[0] == kGhost || c->mode[1] == kGhost)
    return inval("vector PCG runs on whole-mesh contexts");
  if (max_iter < 0) return inval("max_iter must be >= 0");
  std::lock_guard<std::mutex> lock(c->mu);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = 3 * c->n_dofs;
  int rc = ensure_vwork(c, 4, n);
  if (rc) return rc;
  double *r = c->vwork[0], *z = c->vwork[1], *p = c->vwork[2], *Ap = c->vwork[3];
  double *scal = c->d_scal + 10;  // [rz, pAp, rz_new]
  double *hs = c->h_scal + 10;
  auto apply = [&](const double *src, double *dst, cudaStream_t s) {
    return op == 0 ? dg_helmholtz_vmult(c, src, dst, gamma0_dt, nu, s)
                   : dg_projection_vmult(c, src, dst, tau_d, tau_c, s);
  };
  const int gb = vgrid(n);
  // r = b - A x0 ; z = M^-1 r ; rz
  if ((rc = apply(x, Ap, st))) return rc;
  vpcg_sub_kernel<<<gb, 256, 0, st>>>(r, b, Ap, n);
  DG_LAUNCH_CHECK("vpcg_sub_kernel");
  if ((rc = dg_inverse_mass(c, r, z, 3, stream))) return rc;
  dot_partial_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(r, z, n, c->d_red);
  sum_partials_kernel<<<1, 1024, 0, st>>>(c->d_red, kRedBlocks, scal + 0);
  DG_LAUNCH_CHECK("dot");
  DG_CUDA_CHECK(cudaMemcpyAsync(hs, scal, sizeof(double), cudaMemcpyDeviceToHost, st));
  DG_CUDA_CHECK(cudaStreamSynchronize(st));
  double rz = hs[0];
  stats->iterations = 0;
  stats->converged = 0;
  stats->breakdown = 0;
  if (rz < 0) {
    stats->residual = std::sqrt(std::fabs(rz));
    stats->breakdown = 1;
    return DG_OK;
  }
  const double norm0 = std::sqrt(rz);
  const double tol = std::max(rel_tol * norm0, abs_tol);
  if (hist) hist[0] = norm0;
  double norm = norm0;
  stats->residual = norm0;
  if (norm0 <= tol || max_iter == 0) {
    stats->converged = norm0 <= tol;
    return DG_OK;
  }
  DG_CUDA_CHECK(cudaMemcpyAsync(p, z, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, st));
  // buffers of the loop body
  {
    const int64_t need = c->n_cells;  // >= CTAs of every fast-path apply
    if (c->apdot_n < need) {
      cudaFree(c->d_apdot);
      c->d_apdot = nullptr;
      c->apdot_n = 0;
      DG_CUDA_CHECK(cudaMalloc((void **)&c->d_apdot, sizeof(double) * (size_t)std::max<int64_t>(need, 1)));
      c->apdot_n = need;
    }
    int nb0 = 0;
    if ((rc = vpcg_ensure_part(c, &nb0))) return rc;
  }
  // one iteration up to the new r.z: Ap = A p with p.Ap from the apply kernel
  // (or a separate dot where the generic operator runs), the fused update;
  // the partial sums are reduced in a fixed order
  // pending p update (p = z + beta p, scal[0] = rz_new) of the previous
  // iteration: folded into the next trace kernel when the fast path has one
  static const bool generic = [] {
    const char *v = getenv("DG_VEC_GENERIC");
    return v && atoi(v) != 0;
  }();
  const bool fold_p = !generic && c->basis.nq == c->n && (op == 0 ? nu != 0.0 : tau_c != nullptr);
  bool pend = false;
  double pbeta = 0.0, prz = 0.0;
  const int gb2 = vgrid(n);
  auto flush_p = [&](cudaStream_t s) {
    if (!pend) return;
    vpcg_p_kernel<<<gb2, 256, 0, s>>>(p, z, pbeta, prz, scal, n);
    pend = false;
  };
  auto body = [&](cudaStream_t s) -> int {
    int64_t np = 0;
    bool fused = false;
    int rc2 = vcart_apply_dot(c, op, p, Ap, gamma0_dt, nu, tau_d, tau_c, c->d_apdot, &np, s,
                              pend ? z : nullptr, pbeta, scal, prz, &fused);
    if (pend && rc2 == DG_OK && !fused) return inval("vector PCG: direction update not applied");
    if (rc2 == DG_OK) pend = false;
    if (rc2 == DG_ENOTSUP) {
      flush_p(s);
      if ((rc2 = apply(p, Ap, s))) return rc2;
      dot_partial_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(p, Ap, n, c->d_red);
      sum_partials_kernel<<<1, 1024, 0, s>>>(c->d_red, kRedBlocks, scal + 1);
    } else if (rc2) {
      return rc2;
    } else {
      sum_partials_kernel<<<1, 1024, 0, s>>>(c->d_apdot, (int)np, scal + 1);
    }
    DG_LAUNCH_CHECK("dot");
    int nb = 0;
    if ((rc2 = vpcg_update(c, x, r, p, Ap, z, scal, s, &nb))) return rc2;
    sum_partials_kernel<<<1, 1024, 0, s>>>(c->d_vpart, nb, scal + 2);
    DG_LAUNCH_CHECK("sum_partials_kernel");
    return DG_OK;
  };
  // host loop: the stop test reads pAp and r.z each iteration (a CUDA-graph
  // loop with a device stop test measured no faster at ~0.4-0.6 ms per
  // iteration and added graph set-up per solve)
  for (int it = 1; it <= max_iter; ++it) {
    if ((rc = body(st))) return rc;
    DG_CUDA_CHECK(cudaMemcpyAsync(hs + 1, scal + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    DG_CUDA_CHECK(cudaStreamSynchronize(st));
    const double pAp = hs[1];
    if (pAp <= 0.0) {  // the update kernel left x, r untouched
      stats->iterations = it;
      stats->residual = norm;
      stats->breakdown = 1;
      return DG_OK;
    }
    const double rz_new = hs[2];
    norm = std::sqrt(std::max(rz_new, 0.0));
    if (hist) hist[it] = norm;
    stats->iterations = it;
    stats->residual = norm;
    if (norm <= tol) {
      stats->converged = 1;
      return DG_OK;
    }
    if (rz_new <= 0.0) {
      stats->breakdown = 1;
      return DG_OK;
    }
    if (fold_p) {
      pend = true;  // applied by the next iteration's trace kernel
      pbeta = rz_new / rz;
      prz = rz_new;
    } else {
      vpcg_p_kernel<<<gb, 256, 0, st>>>(p, z, rz_new / rz, rz_new, scal, n);
      DG_LAUNCH_CHECK("vpcg_p_kernel");
    }
    rz = rz_new;
  }
  return DG_OK;
}
