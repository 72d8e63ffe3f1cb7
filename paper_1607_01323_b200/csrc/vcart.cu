// Host side of the Cartesian vector-operator fast path (vcart.cuh): tables,
// the per-context trace buffer, launches.  Own translation unit of libdgmf.
#include <cstdlib>

#include "ctx.h"
#include "vcart.cuh"

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

template <int N, int OP>
static int launch_vc(dg_ctx *c, const double *src, double *dst, double gamma0_dt, double nu,
                     const double *tau_d, const double *tau_c, cudaStream_t st) {
  using C = VcCfg<N>;
  static const VcTab<N> tab = vc_tab<N>(c->basis);  // depends on k only
  auto ktr = vc_trace_kernel<N, OP == kVcHelmholtz>;
  auto kap = vc_apply_kernel<N, OP>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(ktr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    DG_CUDA_CHECK(cudaFuncSetAttribute(kap, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr = true;
  }
  if (c->n_cells == 0) return DG_OK;
  const bool faces = OP == kVcHelmholtz ? nu != 0.0 : tau_c != nullptr;
  if (faces) {
    if (int rc = ensure_trc(c, c->n_cells * C::TRC)) return rc;
  }
  const unsigned grid = (unsigned)((c->n_cells + C::CPB - 1) / C::CPB);
  const Geo g = c->geo();
  if (faces) {
    ktr<<<grid, C::THREADS, C::SMEM, st>>>(src, c->d_trc, g, tab, c->n_cells);
    DG_LAUNCH_CHECK("vc_trace_kernel");
  }
  kap<<<grid, C::THREADS, C::SMEM, st>>>(src, c->d_trc, dst, g, tab, gamma0_dt, nu, tau_d, tau_c,
                                          c->n_cells);
  DG_LAUNCH_CHECK("vc_apply_kernel");
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

}  // namespace dg
