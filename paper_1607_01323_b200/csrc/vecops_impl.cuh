// Launch helpers of the quadrature-point operators, shared by the
// translation units that instantiate them (vec_*.cu, split so the many
// template instantiations compile in parallel).
#pragma once
#include "ctx.h"
#include "vecops.cuh"

namespace dg {

template <int N, int NQ>
static QuadTab<N, NQ> quad_tab(const Basis1D &b) {
  QuadTab<N, NQ> t;
  for (int i = 0; i < NQ * N; ++i) {
    t.S[i] = b.S[i];
    t.D[i] = b.D[i];
  }
  for (int i = 0; i < NQ; ++i) t.w[i] = b.wts[i];
  for (int i = 0; i < N; ++i) {
    t.dL[i] = b.ld[i];
    t.dR[i] = b.rd[i];
  }
  return t;
}

template <int DIM, int N, int NQ, int NCI, int NCO>
static int launch_vecop(dg_ctx *c, const double *src, double *dst, const VecParams &prm,
                        const Basis1D &b, cudaStream_t st) {
  using C = VecCfg<DIM, N, NQ, NCI, NCO>;
  auto kern = vecop_kernel<DIM, N, NQ, NCI, NCO>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr = true;
  }
  if (c->n_cells == 0) return DG_OK;
  kern<<<(unsigned)c->n_cells, C::THREADS, C::SMEM, st>>>(src, dst, c->geo(), quad_tab<N, NQ>(b), prm,
                                                         c->n_cells);
  DG_LAUNCH_CHECK("vecop_kernel");
  return DG_OK;
}

// Operators on the linear rule (n_q = k+1) for one dimension and one
// (input, output) component pattern: CI / CO = 0 -> dim components,
// 1 -> scalar.  Defined in vec_lin<dim>_<CI><CO>.cu.
template <int DIM, int CI, int CO>
int vecop_linear_dim(dg_ctx *c, const double *src, double *dst, const VecParams &prm,
                     cudaStream_t st);

#define DG_DECLARE_VECOP_LINEAR(D, CI, CO)                                                    \
  template <>                                                                                 \
  int vecop_linear_dim<D, CI, CO>(dg_ctx * c, const double *src, double *dst,                 \
                                  const VecParams &prm, cudaStream_t st);
DG_DECLARE_VECOP_LINEAR(2, 0, 0)
DG_DECLARE_VECOP_LINEAR(2, 0, 1)
DG_DECLARE_VECOP_LINEAR(2, 1, 0)
DG_DECLARE_VECOP_LINEAR(2, 1, 1)
DG_DECLARE_VECOP_LINEAR(3, 0, 0)
DG_DECLARE_VECOP_LINEAR(3, 0, 1)
DG_DECLARE_VECOP_LINEAR(3, 1, 0)
DG_DECLARE_VECOP_LINEAR(3, 1, 1)
#undef DG_DECLARE_VECOP_LINEAR

#define DG_DEFINE_VECOP_LINEAR(D, CI, CO)                                                     \
  template <>                                                                                   \
  int vecop_linear_dim<D, CI, CO>(dg_ctx * c, const double *src, double *dst,                   \
                                  const VecParams &prm, cudaStream_t st) {                      \
    switch (c->n) {                                                                             \
      case 2: return launch_vecop<D, 2, 2, (CI ? 1 : D), (CO ? 1 : D)>(c, src, dst, prm, c->basis, st); \
      case 3: return launch_vecop<D, 3, 3, (CI ? 1 : D), (CO ? 1 : D)>(c, src, dst, prm, c->basis, st); \
      case 4: return launch_vecop<D, 4, 4, (CI ? 1 : D), (CO ? 1 : D)>(c, src, dst, prm, c->basis, st); \
      case 5: return launch_vecop<D, 5, 5, (CI ? 1 : D), (CO ? 1 : D)>(c, src, dst, prm, c->basis, st); \
      case 6: return launch_vecop<D, 6, 6, (CI ? 1 : D), (CO ? 1 : D)>(c, src, dst, prm, c->basis, st); \
      case 7: return launch_vecop<D, 7, 7, (CI ? 1 : D), (CO ? 1 : D)>(c, src, dst, prm, c->basis, st); \
      case 8: return launch_vecop<D, 8, 8, (CI ? 1 : D), (CO ? 1 : D)>(c, src, dst, prm, c->basis, st); \
    }                                                                                           \
    return inval("unsupported degree");                                                         \
  }

// convective term on the over-integration rule (vec_over.cu)
int vecop_over(dg_ctx *c, const double *src, double *dst, const VecParams &prm, cudaStream_t st);

}  // namespace dg
