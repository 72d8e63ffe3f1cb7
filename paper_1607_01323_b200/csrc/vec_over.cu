// Instantiations of the convective term on the over-integration rule:
// (n, n_q) pairs floor(3k/2)+1 (reference, basis.py:103-105) and 3(k+1)/2
// (BASELINE literal).  See vecops_impl.cuh.
#include <string>

#include <cstdlib>

#include "vconv.cuh"
#include "vecops_impl.cuh"

namespace dg {

template <int N, int NQ>
static int launch_vconv(dg_ctx *c, double *dst, const VecParams &prm, cudaStream_t st) {
  using C = CvCfg<N, NQ>;
  auto kern = vconv_kernel<N, NQ>;
  static bool attr = false;
  if (!attr) {
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    DG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    attr = true;
  }
  if (c->n_cells == 0) return DG_OK;
  kern<<<(unsigned)c->n_cells, C::T, C::SMEM, st>>>(dst, c->geo(), quad_tab<N, NQ>(c->over), prm,
                                                    c->n_cells);
  DG_LAUNCH_CHECK("vconv_kernel");
  return DG_OK;
}

int vecop_over(dg_ctx *c, const double *src, double *dst, const VecParams &prm, cudaStream_t st) {
  static const bool generic = [] {
    const char *v = getenv("DG_VEC_GENERIC");
    return v && atoi(v) != 0;
  }();
  if (c->dim == 3 && !generic) {
    for (int j = 0; j < prm.n_hist; ++j)
      if (prm.hist[j] == dst) return inval("convective term: dst must not alias a history level");
#define DG_V(NN, QQ) \
  if (c->n == NN && c->nq_over == QQ) return launch_vconv<NN, QQ>(c, dst, prm, st);
    DG_V(2, 2) DG_V(2, 3) DG_V(3, 4) DG_V(4, 5) DG_V(4, 6) DG_V(5, 7) DG_V(6, 8) DG_V(6, 9)
#undef DG_V
  }
#define DG_O(D, NN, QQ) \
  if (c->n == NN && c->nq_over == QQ) return launch_vecop<D, NN, QQ, D, D>(c, src, dst, prm, c->over, st);
  if (c->dim == 3) {
    DG_O(3, 2, 2) DG_O(3, 2, 3) DG_O(3, 3, 4) DG_O(3, 4, 5) DG_O(3, 4, 6)
    DG_O(3, 5, 7) DG_O(3, 6, 8) DG_O(3, 6, 9)
  } else {
    DG_O(2, 2, 2) DG_O(2, 2, 3) DG_O(2, 3, 4) DG_O(2, 4, 5) DG_O(2, 4, 6)
    DG_O(2, 5, 7) DG_O(2, 6, 8) DG_O(2, 6, 9)
  }
#undef DG_O
  return inval("convective term: unsupported (k, n_q) = (" + std::to_string(c->k) + ", " +
               std::to_string(c->nq_over) + "); supported k <= 5 with n_q in "
               "{floor(3k/2)+1, 3(k+1)/2}");
}

}  // namespace dg
