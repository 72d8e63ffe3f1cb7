// Instantiations of the convective term on the over-integration rule:
// (n, n_q) pairs floor(3k/2)+1 (reference, basis.py:103-105) and 3(k+1)/2
// (BASELINE literal).  See vecops_impl.cuh.
#include <string>

#include "vecops_impl.cuh"

namespace dg {

int vecop_over(dg_ctx *c, const double *src, double *dst, const VecParams &prm, cudaStream_t st) {
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
