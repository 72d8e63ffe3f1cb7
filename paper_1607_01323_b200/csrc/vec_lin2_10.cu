// Instantiations of the quadrature-point operators: dim 2, (input, output)
// component pattern 10 (0 = dim components, 1 = scalar).  See vecops_impl.cuh.
#include "vecops_impl.cuh"

namespace dg {
DG_DEFINE_VECOP_LINEAR(2, 1, 0)
}  // namespace dg
