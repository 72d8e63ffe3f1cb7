// Instantiations of the quadrature-point operators: dim 3, (input, output)
// component pattern 01 (0 = dim components, 1 = scalar).  See vecops_impl.cuh.
#include "vecops_impl.cuh"

namespace dg {
DG_DEFINE_VECOP_LINEAR(3, 0, 1)
}  // namespace dg
