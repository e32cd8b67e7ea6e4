// ps_kern_f64_t5.cu — fused kernels of depth 5 for (double, ARITH_REF): shared-product
// kernels only (radius 1, Dirichlet); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE_TB(f64, double, ARITH_REF, 5)
}  // namespace ps
