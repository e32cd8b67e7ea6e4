// ps_kern_f64_t2.cu — fused kernels of depth 2 for (double, ARITH_REF); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE_TB(f64, double, ARITH_REF, 2)
}  // namespace ps
