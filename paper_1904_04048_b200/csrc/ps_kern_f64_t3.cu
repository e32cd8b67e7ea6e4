// ps_kern_f64_t3.cu — fused kernels of depth 3 for (double, ARITH_REF); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE_TB(f64, double, ARITH_REF, 3)
}  // namespace ps
