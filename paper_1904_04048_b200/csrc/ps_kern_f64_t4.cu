// ps_kern_f64_t4.cu — fused kernels of depth 4 for (double, ARITH_REF); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE_TB(f64, double, ARITH_REF, 4)
}  // namespace ps
