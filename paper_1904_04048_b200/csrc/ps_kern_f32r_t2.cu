// ps_kern_f32r_t2.cu — fused kernels of depth 2 for (float, ARITH_REF); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE_TB(f32r, float, ARITH_REF, 2)
}  // namespace ps
