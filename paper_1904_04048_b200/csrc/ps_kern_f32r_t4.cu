// ps_kern_f32r_t4.cu — fused kernels of depth 4 for (float, ARITH_REF); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE_TB(f32r, float, ARITH_REF, 4)
}  // namespace ps
