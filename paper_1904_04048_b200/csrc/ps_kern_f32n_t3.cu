// ps_kern_f32n_t3.cu — fused kernels of depth 3 for (float, ARITH_NATIVE); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE_TB(f32n, float, ARITH_NATIVE, 3)
}  // namespace ps
