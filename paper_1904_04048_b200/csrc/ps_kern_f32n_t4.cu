// ps_kern_f32n_t4.cu — fused kernels of depth 4 for (float, ARITH_NATIVE); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE_TB(f32n, float, ARITH_NATIVE, 4)
}  // namespace ps
