// ps_kern_f32n_t2.cu — fused kernels of depth 2 for (float, ARITH_NATIVE); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE_TB(f32n, float, ARITH_NATIVE, 2)
}  // namespace ps
