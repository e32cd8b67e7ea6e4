// ps_kern_f32r.cu — streaming, temporal-blocking and first-step kernels for
// (float, ARITH_REF); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE(f32r, float, ARITH_REF)
}  // namespace ps
