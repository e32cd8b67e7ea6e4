// ps_kern_f32n.cu — streaming, temporal-blocking and first-step kernels for
// (float, ARITH_NATIVE); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE(f32n, float, ARITH_NATIVE)
}  // namespace ps
