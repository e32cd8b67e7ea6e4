// ps_kern_f64.cu — streaming, temporal-blocking and first-step kernels for
// (double, ARITH_REF); see ps_common.cuh.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE(f64, double, ARITH_REF)
}  // namespace ps
