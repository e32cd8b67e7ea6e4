// ps_kern_f64.cu — streaming and first-step kernels for (double, ARITH_REF); the fused
// (temporally blocked) kernels of this contract are in ps_kern_f64_t<depth>.cu.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE(f64, double, ARITH_REF)
}  // namespace ps
