// ps_kern_f32r.cu — streaming and first-step kernels for (float, ARITH_REF); the fused
// (temporally blocked) kernels of this contract are in ps_kern_f32r_t<depth>.cu.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE(f32r, float, ARITH_REF)
PS_TYPED_DEFINE_TB_STUB(f32r, 5)
PS_TYPED_DEFINE_TB_STUB(f32r, 6)
}  // namespace ps
