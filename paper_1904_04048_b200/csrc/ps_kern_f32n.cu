// ps_kern_f32n.cu — streaming and first-step kernels for (float, ARITH_NATIVE); the fused
// (temporally blocked) kernels of this contract are in ps_kern_f32n_t<depth>.cu.
#include "ps_common.cuh"

namespace ps {
PS_TYPED_DEFINE(f32n, float, ARITH_NATIVE)
PS_TYPED_DEFINE_TB_STUB(f32n, 5)
PS_TYPED_DEFINE_TB_STUB(f32n, 6)
}  // namespace ps
