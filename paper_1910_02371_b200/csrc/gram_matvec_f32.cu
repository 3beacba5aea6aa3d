// gram_matvec_f32.cu -- instantiation unit: Gram-free matvec (MV) kernels for float.
#include "sparse_kernels.cuh"

namespace cpfit {
template int dispatch_mttkrp_mv<float>(const MttkrpParams<float> &p, int vec, cudaStream_t s);
}  // namespace cpfit
