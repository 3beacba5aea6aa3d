// mttkrp_f32.cu -- instantiation unit: mttkrp kernels for float.
#include "sparse_kernels.cuh"

namespace cpfit {
template int dispatch_mttkrp<float>(const MttkrpParams<float> &p, int vec, cudaStream_t s);
}  // namespace cpfit
