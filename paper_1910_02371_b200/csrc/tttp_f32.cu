// tttp_f32.cu -- instantiation unit: tttp kernels for float.
#include "sparse_kernels.cuh"

namespace cpfit {
template int dispatch_tttp<float>(const TttpParams<float> &p, int vec, cudaStream_t s);
}  // namespace cpfit
