// tttp_f64.cu -- instantiation unit: tttp kernels for double.
#include "sparse_kernels.cuh"

namespace cpfit {
template int dispatch_tttp<double>(const TttpParams<double> &p, int vec, cudaStream_t s);
}  // namespace cpfit
