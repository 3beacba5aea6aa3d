// mttkrp_f64.cu -- instantiation unit: mttkrp kernels for double.
#include "sparse_kernels.cuh"

namespace cpfit {
template int dispatch_mttkrp<double>(const MttkrpParams<double> &p, int vec, cudaStream_t s);
}  // namespace cpfit
