// gram_matvec_f64.cu -- instantiation unit: Gram-free matvec (MV) kernels for double.
#include "sparse_kernels.cuh"

namespace cpfit {
template int dispatch_mttkrp_mv<double>(const MttkrpParams<double> &p, int vec, cudaStream_t s);
}  // namespace cpfit
