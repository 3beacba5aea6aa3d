// dense.cu -- dense-tensor MTTKRP helpers (BASELINE cfg 4) for sm_100a.
//
// The dense MTTKRP einsum('ijk,jr,kr->ir') is split into one plain GEMM and
// a bandwidth-bound epilogue:
//   modes 0 / 1:  T[i, j, :] = X[i, j, :] @ C     (plain DGEMM, (I*J x K)(K x R))
//                 M0[i, r] = sum_j T[i,j,r] B[j,r]  (cpfit_dense_reduce, axis 1)
//                 M1[j, r] = sum_i T[i,j,r] A[i,r]  (cpfit_dense_reduce, axis 0)
//   mode 2:       KR[(i,j), r] = A[i,r] B[j,r]      (cpfit_khatri_rao)
//                 M2 = X^T (K x I*J) @ KR           (plain DGEMM)
// so a CP-ALS sweep needs two GEMMs (T is shared by modes 0 and 1 because C
// does not change between them).  The epilogue kernels sum in a fixed order
// (thread per output element): deterministic.
//
// Reference: no dense path exists in the reference; its oracle
// is kernels.mttkrp on a fully observed SparseTensor (kernels.py:46-91).
#include "common.cuh"

namespace cpfit {

template <typename T>
__global__ void dense_reduce_kernel(int64_t I, int64_t J, int R, const T *__restrict__ Tm,
                                    const T *__restrict__ W, int axis, T *__restrict__ out) {
  const int64_t rows = axis == 1 ? I : J;
  const int64_t total = rows * R;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = o / R;
    const int r = (int)(o - row * R);
    double acc = 0.0;
    if (axis == 1) {
      const T *t = Tm + row * J * R + r;
      for (int64_t j = 0; j < J; ++j) acc += (double)t[j * R] * (double)__ldg(W + j * R + r);
    } else {
      const T *t = Tm + row * R + r;
      for (int64_t i = 0; i < I; ++i)
        acc += (double)t[i * J * R] * (double)__ldg(W + i * R + r);
    }
    out[o] = (T)acc;
  }
}

template <typename T>
__global__ void khatri_rao_kernel(int64_t I, int64_t J, int R, const T *__restrict__ A,
                                  const T *__restrict__ B, T *__restrict__ out) {
  const int64_t total = I * J * R;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ij = o / R;
    const int r = (int)(o - ij * R);
    const int64_t i = ij / J, j = ij - i * J;
    out[o] = __ldg(A + i * R + r) * __ldg(B + j * R + r);
  }
}

}  // namespace cpfit

using namespace cpfit;

extern "C" {

int cpfit_dense_reduce(int dtype, int64_t I, int64_t J, int rank, const void *Tm, const void *W,
                       int axis, void *out, void *stream) {
  if (I < 1 || J < 1 || rank < 1 || (axis != 0 && axis != 1)) {
    set_error("invalid dense_reduce arguments");
    return CPFIT_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t total = (axis == 1 ? I : J) * rank;
  if (dtype == CPFIT_F64)
    dense_reduce_kernel<double><<<grid_for(total, 256), 256, 0, s>>>(
        I, J, rank, (const double *)Tm, (const double *)W, axis, (double *)out);
  else if (dtype == CPFIT_F32)
    dense_reduce_kernel<float><<<grid_for(total, 256), 256, 0, s>>>(
        I, J, rank, (const float *)Tm, (const float *)W, axis, (float *)out);
  else {
    set_error("unknown dtype %d", dtype);
    return CPFIT_EINVAL;
  }
  CPFIT_LAUNCH_CHECK("dense_reduce");
  return CPFIT_OK;
}

int cpfit_khatri_rao(int dtype, int64_t I, int64_t J, int rank, const void *A, const void *B,
                     void *out, void *stream) {
  if (I < 1 || J < 1 || rank < 1) {
    set_error("invalid khatri_rao arguments");
    return CPFIT_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t total = I * J * rank;
  if (dtype == CPFIT_F64)
    khatri_rao_kernel<double><<<grid_for(total, 256, 4), 256, 0, s>>>(
        I, J, rank, (const double *)A, (const double *)B, (double *)out);
  else if (dtype == CPFIT_F32)
    khatri_rao_kernel<float><<<grid_for(total, 256, 4), 256, 0, s>>>(
        I, J, rank, (const float *)A, (const float *)B, (float *)out);
  else {
    set_error("unknown dtype %d", dtype);
    return CPFIT_EINVAL;
  }
  CPFIT_LAUNCH_CHECK("khatri_rao");
  return CPFIT_OK;
}

}  // extern "C"
