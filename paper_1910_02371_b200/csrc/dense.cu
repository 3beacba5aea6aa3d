// dense.cu -- epilogue kernels of the dense CP-ALS sweep (BASELINE cfg 4).
//
// A sweep computes T = X_(IJ x K) C once (cpfit_dense_xc, dense_dmma.cu /
// dense_tc.cu; C does not change while modes 0 and 1 update) and reduces it:
//   M0[i, r] = sum_j T[i,j,r] B[j,r]   (cpfit_dense_reduce, axis 1)
//   M1[j, r] = sum_i T[i,j,r] A[i,r]   (cpfit_dense_reduce, axis 0, with the new A)
// Both reductions read T once, coalesced, with fixed-order partial sums
// (deterministic).  cpfit_khatri_rao materialises KR(A, B) for callers that
// want it; the dense MTTKRP itself never does (it forms KR tiles in smem).
//
// Reference: no dense path exists in the reference; its oracle
// is kernels.mttkrp on a fully observed SparseTensor (kernels.py:46-91).
#include "common.cuh"

namespace cpfit {

// axis 1: out[i, r] = sum_j T[i,j,r] W[j,r]; one CTA per i, thread (slice, r) sums the
// j of its slice, slices combined in order through shared memory.
// axis 0: out[j, r] = sum_i T[i,j,r] W[i,r]; one CTA per block of JB j's, thread
// (slice, j, r) sums the i of its slice.  Both read T coalesced (contiguous (j, r)).
template <typename T>
__global__ void dense_reduce_kernel(int64_t I, int64_t J, int R, int JB, int S,
                                    const T *__restrict__ Tm, const T *__restrict__ W, int axis,
                                    T *__restrict__ out) {
  extern __shared__ double red[];
  const int lanes = (axis == 1 ? 1 : JB) * R;  // outputs per CTA
  const int t = threadIdx.x;
  const int o = t % lanes, sl = t / lanes;
  double acc = 0.0;
  if (sl < S) {
    if (axis == 1) {
      const int64_t i = blockIdx.x;
      const int r = o;
      const int64_t per = (J + S - 1) / S, j0 = sl * per, j1 = min(J, j0 + per);
      const T *tp = Tm + i * J * R + r;
      for (int64_t j = j0; j < j1; ++j) acc += (double)tp[j * R] * (double)__ldg(W + j * R + r);
    } else {
      const int64_t j = (int64_t)blockIdx.x * JB + o / R;
      const int r = o % R;
      if (j < J) {
        const int64_t per = (I + S - 1) / S, i0 = sl * per, i1 = min(I, i0 + per);
        const T *tp = Tm + j * R + r;
        for (int64_t i = i0; i < i1; ++i)
          acc += (double)tp[i * J * R] * (double)__ldg(W + i * R + r);
      }
    }
  }
  red[t] = acc;
  __syncthreads();
  if (sl == 0) {
    double tot = red[o];
    for (int k = 1; k < S; ++k) tot += red[k * lanes + o];
    const int64_t row = axis == 1 ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * JB + o / R;
    if (row < (axis == 1 ? I : J)) out[row * R + o % R] = (T)tot;
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
  if (I < 1 || J < 1 || rank < 1 || rank > 1024 || (axis != 0 && axis != 1)) {
    set_error("invalid dense_reduce arguments");
    return CPFIT_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  // axis 1: R lanes x S slices (<= 256 threads); axis 0: JB j's x R lanes x S slices
  int JB = 1, S;
  if (axis == 1) {
    S = 256 / rank > 0 ? 256 / rank : 1;
  } else {
    JB = 256 / rank > 0 ? 256 / rank : 1;
    S = 1024 / (JB * rank) < 4 ? (1024 / (JB * rank) > 0 ? 1024 / (JB * rank) : 1) : 4;
  }
  const int threads = (axis == 1 ? 1 : JB) * rank * S;
  const unsigned grid = (unsigned)(axis == 1 ? I : (J + JB - 1) / JB);
  const size_t shm = (size_t)threads * sizeof(double);
  if (dtype == CPFIT_F64)
    dense_reduce_kernel<double><<<grid, threads, shm, s>>>(I, J, rank, JB, S, (const double *)Tm,
                                                           (const double *)W, axis, (double *)out);
  else if (dtype == CPFIT_F32)
    dense_reduce_kernel<float><<<grid, threads, shm, s>>>(I, J, rank, JB, S, (const float *)Tm,
                                                          (const float *)W, axis, (float *)out);
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
