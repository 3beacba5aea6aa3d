// gn.cu -- kernels of the implicit second-order (Gauss-Newton / Newton) step.
//
// The reference's second-order operator (optim.py:348-464, hessian_matvec /
// _SecondOrderOperator) needs, per CG iteration,
//   z_e = phi2_e * sum_d sum_r X_d[i_d(e), r] * prod_{p != d} A_p[i_p(e), r]
// (the sum of the N TTTPs with one factor slot substituted by its update
// block) followed by one MTTKRP of z per mode.  tttp_subst_kernel computes z
// in ONE pass: every entry gathers its N factor rows and N update rows once
// (2N rows instead of the N^2 of N separate TTTPs) and forms the
// leave-one-out products with prefix / suffix products per column.
// axpby_kernel is the vector update of PCG (optim.py:492-531).
#include "common.cuh"

namespace cpfit {

struct SubstParams {
  int order, rank;
  int64_t nnz;
  const int32_t *idx[CPFIT_MAXN];
  const void *fac[CPFIT_MAXN];
  const void *x[CPFIT_MAXN];
  const void *w;  // nullable: unit weights
  void *out;
};

// LPE lanes per entry (power of two), each owning columns q, q+LPE, ...
template <typename T, int LPE>
__global__ void __launch_bounds__(256) tttp_subst_kernel(const SubstParams p) {
  const int lane = threadIdx.x & 31;
  const int q = lane % LPE;
  constexpr int G = 32 / LPE;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T *__restrict__ const *fac = reinterpret_cast<const T *const *>(p.fac);
  const T *__restrict__ const *xb = reinterpret_cast<const T *const *>(p.x);
  for (int64_t base = warp * G; base < p.nnz; base += nwarps * G) {
    const int64_t e = base + lane / LPE;
    const bool live = e < p.nnz;
    double s = 0.0;
    if (live) {
      uint32_t row[CPFIT_MAXN];
#pragma unroll
      for (int n = 0; n < CPFIT_MAXN; ++n)
        if (n < p.order) row[n] = (uint32_t)__ldg(p.idx[n] + e);
      for (int c = q; c < p.rank; c += LPE) {
        double f[CPFIT_MAXN], xv[CPFIT_MAXN];
#pragma unroll
        for (int n = 0; n < CPFIT_MAXN; ++n) {
          if (n < p.order) {
            const size_t off = (size_t)row[n] * (unsigned)p.rank + c;
            f[n] = (double)__ldg(fac[n] + off);
            xv[n] = (double)__ldg(xb[n] + off);
          }
        }
        // sum_d x_d * prod_{p<d} f_p * prod_{p>d} f_p
        double pre = 1.0, acc = 0.0;
        double suf[CPFIT_MAXN];
        suf[CPFIT_MAXN - 1] = 1.0;
#pragma unroll
        for (int n = CPFIT_MAXN - 1; n > 0; --n)
          suf[n - 1] = (n < p.order) ? suf[n] * f[n] : 1.0;
#pragma unroll
        for (int n = 0; n < CPFIT_MAXN; ++n) {
          if (n < p.order) {
            acc += xv[n] * (pre * suf[n]);
            pre *= f[n];
          }
        }
        s += acc;
      }
    }
#pragma unroll
    for (int o = LPE / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (live && q == 0) {
      const T *w = (const T *)p.w;
      ((T *)p.out)[e] = (T)(w ? (double)w[e] * s : s);
    }
  }
}

template <typename T>
__global__ void axpby_kernel(int64_t n, double a, const T *__restrict__ x, double b,
                             const T *__restrict__ y, T *__restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = (T)(a * (double)x[k] + b * (double)y[k]);
}

template <typename T, int LPE>
static int launch_subst(const SubstParams &p, cudaStream_t s) {
  constexpr int G = 32 / LPE;
  const int64_t warps = (p.nnz + G - 1) / G;
  int64_t blocks = (warps + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  tttp_subst_kernel<T, LPE><<<(unsigned)blocks, 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("tttp_subst");
  return CPFIT_OK;
}

template <typename T>
static int run_subst(const SubstParams &p, cudaStream_t s) {
  if (p.rank <= 1) return launch_subst<T, 1>(p, s);
  if (p.rank <= 2) return launch_subst<T, 2>(p, s);
  if (p.rank <= 4) return launch_subst<T, 4>(p, s);
  if (p.rank <= 8) return launch_subst<T, 8>(p, s);
  if (p.rank <= 16) return launch_subst<T, 16>(p, s);
  return launch_subst<T, 32>(p, s);
}

}  // namespace cpfit

using namespace cpfit;

extern "C" {

int cpfit_tttp_subst(cpfit_pattern *pt, int dtype, int rank, const void *w,
                     const void *const *factors, const void *const *xblocks, void *out,
                     void *stream) {
  if (!pt) { set_error("null pattern"); return CPFIT_EINVAL; }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  SubstParams p{};
  p.order = pt->order;
  p.rank = rank;
  p.nnz = pt->nnz;
  for (int n = 0; n < pt->order; ++n) {
    if (!factors[n] || !xblocks[n]) {
      set_error("factor[%d] and its update block are required", n);
      return CPFIT_EINVAL;
    }
    p.idx[n] = pt->coords[n];
    p.fac[n] = factors[n];
    p.x[n] = xblocks[n];
  }
  p.w = w;
  p.out = out;
  if (pt->nnz == 0) return CPFIT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64) return run_subst<double>(p, s);
  if (dtype == CPFIT_F32) return run_subst<float>(p, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_axpby(int dtype, int64_t n, double a, const void *x, double b, const void *y,
                void *out, void *stream) {
  if (n <= 0) return CPFIT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    axpby_kernel<double><<<grid_for(n, 256, 4), 256, 0, s>>>(n, a, (const double *)x, b,
                                                             (const double *)y, (double *)out);
  else if (dtype == CPFIT_F32)
    axpby_kernel<float><<<grid_for(n, 256, 4), 256, 0, s>>>(n, a, (const float *)x, b,
                                                            (const float *)y, (float *)out);
  else { set_error("unknown dtype %d", dtype); return CPFIT_EINVAL; }
  CPFIT_LAUNCH_CHECK("axpby");
  return CPFIT_OK;
}

}  // extern "C"
