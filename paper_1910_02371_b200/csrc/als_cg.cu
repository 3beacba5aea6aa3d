// als_cg.cu -- per-row conjugate-gradient state updates of the implicit-CG
// ALS mode update (BASELINE cfg 3 "ALS completion with implicit CG").
//
// The normal equations of one ALS mode are block diagonal: row i solves
// (G_i + reg I) x_i = b_i with G_i = sum_{e in row i} w_e h_e h_e^T.  Instead of
// materialising the I x R x R Gram blocks (3.9 GB for cfg 3 mode 0) the
// product G_i p_i comes from cpfit_gram_matvec (one pass over the nonzeros,
// sparse_kernels.cuh MV kernels) and every row runs its own CG recurrence
// with its own alpha / beta -- the rows are independent systems, so this is
// CG applied to each block, not one global Krylov space.  A row leaves the
// iteration when ||r_i|| <= tol ||b_i|| (pcg_solve's test, optim.py:521-523,
// applied per row) or on nonpositive curvature (optim.py:513-514); finished
// rows are skipped by the next matvec through `active`.
//
// One warp per row, lane = column (+32, ...); scalars in double for both
// dtypes; dot products are xor-butterflies (fixed order, deterministic).
// The reference has no counterpart of this solver (its ALS solves each row
// with LAPACK gesv, kernels.py:259); parity is to the CG tolerance.
#include "common.cuh"

namespace cpfit {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// status[0]: rows still active after this launch; status[1]: non-finite flag
template <typename T, bool INIT>
__global__ void __launch_bounds__(256)
cg_rows_kernel(int64_t nrows, int rank, double reg, double tol, const T *__restrict__ b,
               const T *__restrict__ q, T *__restrict__ x, T *__restrict__ r,
               T *__restrict__ p, double *__restrict__ rho, double *__restrict__ thresh2,
               int32_t *__restrict__ active, unsigned long long *status) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long live = 0;
  bool bad = false;
  for (int64_t i = warp; i < nrows; i += nwarps) {
    const int64_t o = i * rank;
    if constexpr (INIT) {
      // r = b - (q + reg x) with q = G x0 (q == nullptr: x0 = 0), p = r
      double bb = 0.0, rr = 0.0;
      for (int c = lane; c < rank; c += 32) {
        const double bv = (double)b[o + c];
        double rv = bv;
        if (q) rv -= (double)q[o + c] + reg * (double)x[o + c];
        bb += bv * bv;
        rr += rv * rv;
        r[o + c] = (T)rv;
        p[o + c] = (T)rv;
      }
      bb = warp_sum(bb);
      rr = warp_sum(rr);
      const double th = tol * tol * bb;
      // b_i = 0 (e.g. a row without entries): the solution is x_i = 0
      const bool zero_rhs = bb == 0.0;
      if (zero_rhs)
        for (int c = lane; c < rank; c += 32) x[o + c] = T(0);
      const bool on = !zero_rhs && rr > th;
      if (!isfinite(rr) || !isfinite(bb)) bad = true;
      if (lane == 0) {
        rho[i] = rr;
        thresh2[i] = th;
        active[i] = on ? 1 : 0;
      }
      live += on ? 1 : 0;
    } else {
      if (!active[i]) continue;  // warp-uniform
      const double rh = rho[i];
      double pq = 0.0;
      for (int c = lane; c < rank; c += 32) {
        const double pv = (double)p[o + c];
        pq += pv * ((double)q[o + c] + reg * pv);
      }
      pq = warp_sum(pq);
      if (!isfinite(pq)) bad = true;
      if (!(pq > 0.0)) {  // nonpositive curvature: keep the current iterate
        if (lane == 0) active[i] = 0;
        continue;
      }
      const double alpha = rh / pq;
      double rr = 0.0;
      for (int c = lane; c < rank; c += 32) {
        const double pv = (double)p[o + c];
        const double rv = (double)r[o + c] - alpha * ((double)q[o + c] + reg * pv);
        x[o + c] = (T)((double)x[o + c] + alpha * pv);
        r[o + c] = (T)rv;
        rr += rv * rv;
      }
      rr = warp_sum(rr);
      if (!isfinite(rr)) bad = true;
      const bool on = rr > thresh2[i];
      if (on) {
        const double beta = rr / rh;
        for (int c = lane; c < rank; c += 32)
          p[o + c] = (T)((double)r[o + c] + beta * (double)p[o + c]);
      }
      if (lane == 0) {
        rho[i] = rr;
        active[i] = on ? 1 : 0;
      }
      live += on ? 1 : 0;
    }
  }
  if (lane == 0) {
    if (live) atomicAdd(status, live);
    if (bad) atomicExch(status + 1, 1ull);
  }
}

template <typename T>
static int run_cg_rows(bool init, int64_t nrows, int rank, double reg, double tol, const void *b,
                       const void *q, void *x, void *r, void *p, double *rho, double *thresh2,
                       int32_t *active, int64_t *status, cudaStream_t s) {
  CPFIT_CUDA(cudaMemsetAsync(status, 0, sizeof(int64_t), s));  // live count; the flag is sticky
  if (nrows == 0) return CPFIT_OK;
  const unsigned grid = grid_for(nrows * 32, 256);
  if (init)
    cg_rows_kernel<T, true><<<grid, 256, 0, s>>>(nrows, rank, reg, tol, (const T *)b,
                                                 (const T *)q, (T *)x, (T *)r, (T *)p, rho,
                                                 thresh2, active, (unsigned long long *)status);
  else
    cg_rows_kernel<T, false><<<grid, 256, 0, s>>>(nrows, rank, reg, tol, nullptr, (const T *)q,
                                                  (T *)x, (T *)r, (T *)p, rho, thresh2, active,
                                                  (unsigned long long *)status);
  CPFIT_LAUNCH_CHECK("cg_rows_kernel");
  return CPFIT_OK;
}

}  // namespace cpfit

using namespace cpfit;

extern "C" {

int cpfit_cg_rows_init(int dtype, int64_t nrows, int rank, double reg, double tol, const void *b,
                       const void *ax, void *x, void *r, void *p, double *rho, double *thresh2,
                       int32_t *active, int64_t *status, void *stream) {
  if (nrows < 0 || rank < 1) { set_error("bad shape"); return CPFIT_EINVAL; }
  if (!(tol > 0.0 && tol < 1.0)) { set_error("rel_tol must be in (0, 1)"); return CPFIT_EINVAL; }
  if (nrows > 0 && (!b || !x || !r || !p || !rho || !thresh2 || !active || !status)) {
    set_error("null array");
    return CPFIT_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    return run_cg_rows<double>(true, nrows, rank, reg, tol, b, ax, x, r, p, rho, thresh2, active,
                               status, s);
  if (dtype == CPFIT_F32)
    return run_cg_rows<float>(true, nrows, rank, reg, tol, b, ax, x, r, p, rho, thresh2, active,
                              status, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_cg_rows_step(int dtype, int64_t nrows, int rank, double reg, const void *q, void *x,
                       void *r, void *p, double *rho, const double *thresh2, int32_t *active,
                       int64_t *status, void *stream) {
  if (nrows < 0 || rank < 1) { set_error("bad shape"); return CPFIT_EINVAL; }
  if (nrows > 0 && (!q || !x || !r || !p || !rho || !thresh2 || !active || !status)) {
    set_error("null array");
    return CPFIT_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    return run_cg_rows<double>(false, nrows, rank, reg, 0.5, nullptr, q, x, r, p, rho,
                               const_cast<double *>(thresh2), active, status, s);
  if (dtype == CPFIT_F32)
    return run_cg_rows<float>(false, nrows, rank, reg, 0.5, nullptr, q, x, r, p, rho,
                              const_cast<double *>(thresh2), active, status, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

}  // extern "C"
