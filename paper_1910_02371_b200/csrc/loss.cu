// loss.cu -- generalized (non least-squares) losses on the device.
//
// The reference evaluates its pluggable elementwise losses on host arrays
// (losses.py:22-104): phi / dphi / d2phi of (t, m) with the Poisson log link
// clamping m at 50 before exp and counting the clamp events.  Here the
// built-in losses run as device epilogues: fused into TTTP for the
// derivative tensors of ALS / SGD / Gauss-Newton (cpfit_tttp_loss,
// sparse_api.cu), elementwise for objective values (cpfit_loss_eval), and
// the inner-Newton CCD++ column step of optim.py:269-294 as three small
// kernels around two R = 1 segmented sums (cpfit_mttkrp).
#include "common.cuh"

namespace cpfit {

template <typename T>
__global__ void loss_eval_kernel(int loss, int64_t n, const T *__restrict__ t,
                                 const T *__restrict__ m, T *__restrict__ phi,
                                 T *__restrict__ d1o, T *__restrict__ d2o,
                                 unsigned long long *__restrict__ clamped) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count so the ballot sees every lane
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n;
       base += stride) {
    const int64_t k = base + lane;
    bool cl = false;
    if (k < n) {
      double f, a, b;
      cl = loss_eval1(loss, (double)t[k], (double)m[k], f, a, b);
      if (phi) phi[k] = (T)f;
      if (d1o) d1o[k] = (T)a;
      if (d2o) d2o[k] = (T)b;
    }
    const unsigned nc = __ballot_sync(0xffffffffu, cl);
    if (nc && lane == 0 && clamped) atomicAdd(clamped, (unsigned long long)__popc(nc));
  }
}

// Inner-Newton CCD++ weights (optim.py:276-286), canonical entry order:
// part = prod_{p != mode} col_p[i_p] (p ascending), w1 = part * dphi,
// w2 = (part * part) * d2phi.  part is kept for the model update.
__global__ void ccd_gen_weights_kernel(int order, int mode, int loss, int64_t n,
                                       const int32_t *const *__restrict__ coords_unused,
                                       CpfitCols cols, const double *__restrict__ t,
                                       const double *__restrict__ model, double *__restrict__ w1,
                                       double *__restrict__ w2, double *__restrict__ part_out,
                                       unsigned long long *__restrict__ clamped) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n;
       base += stride) {
    const int64_t e = base + lane;
    bool cl = false;
    if (e < n) {
      double part = 1.0;
#pragma unroll
      for (int q = 0; q < CPFIT_MAXN; ++q) {
        if (q >= order) break;
        if (q == mode) continue;
        part = __dmul_rn(part, __ldg(cols.col[q] + __ldg(cols.idx[q] + e)));
      }
      double f, d1, d2;
      if (loss == 2) {  // derivatives evaluated by the caller (user-registered loss)
        d1 = t[e];
        d2 = model[e];
      } else {
        cl = loss_eval1(loss, t[e], model[e], f, d1, d2);
      }
      w1[e] = __dmul_rn(part, d1);
      w2[e] = __dmul_rn(__dmul_rn(part, part), d2);
      part_out[e] = part;
    }
    // raw count of clamped entries (the caller scales by its exp() calls)
    const unsigned nc = __ballot_sync(0xffffffffu, cl);
    if (nc && lane == 0 && clamped) atomicAdd(clamped, (unsigned long long)__popc(nc));
  }
}

// num += 2 reg col; den += 2 reg; delta = den > 0 ? -num / den : 0; col += delta
// (optim.py:280-289, numpy's evaluation order; reg2 = 2.0 * reg).
__global__ void ccd_gen_update_kernel(int64_t dim, const double *__restrict__ num,
                                      const double *__restrict__ den, double reg2,
                                      double *__restrict__ col, double *__restrict__ delta) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double nm = __dadd_rn(num[i], __dmul_rn(reg2, col[i]));
    const double dn = __dadd_rn(den[i], reg2);
    const double d = dn > 0.0 ? -(nm / dn) : 0.0;
    delta[i] = d;
    col[i] = __dadd_rn(col[i], d);
  }
}

// model += part * delta[i_mode]  (optim.py:290)
__global__ void ccd_gen_model_kernel(int64_t n, const int32_t *__restrict__ idx,
                                     const double *__restrict__ part,
                                     const double *__restrict__ delta, double *__restrict__ model) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    model[e] = __dadd_rn(model[e], __dmul_rn(part[e], __ldg(delta + __ldg(idx + e))));
}

static int fetch_count(unsigned long long *dev, int64_t *host, cudaStream_t s) {
  unsigned long long h = 0;
  CPFIT_CUDA(cudaMemcpyAsync(&h, dev, sizeof(h), cudaMemcpyDeviceToHost, s));
  CPFIT_CUDA(cudaStreamSynchronize(s));
  *host = (int64_t)h;
  return CPFIT_OK;
}

}  // namespace cpfit

using namespace cpfit;

extern "C" {

int cpfit_loss_eval(int loss, int dtype, int64_t n, const void *t, const void *m, void *phi,
                    void *dphi, void *d2phi, int64_t *clamped, void *stream) {
  if (loss < 0 || loss > 1) { set_error("unknown loss id %d", loss); return CPFIT_EINVAL; }
  if (n <= 0) {
    if (clamped) *clamped = 0;
    return CPFIT_OK;
  }
  if (!t || !m) { set_error("null input"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  Scratch<unsigned long long> cnt(s);
  if (clamped) {
    CPFIT_TRY(cnt.alloc(1));
    CPFIT_CUDA(cudaMemsetAsync(cnt.ptr, 0, sizeof(unsigned long long), s));
  }
  const unsigned grid = grid_for(n, 256, 4);
  if (dtype == CPFIT_F64)
    loss_eval_kernel<double><<<grid, 256, 0, s>>>(loss, n, (const double *)t,
                                                   (const double *)m, (double *)phi,
                                                   (double *)dphi, (double *)d2phi, cnt.ptr);
  else if (dtype == CPFIT_F32)
    loss_eval_kernel<float><<<grid, 256, 0, s>>>(loss, n, (const float *)t, (const float *)m,
                                                 (float *)phi, (float *)dphi, (float *)d2phi,
                                                 cnt.ptr);
  else {
    set_error("unknown dtype %d", dtype);
    return CPFIT_EINVAL;
  }
  CPFIT_LAUNCH_CHECK("loss_eval");
  if (clamped) return fetch_count(cnt.ptr, clamped, s);
  return CPFIT_OK;
}

int cpfit_ccd_gen_weights(cpfit_pattern *pt, int mode, int loss, const double *const *cols,
                          const double *t, const double *model, double *w1, double *w2,
                          double *part, int64_t *clamped, void *stream) {
  if (!pt || mode < 0 || mode >= pt->order) { set_error("mode %d out of range", mode); return CPFIT_EINVAL; }
  if (loss < 0 || loss > 2) { set_error("unknown loss id %d", loss); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (clamped) *clamped = 0;
  if (pt->nnz == 0) return CPFIT_OK;
  CpfitCols c{};
  for (int q = 0; q < pt->order; ++q) {
    if (q != mode && !cols[q]) { set_error("column of mode %d is null", q); return CPFIT_EINVAL; }
    c.col[q] = cols[q];
    c.idx[q] = pt->coords[q];
  }
  Scratch<unsigned long long> cnt(s);
  if (clamped) {
    CPFIT_TRY(cnt.alloc(1));
    CPFIT_CUDA(cudaMemsetAsync(cnt.ptr, 0, sizeof(unsigned long long), s));
  }
  ccd_gen_weights_kernel<<<grid_for(pt->nnz, 256, 4), 256, 0, s>>>(
      pt->order, mode, loss, pt->nnz, nullptr, c, t, model, w1, w2, part, cnt.ptr);
  CPFIT_LAUNCH_CHECK("ccd_gen_weights");
  if (clamped) return fetch_count(cnt.ptr, clamped, s);
  return CPFIT_OK;
}

int cpfit_ccd_gen_update(int64_t dim, const double *num, const double *den, double reg,
                         double *col, double *delta, void *stream) {
  if (dim <= 0) return CPFIT_OK;
  ccd_gen_update_kernel<<<grid_for(dim, 256), 256, 0, (cudaStream_t)stream>>>(
      dim, num, den, 2.0 * reg, col, delta);
  CPFIT_LAUNCH_CHECK("ccd_gen_update");
  return CPFIT_OK;
}

int cpfit_ccd_gen_model(cpfit_pattern *pt, int mode, const double *part, const double *delta,
                        double *model, void *stream) {
  if (!pt || mode < 0 || mode >= pt->order) { set_error("mode %d out of range", mode); return CPFIT_EINVAL; }
  if (pt->nnz == 0) return CPFIT_OK;
  ccd_gen_model_kernel<<<grid_for(pt->nnz, 256, 4), 256, 0, (cudaStream_t)stream>>>(
      pt->nnz, pt->coords[mode], part, delta, model);
  CPFIT_LAUNCH_CHECK("ccd_gen_model");
  return CPFIT_OK;
}

}  // extern "C"
