// sparse_api.cu -- C-ABI of TTTP / MTTKRP (kernels in sparse_kernels.cuh).
//
// Reference: kernels.tttp (kernels.py:105-149) / _jit.tttp3 (_jit.py:49-59);
// kernels.mttkrp (kernels.py:46-91) / _jit.mttkrp3 (_jit.py:35-47).
#include "sparse_kernels.cuh"

namespace cpfit {

extern template int dispatch_tttp<double>(const TttpParams<double> &, int, cudaStream_t);
extern template int dispatch_tttp<float>(const TttpParams<float> &, int, cudaStream_t);
extern template int dispatch_mttkrp<double>(const MttkrpParams<double> &, int, cudaStream_t);
extern template int dispatch_mttkrp<float>(const MttkrpParams<float> &, int, cudaStream_t);
extern template int dispatch_mttkrp_mv<double>(const MttkrpParams<double> &, int, cudaStream_t);
extern template int dispatch_mttkrp_mv<float>(const MttkrpParams<float> &, int, cudaStream_t);

template <typename T>
static int run_tttp(cpfit_pattern *pt, int rank, const void *vals, const void *const *factors,
                    void *out, cudaStream_t s, int epi = 0, double alpha = 0.0,
                    double beta = 0.0, int64_t begin = 0, int64_t end = -1, int loss = 0,
                    void *out2 = nullptr, unsigned long long *clamped = nullptr) {
  if (end < 0) end = pt->nnz;
  TttpParams<T> p{};
  p.epi = epi;
  p.loss = loss;
  p.out2 = out2 ? (T *)out2 + begin : nullptr;
  p.clamped = clamped;
  p.alpha = (T)alpha;
  p.beta = (T)beta;
  p.rank = rank;
  p.nnz = end - begin;
  p.vals = (const T *)vals + begin;
  p.out = (T *)out + begin;
  int np = 0;
  const void *ptrs[CPFIT_MAXN];
  for (int n = 0; n < pt->order; ++n) {
    if (!factors[n]) continue;
    p.idx[np] = pt->coords[n] + begin;
    p.fac[np] = (const T *)factors[n];
    ptrs[np] = factors[n];
    ++np;
  }
  if (np == 0) {
    set_error("at least one factor matrix must be provided");
    return CPFIT_EINVAL;
  }
  p.np = np;
  if (p.nnz <= 0) return CPFIT_OK;
  return dispatch_tttp<T>(p, pick_vec<T>(rank, ptrs, np), s);
}

// Chunked TTTP whose chunks are copied to host memory while later chunks
// compute: chunk c's copy (on a library-owned copy stream) waits on an event
// recorded after chunk c's kernel, and `s` finally waits on the copy stream,
// so synchronising `s` covers results on both sides.
template <typename T>
static int run_tttp_host(cpfit_pattern *pt, int rank, const void *vals,
                         const void *const *factors, void *dev_out, void *host_out,
                         int64_t chunk, cudaStream_t s, cudaEvent_t *done = nullptr) {
  static cudaStream_t copy_stream[64] = {};
  static cudaEvent_t evs[64][17] = {};
  int dev = 0;
  CPFIT_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) { set_error("device index %d unsupported", dev); return CPFIT_EINVAL; }
  if (!copy_stream[dev]) {
    CPFIT_CUDA(cudaStreamCreateWithFlags(&copy_stream[dev], cudaStreamNonBlocking));
    for (int k = 0; k < 17; ++k)
      CPFIT_CUDA(cudaEventCreateWithFlags(&evs[dev][k], cudaEventDisableTiming));
  }
  const int64_t nnz = pt->nnz;
  if (chunk <= 0) chunk = (nnz + 7) / 8;
  if ((nnz + chunk - 1) / chunk > 16) chunk = (nnz + 15) / 16;
  chunk = (chunk + 31) & ~int64_t(31);
  cudaStream_t cs = copy_stream[dev];
  int k = 0;
  for (int64_t b = 0; b < nnz; b += chunk, ++k) {
    const int64_t e = b + chunk < nnz ? b + chunk : nnz;
    CPFIT_TRY(run_tttp<T>(pt, rank, vals, factors, dev_out, s, 0, 0.0, 0.0, b, e));
    CPFIT_CUDA(cudaEventRecord(evs[dev][k], s));
    CPFIT_CUDA(cudaStreamWaitEvent(cs, evs[dev][k], 0));
    CPFIT_CUDA(cudaMemcpyAsync((T *)host_out + b, (const T *)dev_out + b, (e - b) * sizeof(T),
                               cudaMemcpyDeviceToHost, cs));
  }
  if (done) {
    // no join: `s` runs on while the copies drain; the caller waits on *done
    CPFIT_CUDA(cudaEventCreateWithFlags(done, cudaEventDisableTiming));
    CPFIT_CUDA(cudaEventRecord(*done, cs));
    return CPFIT_OK;
  }
  CPFIT_CUDA(cudaEventRecord(evs[dev][16], cs));
  CPFIT_CUDA(cudaStreamWaitEvent(s, evs[dev][16], 0));
  return CPFIT_OK;
}

// rows of the target mode without entries -> exact zeros (warp per row)
template <typename T>
__global__ void mttkrp_zero_empty_rows(int64_t dim, const int64_t *__restrict__ offsets, int rank,
                                       T *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < dim; i += nwarps) {
    if (offsets[i + 1] != offsets[i]) continue;
    for (int c = lane; c < rank; c += 32) out[i * rank + c] = T(0);
  }
}

template <typename T>
static int run_mttkrp(cpfit_pattern *pt, int mode, int rank, const void *vals, int vals_sorted,
                      const void *const *factors, void *out, cudaStream_t s,
                      const void *xvec = nullptr, const int32_t *row_active = nullptr) {
  const int64_t dim = pt->dims[mode];
  if (pt->nnz == 0) {
    CPFIT_CUDA(cudaMemsetAsync(out, 0, (size_t)dim * rank * sizeof(T), s));
    return CPFIT_OK;
  }
  CPFIT_TRY(ensure_layout(pt, mode, s));
  CpfitModeLayout &L = pt->modes[mode];
  // every non-empty row is stored by its task (or by the combine of its split
  // tasks), so only the rows without entries are zeroed: `out` is written
  // exactly once, which also lets it be pinned host memory (the numpy API
  // passes its result buffer, no separate read-back pass)
  mttkrp_zero_empty_rows<T><<<grid_for(dim * 32, 256), 256, 0, s>>>(dim, L.offsets, rank, (T *)out);
  CPFIT_LAUNCH_CHECK("mttkrp_zero_empty_rows");
  MttkrpParams<T> p{};
  p.rank = rank;
  int np = 0;
  const void *ptrs[CPFIT_MAXN];
  for (int n = 0; n < pt->order; ++n) {
    if (n == mode) continue;
    if (!factors[n]) {
      set_error("factor[%d] is required but missing", n);
      return CPFIT_EINVAL;
    }
    p.idx[np] = L.sorted_idx[n];
    p.fac[np] = (const T *)factors[n];
    ptrs[np] = factors[n];
    ++np;
  }
  p.np = np;
  p.vals = (const T *)vals;
  p.perm = vals_sorted ? nullptr : L.perm;
  p.task_begin = L.task_begin;
  p.task_row = L.task_row;
  p.task_slot = L.task_slot;
  p.ntasks = L.ntasks;
  p.out = (T *)out;
  p.xvec = (const T *)xvec;
  p.row_active = row_active;
  if (xvec) ptrs[np] = xvec;  // alignment of the matvec operand decides the vector width too
  Scratch<T> partial(s);
  if (L.nslots > 0) CPFIT_TRY(partial.alloc((size_t)L.nslots * rank));
  p.partial = partial.ptr;
  if (np == 0) {
    // order-1 tensor: out[i] = sum of values in row i (empty product = 1)
    set_error("mttkrp needs an order >= 2 tensor");
    return CPFIT_EINVAL;
  }
  if (xvec)
    CPFIT_TRY(dispatch_mttkrp_mv<T>(p, pick_vec<T>(rank, ptrs, np + 1), s));
  else
    CPFIT_TRY(dispatch_mttkrp<T>(p, pick_vec<T>(rank, ptrs, np), s));
  if (L.nsplit > 0) {
    combine_partials<T><<<grid_for(L.nsplit * 32, 256), 256, 0, s>>>(
        L.split_row, L.split_slot, L.nsplit, rank, partial.ptr, (T *)out);
    CPFIT_LAUNCH_CHECK("combine_partials");
    if (L.max_slots > COMBINE_LONG) {  // block per long row; the others exit
      const int64_t lb = L.nsplit < (int64_t)num_sms() * 8 ? L.nsplit : (int64_t)num_sms() * 8;
      combine_partials_long<T><<<(unsigned)(lb > 0 ? lb : 1), 256, 0, s>>>(
          L.split_row, L.split_slot, L.nsplit, rank, partial.ptr, (T *)out);
      CPFIT_LAUNCH_CHECK("combine_partials_long");
    }
  }
  return CPFIT_OK;
}

}  // namespace cpfit

using namespace cpfit;

extern "C" {

int cpfit_tttp(cpfit_pattern *p, int dtype, int rank, const void *vals,
               const void *const *factors, void *out, void *stream) {
  if (!p) { set_error("null pattern"); return CPFIT_EINVAL; }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64) return run_tttp<double>(p, rank, vals, factors, out, s);
  if (dtype == CPFIT_F32) return run_tttp<float>(p, rank, vals, factors, out, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_tttp_host(cpfit_pattern *p, int dtype, int rank, const void *vals,
                    const void *const *factors, void *dev_out, void *host_out, int64_t chunk,
                    void *stream) {
  if (!p) { set_error("null pattern"); return CPFIT_EINVAL; }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  if (p->nnz > 0 && (!dev_out || !host_out)) { set_error("null output"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    return run_tttp_host<double>(p, rank, vals, factors, dev_out, host_out, chunk, s);
  if (dtype == CPFIT_F32)
    return run_tttp_host<float>(p, rank, vals, factors, dev_out, host_out, chunk, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_tttp_host_async(cpfit_pattern *p, int dtype, int rank, const void *vals,
                          const void *const *factors, void *dev_out, void *host_out,
                          int64_t chunk, void **done, void *stream) {
  if (!p) { set_error("null pattern"); return CPFIT_EINVAL; }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  if (!done) { set_error("null event out"); return CPFIT_EINVAL; }
  *done = nullptr;
  if (p->nnz > 0 && (!dev_out || !host_out)) { set_error("null output"); return CPFIT_EINVAL; }
  if (p->nnz == 0) return CPFIT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t ev = nullptr;
  int st;
  if (dtype == CPFIT_F64)
    st = run_tttp_host<double>(p, rank, vals, factors, dev_out, host_out, chunk, s, &ev);
  else if (dtype == CPFIT_F32)
    st = run_tttp_host<float>(p, rank, vals, factors, dev_out, host_out, chunk, s, &ev);
  else {
    set_error("unknown dtype %d", dtype);
    return CPFIT_EINVAL;
  }
  *done = (void *)ev;
  return st;
}

int cpfit_event_wait(void *event, int destroy) {
  if (!event) return CPFIT_OK;
  cudaEvent_t ev = (cudaEvent_t)event;
  CPFIT_CUDA(cudaEventSynchronize(ev));
  if (destroy) CPFIT_CUDA(cudaEventDestroy(ev));
  return CPFIT_OK;
}

int cpfit_tttp_axpby(cpfit_pattern *p, int dtype, int rank, const void *vals,
                     const void *const *factors, double alpha, double beta, void *out,
                     void *stream) {
  if (!p) { set_error("null pattern"); return CPFIT_EINVAL; }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64) return run_tttp<double>(p, rank, vals, factors, out, s, 1, alpha, beta);
  if (dtype == CPFIT_F32) return run_tttp<float>(p, rank, vals, factors, out, s, 1, alpha, beta);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_tttp_loss(cpfit_pattern *p, int dtype, int rank, const void *t_vals,
                    const void *const *factors, int loss, void *dphi, void *d2phi,
                    int64_t *clamped, void *stream) {
  if (!p) { set_error("null pattern"); return CPFIT_EINVAL; }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  if (loss < 0 || loss > 1) { set_error("unknown loss id %d", loss); return CPFIT_EINVAL; }
  if (p->nnz > 0 && (!t_vals || !dphi || !d2phi)) { set_error("null array"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  Scratch<unsigned long long> cnt(s);
  if (clamped) {
    CPFIT_TRY(cnt.alloc(1));
    CPFIT_CUDA(cudaMemsetAsync(cnt.ptr, 0, sizeof(unsigned long long), s));
  }
  int st;
  if (dtype == CPFIT_F64)
    st = run_tttp<double>(p, rank, t_vals, factors, dphi, s, 2, 0.0, 0.0, 0, -1, loss, d2phi,
                          cnt.ptr);
  else if (dtype == CPFIT_F32)
    st = run_tttp<float>(p, rank, t_vals, factors, dphi, s, 2, 0.0, 0.0, 0, -1, loss, d2phi,
                         cnt.ptr);
  else {
    set_error("unknown dtype %d", dtype);
    return CPFIT_EINVAL;
  }
  if (st != CPFIT_OK) return st;
  if (clamped) {
    unsigned long long h = 0;
    CPFIT_CUDA(cudaMemcpyAsync(&h, cnt.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
    CPFIT_CUDA(cudaStreamSynchronize(s));
    *clamped = (int64_t)h;
  }
  return CPFIT_OK;
}

int cpfit_mttkrp(cpfit_pattern *p, int mode, int dtype, int rank, const void *vals,
                 int vals_sorted, const void *const *factors, void *out, void *stream) {
  if (!p || mode < 0 || mode >= p->order) {
    set_error("mode %d out of range for order-%d tensor", mode, p ? p->order : 0);
    return CPFIT_EINVAL;
  }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    return run_mttkrp<double>(p, mode, rank, vals, vals_sorted, factors, out, s);
  if (dtype == CPFIT_F32)
    return run_mttkrp<float>(p, mode, rank, vals, vals_sorted, factors, out, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_gram_matvec(cpfit_pattern *p, int mode, int dtype, int rank, const void *weights,
                      int weights_sorted, const void *const *factors, const void *x,
                      const int32_t *row_active, void *out, void *stream) {
  if (!p || mode < 0 || mode >= p->order) {
    set_error("mode %d out of range for order-%d tensor", mode, p ? p->order : 0);
    return CPFIT_EINVAL;
  }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  if (!x || !out) { set_error("null operand"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    return run_mttkrp<double>(p, mode, rank, weights, weights_sorted, factors, out, s, x,
                              row_active);
  if (dtype == CPFIT_F32)
    return run_mttkrp<float>(p, mode, rank, weights, weights_sorted, factors, out, s, x,
                             row_active);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

}  // extern "C"
