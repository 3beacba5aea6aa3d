// elementwise.cu -- Bernoulli sampling (bit-exact numpy Philox4x64-10),
// value gathers, deterministic reductions and the SGD factor update.
//
// Reference: SparseTensor.sample (core.py:173-183) with RngState's numpy
// Philox stream (core.py:25-46); sgd_sweep's update (optim.py:313-330);
// objective / rmse sums (losses.py:126-150, optim.py:642-652).
#include "common.cuh"

namespace cpfit {

// ---------------------------------------------------------------------------
// Philox4x64-10, exactly numpy.random.Philox: draw e of Generator.random()
// is word e % 4 of philox(counter = [e/4 + 1, 0, 0, 0], key), mapped to
// (w >> 11) * 2^-53.

__device__ __forceinline__ void philox4x64_10(uint64_t c0, uint64_t key0, uint64_t key1,
                                              uint64_t (&out)[4]) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
  uint64_t x0 = c0, x1 = 0, x2 = 0, x3 = 0, k0 = key0, k1 = key1;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint64_t hi0 = __umul64hi(M0, x0), lo0 = M0 * x0;
    const uint64_t hi1 = __umul64hi(M1, x2), lo1 = M1 * x2;
    const uint64_t n0 = hi1 ^ x1 ^ k0, n2 = hi0 ^ x3 ^ k1;
    x0 = n0; x1 = lo1; x2 = n2; x3 = lo0;
    k0 += W0; k1 += W1;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

constexpr int SMP_THREADS = 256;
constexpr int SMP_BLOCKS_PER_THREAD = 8;  // Philox blocks (4 draws each) per thread: 32 bits

// u = (w >> 11) * 2^-53 < rate  <=>  (w >> 11) < ceil(rate * 2^53): scaling by a
// power of two is exact, so the integer test decides exactly like numpy's
// double comparison.
__host__ __device__ inline uint64_t sample_threshold(double rate) {
  return (uint64_t)ceil(rate * 9007199254740992.0);
}

// keep-bits of the draws of local entries [4*b - phase, ...): one Philox call
// serves 4 consecutive global entries.  Bit j*4+w = word w of block j.
__device__ __forceinline__ uint32_t sample_bits(int64_t tile, int64_t n, int64_t off,
                                                uint64_t key0, uint64_t key1, uint64_t thr,
                                                int64_t *first_local) {
  // global philox blocks covering local [0, n): g = off .. off + n - 1
  const int64_t gb0 = off >> 2;  // first global block
  const int64_t b = gb0 + tile * (SMP_THREADS * SMP_BLOCKS_PER_THREAD) +
                    (int64_t)threadIdx.x * SMP_BLOCKS_PER_THREAD;
  *first_local = b * 4 - off;  // local index of word 0 of block b
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < SMP_BLOCKS_PER_THREAD; ++j) {
    const int64_t lb = (b + j) * 4 - off;  // local index of word 0
    if (lb + 3 < 0 || lb >= n) continue;
    uint64_t w[4];
    philox4x64_10((uint64_t)(b + j) + 1u, key0, key1, w);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t l = lb + q;
      if (l >= 0 && l < n && (w[q] >> 11) < thr) bits |= 1u << (j * 4 + q);
    }
  }
  return bits;
}

// Pass 1 (the only Philox pass): keep-masks, one 32-bit word per thread and
// tile, plus per-tile survivor counts.
__global__ void __launch_bounds__(SMP_THREADS)
sample_count_kernel(int64_t n, int64_t off, uint64_t key0, uint64_t key1, uint64_t thr,
                    int64_t ntiles, int64_t *tile_counts, uint32_t *__restrict__ masks) {
  __shared__ int warp_tot[SMP_THREADS / 32];
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int64_t fl;
    const uint32_t bits = sample_bits(tile, n, off, key0, key1, thr, &fl);
    masks[tile * SMP_THREADS + threadIdx.x] = bits;
    int c = __popc(bits);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t s = 0;
      for (int w = 0; w < SMP_THREADS / 32; ++w) s += warp_tot[w];
      tile_counts[tile] = s;
    }
    __syncthreads();
  }
}

// Pass 2: compaction driven by the stored masks (no Philox recomputation).
__global__ void __launch_bounds__(SMP_THREADS)
sample_select_kernel(int64_t n, int64_t off, int64_t ntiles,
                     const int64_t *__restrict__ tile_offsets,
                     const uint32_t *__restrict__ masks, int32_t *__restrict__ kept) {
  __shared__ int warp_pre[SMP_THREADS / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b = (off >> 2) + tile * (SMP_THREADS * SMP_BLOCKS_PER_THREAD) +
                      (int64_t)threadIdx.x * SMP_BLOCKS_PER_THREAD;
    const int64_t fl = b * 4 - off;
    uint32_t bits = masks[tile * SMP_THREADS + threadIdx.x];
    const int c = __popc(bits);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_pre[w] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int k = 0; k < SMP_THREADS / 32; ++k) {
        int t = warp_pre[k];
        warp_pre[k] = run;
        run += t;
      }
    }
    __syncthreads();
    int64_t pos = tile_offsets[tile] + warp_pre[w] + (incl - c);
    while (bits) {
      const int bit = __ffs(bits) - 1;
      bits &= bits - 1;
      kept[pos++] = (int32_t)(fl + bit);  // bit = j*4 + q -> local fl + 4j + q
    }
    __syncthreads();
  }
}

struct GatherCoords {
  int order;
  const int32_t *src[CPFIT_MAXN];
  int32_t *dst[CPFIT_MAXN];
};

__global__ void gather_coords_kernel(const int32_t *__restrict__ idx, int64_t n,
                                     GatherCoords g) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = idx[k];
#pragma unroll
    for (int m = 0; m < CPFIT_MAXN; ++m)
      if (m < g.order) g.dst[m][k] = __ldg(g.src[m] + e);
  }
}

template <typename T>
__global__ void gather_values_kernel(const int32_t *__restrict__ idx, int64_t n,
                                     const T *__restrict__ in, T *__restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = __ldg(in + idx[k]);
}

// ---------------------------------------------------------------------------
// deterministic reductions: fixed grid, fixed per-block order, then one block

constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = 592;  // 4 x 148 SMs; fixed so the order never varies

template <typename T, int OP>  // OP 0: sum x^2, 1: sum (x - y)^2, 2: sum x*y, 3: sum x
__global__ void __launch_bounds__(RED_THREADS)
reduce_partials(int64_t n, const T *__restrict__ x, const T *__restrict__ y,
                double *__restrict__ partial) {
  double acc = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; k < n;
       k += (int64_t)RED_BLOCKS * RED_THREADS) {
    const double a = (double)x[k];
    if (OP == 0) acc += a * a;
    if (OP == 1) { const double d = a - (double)y[k]; acc += d * d; }
    if (OP == 2) acc += a * (double)y[k];
    if (OP == 3) acc += a;
  }
  __shared__ double sm[RED_THREADS];
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int s = RED_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sm[0];
}

__global__ void reduce_final(const double *__restrict__ partial, int n, double *out) {
  __shared__ double sm[1024];
  double acc = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) acc += partial[k];
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

template <typename T>
static int run_reduce(int op, int64_t n, const T *x, const T *y, double *result,
                      cudaStream_t s) {
  Scratch<double> part(s);
  CPFIT_TRY(part.alloc(RED_BLOCKS + 1));
  if (op == 0) reduce_partials<T, 0><<<RED_BLOCKS, RED_THREADS, 0, s>>>(n, x, y, part.ptr);
  if (op == 1) reduce_partials<T, 1><<<RED_BLOCKS, RED_THREADS, 0, s>>>(n, x, y, part.ptr);
  if (op == 2) reduce_partials<T, 2><<<RED_BLOCKS, RED_THREADS, 0, s>>>(n, x, y, part.ptr);
  if (op == 3) reduce_partials<T, 3><<<RED_BLOCKS, RED_THREADS, 0, s>>>(n, x, y, part.ptr);
  CPFIT_LAUNCH_CHECK("reduce_partials");
  reduce_final<<<1, 1024, 0, s>>>(part.ptr, RED_BLOCKS, part.ptr + RED_BLOCKS);
  CPFIT_LAUNCH_CHECK("reduce_final");
  CPFIT_CUDA(cudaMemcpyAsync(result, part.ptr + RED_BLOCKS, sizeof(double),
                             cudaMemcpyDeviceToHost, s));
  CPFIT_CUDA(cudaStreamSynchronize(s));
  return CPFIT_OK;
}

// ---------------------------------------------------------------------------
// SGD update: out = (a - step * g) - shrink * a, evaluated in numpy's order
// without contraction (optim.py:324-325), plus a non-finite flag.

template <typename T>
__global__ void sgd_update_kernel(int64_t n, const T *__restrict__ a, const T *__restrict__ g,
                                  double step, double shrink, T *__restrict__ out, int *flag) {
  int bad = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    T v;
    if constexpr (sizeof(T) == 8) {
      const double t1 = __dmul_rn(step, (double)g[k]);
      const double t2 = __dsub_rn((double)a[k], t1);
      const double t3 = __dmul_rn(shrink, (double)a[k]);
      v = (T)__dsub_rn(t2, t3);
    } else {
      const float t1 = __fmul_rn((float)step, (float)g[k]);
      const float t2 = __fsub_rn((float)a[k], t1);
      const float t3 = __fmul_rn((float)shrink, (float)a[k]);
      v = (T)__fsub_rn(t2, t3);
    }
    out[k] = v;
    bad |= !isfinite((double)v);
  }
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}

// Factor validation on the device (validation.py:47-59 "contains non-finite
// entries"): *flag |= 1 if any element is NaN/Inf.  The caller reads the flag
// after its own result synchronisation, so the check costs no extra host pass.
template <typename T>
__global__ void check_finite_kernel(int64_t n, const T *__restrict__ x, int *flag) {
  int bad = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[k]);
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}

}  // namespace cpfit

using namespace cpfit;

extern "C" {

int cpfit_sample(cpfit_pattern *src, uint64_t key0, uint64_t key1, int64_t counter_offset,
                 double rate, void *stream, cpfit_pattern **out) {
  *out = nullptr;
  if (!src) { set_error("null pattern"); return CPFIT_EINVAL; }
  if (!(rate > 0.0 && rate <= 1.0)) {
    set_error("sample rate must be in (0, 1], got %g", rate);
    return CPFIT_EINVAL;
  }
  if (counter_offset < 0) { set_error("counter offset must be >= 0"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = src->nnz;
  // philox blocks touched: from floor(off/4) to floor((off+n-1)/4)
  const int64_t nblk = n > 0 ? ((counter_offset + n - 1) >> 2) - (counter_offset >> 2) + 1 : 0;
  const int64_t per_tile = (int64_t)SMP_THREADS * SMP_BLOCKS_PER_THREAD;
  const int64_t ntiles = (nblk + per_tile - 1) / per_tile;
  Scratch<int64_t> counts(s), offs(s);
  Scratch<uint32_t> masks(s);
  int64_t total = 0;
  int32_t *kept = nullptr;
  if (ntiles > 0) {
    CPFIT_TRY(counts.alloc(ntiles));
    CPFIT_TRY(offs.alloc(ntiles + 1));
    CPFIT_TRY(masks.alloc((size_t)ntiles * SMP_THREADS));
    unsigned grid = (unsigned)(ntiles < (int64_t)num_sms() * 16 ? ntiles : num_sms() * 16);
    sample_count_kernel<<<grid, SMP_THREADS, 0, s>>>(n, counter_offset, key0, key1,
                                                    sample_threshold(rate), ntiles, counts.ptr,
                                                    masks.ptr);
    CPFIT_LAUNCH_CHECK("sample_count");
    CPFIT_TRY(exclusive_scan<int64_t>(counts.ptr, offs.ptr, ntiles, s));
    CPFIT_CUDA(cudaMemcpyAsync(&total, offs.ptr + ntiles, sizeof(int64_t),
                               cudaMemcpyDeviceToHost, s));
    CPFIT_CUDA(cudaStreamSynchronize(s));
    CPFIT_TRY(dalloc(&kept, total > 0 ? total : 1, s));
    sample_select_kernel<<<grid, SMP_THREADS, 0, s>>>(n, counter_offset, ntiles, offs.ptr,
                                                     masks.ptr, kept);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { dfree(kept, s); return cuda_status(e, "sample_select"); }
  } else {
    CPFIT_TRY(dalloc(&kept, 1, s));
  }
  cpfit_pattern *p = new cpfit_pattern();
  p->order = src->order;
  p->nnz = total;
  // a sample's layouts are rebuilt every SGD step: long tasks (measured at
  // cfg 5: 256-entry tasks 13.2 ms per step, 1024: 11.4); an explicit source
  // task size is inherited
  p->task_size = src->task_size > 0 ? src->task_size : 1024;
  p->parent = kept;
  GatherCoords g;
  g.order = src->order;
  for (int m = 0; m < src->order; ++m) {
    p->dims[m] = src->dims[m];
    int st = dalloc(&p->coords[m], total > 0 ? total : 1, s);
    if (st) { cpfit_pattern_destroy(p); return st; }
    g.src[m] = src->coords[m];
    g.dst[m] = p->coords[m];
  }
  if (total > 0) {
    gather_coords_kernel<<<grid_for(total, 256, 4), 256, 0, s>>>(kept, total, g);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { cpfit_pattern_destroy(p); return cuda_status(e, "gather_coords"); }
  }
  *out = p;
  return CPFIT_OK;
}

int cpfit_pattern_parent_index(const cpfit_pattern *p, const int32_t **idx) {
  if (!p || !p->parent) { set_error("pattern has no parent index"); return CPFIT_EINVAL; }
  *idx = p->parent;
  return CPFIT_OK;
}

int cpfit_gather_values(int dtype, int64_t n, const int32_t *idx, const void *in, void *out,
                        void *stream) {
  if (n <= 0) return CPFIT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    gather_values_kernel<double><<<grid_for(n, 256, 4), 256, 0, s>>>(idx, n, (const double *)in,
                                                                     (double *)out);
  else if (dtype == CPFIT_F32)
    gather_values_kernel<float><<<grid_for(n, 256, 4), 256, 0, s>>>(idx, n, (const float *)in,
                                                                    (float *)out);
  else { set_error("unknown dtype %d", dtype); return CPFIT_EINVAL; }
  CPFIT_LAUNCH_CHECK("gather_values");
  return CPFIT_OK;
}

int cpfit_reduce(int op, int dtype, int64_t n, const void *x, const void *y, double *result,
                 void *stream) {
  *result = 0.0;
  if (op < 0 || op > 3) { set_error("unknown reduction %d", op); return CPFIT_EINVAL; }
  if (n <= 0) return CPFIT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    return run_reduce<double>(op, n, (const double *)x, (const double *)y, result, s);
  if (dtype == CPFIT_F32)
    return run_reduce<float>(op, n, (const float *)x, (const float *)y, result, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_check_finite(int dtype, int64_t n, const void *x, int *flag, void *stream) {
  if (n <= 0) return CPFIT_OK;
  if (!x || !flag) { set_error("null argument"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    check_finite_kernel<double><<<grid_for(n, 256, 2), 256, 0, s>>>(n, (const double *)x, flag);
  else if (dtype == CPFIT_F32)
    check_finite_kernel<float><<<grid_for(n, 256, 2), 256, 0, s>>>(n, (const float *)x, flag);
  else { set_error("unknown dtype %d", dtype); return CPFIT_EINVAL; }
  CPFIT_LAUNCH_CHECK("check_finite");
  return CPFIT_OK;
}

int cpfit_sgd_update(int dtype, int64_t n, const void *a, const void *grad, double step,
                     double shrink, void *out, int *nonfinite, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  *nonfinite = 0;
  if (n <= 0) return CPFIT_OK;
  Scratch<int> flag(s);
  CPFIT_TRY(flag.alloc(1));
  CPFIT_CUDA(cudaMemsetAsync(flag.ptr, 0, sizeof(int), s));
  if (dtype == CPFIT_F64)
    sgd_update_kernel<double><<<grid_for(n, 256, 4), 256, 0, s>>>(
        n, (const double *)a, (const double *)grad, step, shrink, (double *)out, flag.ptr);
  else if (dtype == CPFIT_F32)
    sgd_update_kernel<float><<<grid_for(n, 256, 4), 256, 0, s>>>(
        n, (const float *)a, (const float *)grad, step, shrink, (float *)out, flag.ptr);
  else { set_error("unknown dtype %d", dtype); return CPFIT_EINVAL; }
  CPFIT_LAUNCH_CHECK("sgd_update");
  CPFIT_CUDA(cudaMemcpyAsync(nonfinite, flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
  CPFIT_CUDA(cudaStreamSynchronize(s));
  return CPFIT_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// SM-driven device -> pinned-host copy: the writes cross PCIe from the SMs, so
// a small result (an MTTKRP row block) is not queued behind a large DMA that
// an earlier call left running on the copy engine (kernels.tttp's values).
namespace cpfit {
__global__ void copy_to_host_kernel(int64_t n16, const uint4 *__restrict__ src,
                                    uint4 *__restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void copy_to_host_tail(int64_t nbytes, int64_t from, const unsigned char *src,
                                  unsigned char *dst) {
  for (int64_t i = from + threadIdx.x; i < nbytes; i += blockDim.x) dst[i] = src[i];
}
}  // namespace cpfit

extern "C" int cpfit_copy_to_host(int64_t nbytes, const void *src, void *host_dst,
                                  void *stream) {
  using namespace cpfit;
  if (nbytes <= 0) return CPFIT_OK;
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, host_dst);
  if (e != cudaSuccess || at.type != cudaMemoryTypeHost || !at.devicePointer) {
    cudaGetLastError();
    set_error("host buffer is not pinned, device-mapped memory");
    return CPFIT_EINVAL;
  }
  void *dst = at.devicePointer;
  cudaStream_t s = (cudaStream_t)stream;
  const bool aligned = ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0);
  int64_t n16 = aligned ? nbytes / 16 : 0;
  if (n16) {
    copy_to_host_kernel<<<grid_for(n16, 256), 256, 0, s>>>(n16, (const uint4 *)src, (uint4 *)dst);
    CPFIT_LAUNCH_CHECK("copy_to_host");
  }
  if (n16 * 16 < nbytes) {
    copy_to_host_tail<<<1, 256, 0, s>>>(nbytes, n16 * 16, (const unsigned char *)src,
                                        (unsigned char *)dst);
    CPFIT_LAUNCH_CHECK("copy_to_host_tail");
  }
  return CPFIT_OK;
}
