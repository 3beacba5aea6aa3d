// ingest.cu -- from_coords on the device.
//
// Reference: linearize_many / from_coords / _merge_sorted (core.py:78-90,
// 208-231): key = ((i_1 I_2 + i_2) I_3 + i_3)... in uint64, a stable argsort of
// the keys, and duplicate keys merged by np.add.reduceat in that stable order.
// Here: a linearize kernel (range check per mode), the library's stable LSD
// radix sort on the significant key bits (pattern.cu), head flags + scan for
// the unique keys, and one thread per unique key summing its duplicates
// exactly as np.add.reduceat does on a contiguous slice -- the first value
// plus numpy's pairwise sum of the rest (blocks < 8 summed sequentially from
// -0.0, <= 128 with eight interleaved accumulators, larger halves split at a
// multiple of 8) -- so keys AND merged values are bit-identical.
#include "common.cuh"

namespace cpfit {

template <typename C>
__global__ void linearize_kernel(int order, CpfitDims dims, int64_t n, CpfitCoordPtrs<C> coords,
                                 uint64_t *__restrict__ keys, int *__restrict__ bad_mode) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = 0;
    for (int q = 0; q < order; ++q) {
      const int64_t c = (int64_t)coords.p[q][e];
      if (c < 0 || c >= dims.d[q]) atomicMin(bad_mode, q);
      k = k * (uint64_t)dims.d[q] + (uint64_t)c;
    }
    keys[e] = k;
  }
}

__global__ void head_flags_kernel(const uint64_t *__restrict__ k, int64_t n,
                                  int32_t *__restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

__global__ void unique_kernel(const uint64_t *__restrict__ k, const int32_t *__restrict__ flag,
                              const int64_t *__restrict__ seg, int64_t n,
                              uint64_t *__restrict__ keys_out, int64_t *__restrict__ starts) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) {
      keys_out[seg[i]] = k[i];
      starts[seg[i]] = i;
    }
}

// numpy pairwise_sum over vals[perm[a + j]], j < len (loops_utils.h):
// recursive halves for len > 128, eight accumulators for 8 <= len <= 128.
__device__ double pairwise_sum(const double *__restrict__ vals, const int32_t *__restrict__ perm,
                               int64_t a, int64_t len) {
  // explicit stack of pending (start, length) ranges; results combined as
  // left + right in the recursion's order
  struct Frame { int64_t a, len; int state; double left; };
  Frame st[48];
  int sp = 0;
  st[0] = {a, len, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame &f = st[sp];
    if (f.len <= 128) {
      double res;
      if (f.len < 8) {
        res = -0.0;
        for (int64_t j = 0; j < f.len; ++j) res += vals[perm[f.a + j]];
      } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = vals[perm[f.a + j]];
        int64_t i = 8;
        const int64_t lim = f.len - (f.len % 8);
        for (; i < lim; i += 8)
#pragma unroll
          for (int j = 0; j < 8; ++j) r[j] += vals[perm[f.a + i + j]];
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < f.len; ++i) res += vals[perm[f.a + i]];
      }
      ret = res;
      --sp;
    } else {
      int64_t n2 = f.len / 2;
      n2 -= n2 % 8;
      if (f.state == 0) {
        f.state = 1;
        st[++sp] = {f.a, n2, 0, 0.0};
        continue;
      }
      if (f.state == 1) {
        f.left = ret;
        f.state = 2;
        st[++sp] = {f.a + n2, f.len - n2, 0, 0.0};
        continue;
      }
      ret = f.left + ret;
      --sp;
    }
    // propagate: the parent resumes with `ret`
  }
  return ret;
}

// np.add.reduceat on one segment: first value + pairwise sum of the rest.
__global__ void merge_values_kernel(const double *__restrict__ vals,
                                    const int32_t *__restrict__ perm,
                                    const int64_t *__restrict__ starts, int64_t nseg, int64_t n,
                                    double *__restrict__ out) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nseg;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = starts[g];
    const int64_t b = g + 1 < nseg ? starts[g + 1] : n;
    double v = vals[perm[a]];
    if (b - a > 1) v = v + pairwise_sum(vals, perm, a + 1, b - a - 1);
    out[g] = v;
  }
}

template <typename C>
static int from_coords_impl(int order, const int64_t *dims, int64_t n, const void *const *coords,
                            const double *vals, uint64_t *keys_out, double *vals_out,
                            int64_t *nnz_out, int *bad_mode, cudaStream_t s) {
  CpfitDims D{};
  CpfitCoordPtrs<C> P{};
  long double space = 1.0L;
  for (int q = 0; q < order; ++q) {
    D.d[q] = dims[q];
    P.p[q] = (const C *)coords[q];
    space *= (long double)dims[q];
  }
  if (space > 18446744073709551615.0L) {
    set_error("shape product exceeds 2^64 - 1");
    return CPFIT_EINVAL;
  }
  uint64_t maxkey = 1;  // prod(dims) - 1 without overflow
  {
    unsigned __int128 prod = 1;
    for (int q = 0; q < order; ++q) prod *= (unsigned __int128)dims[q];
    maxkey = (uint64_t)(prod - 1);
  }
  int bits = 0;
  while (bits < 64 && (maxkey >> bits) != 0) ++bits;
  Scratch<uint64_t> keys(s), sorted(s);
  Scratch<int32_t> perm(s), flag(s);
  Scratch<int64_t> seg(s), starts(s);
  Scratch<int> bad(s);
  CPFIT_TRY(keys.alloc(n));
  CPFIT_TRY(sorted.alloc(n));
  CPFIT_TRY(perm.alloc(n));
  CPFIT_TRY(flag.alloc(n));
  CPFIT_TRY(seg.alloc(n + 1));
  CPFIT_TRY(bad.alloc(1));
  const int big = 1 << 30;
  CPFIT_CUDA(cudaMemcpyAsync(bad.ptr, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  linearize_kernel<C><<<grid_for(n, 256, 4), 256, 0, s>>>(order, D, n, P, keys.ptr, bad.ptr);
  CPFIT_LAUNCH_CHECK("linearize");
  int hbad = big;
  CPFIT_CUDA(cudaMemcpyAsync(&hbad, bad.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
  CPFIT_CUDA(cudaStreamSynchronize(s));
  if (hbad != big) {
    *bad_mode = hbad;
    set_error("coordinate out of range [0, %lld) in mode %d", (long long)dims[hbad], hbad);
    return CPFIT_EINVAL;
  }
  CPFIT_TRY(radix_sort_pairs<uint64_t>(keys.ptr, n, bits, sorted.ptr, perm.ptr, s));
  head_flags_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(sorted.ptr, n, flag.ptr);
  CPFIT_LAUNCH_CHECK("head_flags");
  CPFIT_TRY(exclusive_scan<int32_t>(flag.ptr, seg.ptr, n, s));
  int64_t nseg = 0;
  CPFIT_CUDA(cudaMemcpyAsync(&nseg, seg.ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CPFIT_CUDA(cudaStreamSynchronize(s));
  CPFIT_TRY(starts.alloc(nseg));
  unique_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(sorted.ptr, flag.ptr, seg.ptr, n, keys_out,
                                                    starts.ptr);
  CPFIT_LAUNCH_CHECK("unique");
  merge_values_kernel<<<grid_for(nseg, 256), 256, 0, s>>>(vals, perm.ptr, starts.ptr, nseg, n,
                                                          vals_out);
  CPFIT_LAUNCH_CHECK("merge_values");
  *nnz_out = nseg;
  return CPFIT_OK;
}

}  // namespace cpfit

using namespace cpfit;

extern "C" {

int cpfit_from_coords(int order, const int64_t *dims, int64_t n, int coord_bytes,
                      const void *const *coords, const double *vals, uint64_t *keys_out,
                      double *vals_out, int64_t *nnz_out, int *bad_mode, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (bad_mode) *bad_mode = -1;
  if (order < 1 || order > CPFIT_MAXN) {
    set_error("order %d unsupported (1..%d)", order, CPFIT_MAXN);
    return CPFIT_EINVAL;
  }
  for (int q = 0; q < order; ++q)
    if (dims[q] < 1) {
      set_error("dimension %d of mode %d must be >= 1", (int)dims[q], q);
      return CPFIT_EINVAL;
    }
  if (n < 0 || n > (int64_t)INT32_MAX) {
    set_error("entry count %lld out of range", (long long)n);
    return CPFIT_EINVAL;
  }
  *nnz_out = 0;
  if (n == 0) return CPFIT_OK;
  int dummy = -1;
  int *bm = bad_mode ? bad_mode : &dummy;
  if (coord_bytes == 8)
    return from_coords_impl<int64_t>(order, dims, n, coords, vals, keys_out, vals_out, nnz_out,
                                     bm, s);
  if (coord_bytes == 4)
    return from_coords_impl<int32_t>(order, dims, n, coords, vals, keys_out, vals_out, nnz_out,
                                     bm, s);
  set_error("coordinate width %d unsupported (4 or 8 bytes)", coord_bytes);
  return CPFIT_EINVAL;
}

}  // extern "C"
