// pattern.cu -- device-resident sparsity pattern: delinearize, stable mode
// grouping (LSD radix sort), segment offsets and the work-task tables used by
// the segmented kernels.
//
// Reference: SparseTensor caches (core.py:141-167), delinearize_many
// (core.py:93-102), counting_sort_by_mode (core.py:234-249).
#include <cstdarg>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include <type_traits>

#include "common.cuh"

namespace cpfit {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// ---------------------------------------------------------------------------
// scratch cache (see common.cuh)

namespace {
struct CachedBlock {
  void *p;
  size_t cap;
  cudaStream_t s;
};
std::mutex g_scratch_mu;
std::vector<CachedBlock> g_scratch;
size_t g_scratch_bytes = 0;
constexpr size_t kScratchKeep = 2ull << 30;  // bytes kept cached at most
}  // namespace

void *scratch_get(size_t bytes, cudaStream_t s, size_t *cap) {
  size_t c = 256;
  while (c < bytes) c <<= 1;
  {
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    for (size_t i = 0; i < g_scratch.size(); ++i) {
      if (g_scratch[i].cap == c && g_scratch[i].s == s) {
        void *p = g_scratch[i].p;
        g_scratch_bytes -= c;
        g_scratch[i] = g_scratch.back();
        g_scratch.pop_back();
        *cap = c;
        return p;
      }
    }
  }
  void *p = nullptr;
  if (cudaMallocAsync(&p, c, s) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  *cap = c;
  return p;
}

void scratch_put(void *p, size_t cap, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  if (g_scratch_bytes + cap > kScratchKeep) {
    cudaFreeAsync(p, s);
    return;
  }
  g_scratch.push_back({p, cap, s});
  g_scratch_bytes += cap;
}

int cuda_status(cudaError_t e, const char *what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? CPFIT_ENOMEM : CPFIT_ECUDA;
}

// ---------------------------------------------------------------------------
// exclusive scan (3-phase: tile sums, recursive scan of sums, apply)

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v) {
  int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns exclusive prefix
// and writes the block total to *total.
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t *total) {
  __shared__ int64_t warp_sums[SCAN_THREADS / 32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t incl = warp_incl_scan(v);
  if (lane == 31) warp_sums[w] = incl;
  __syncthreads();
  if (w == 0) {
    int64_t x = lane < SCAN_THREADS / 32 ? warp_sums[lane] : 0;
    int64_t xi = warp_incl_scan(x);
    if (lane < SCAN_THREADS / 32) warp_sums[lane] = xi - x;
    if (lane == 31) *total = xi;  // lanes >= nwarps add zeros: lane 31 holds the total
  }
  __syncthreads();
  int64_t r = incl - v + warp_sums[w];
  __syncthreads();
  return r;
}

template <typename Tin>
__global__ void __launch_bounds__(SCAN_THREADS) scan_tile_sums(const Tin *in, int64_t n,
                                                               int64_t *sums) {
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int64_t acc = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i)
    if (base + i < n) acc += (int64_t)in[base + i];
  __shared__ int64_t tot;
  block_excl_scan(acc, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <typename Tin>
__global__ void __launch_bounds__(SCAN_THREADS) scan_tile_apply(const Tin *in, int64_t n,
                                                                const int64_t *tile_off,
                                                                int64_t *out) {
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS];
  int64_t acc = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    v[i] = (base + i < n) ? (int64_t)in[base + i] : 0;
    acc += v[i];
  }
  __shared__ int64_t tot;
  int64_t pre = block_excl_scan(acc, &tot) + (tile_off ? tile_off[blockIdx.x] : 0);
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    if (base + i < n) out[base + i] = pre;
    pre += v[i];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == SCAN_THREADS - 1) out[n] = pre;
}

template <typename Tin>
int exclusive_scan(const Tin *in, int64_t *out, int64_t n, cudaStream_t s) {
  if (n <= 0) {
    CPFIT_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
    return CPFIT_OK;
  }
  int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles == 1) {
    scan_tile_apply<Tin><<<1, SCAN_THREADS, 0, s>>>(in, n, nullptr, out);
    CPFIT_LAUNCH_CHECK("scan_tile_apply");
    return CPFIT_OK;
  }
  Scratch<int64_t> sums(s), offs(s);
  CPFIT_TRY(sums.alloc(tiles));
  CPFIT_TRY(offs.alloc(tiles + 1));
  scan_tile_sums<Tin><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, n, sums.ptr);
  CPFIT_LAUNCH_CHECK("scan_tile_sums");
  CPFIT_TRY(exclusive_scan<int64_t>(sums.ptr, offs.ptr, tiles, s));
  scan_tile_apply<Tin><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, n, offs.ptr, out);
  CPFIT_LAUNCH_CHECK("scan_tile_apply");
  return CPFIT_OK;
}

template int exclusive_scan<int32_t>(const int32_t *, int64_t *, int64_t, cudaStream_t);
template int exclusive_scan<int64_t>(const int64_t *, int64_t *, int64_t, cudaStream_t);
template int exclusive_scan<uint32_t>(const uint32_t *, int64_t *, int64_t, cudaStream_t);

// ---------------------------------------------------------------------------
// simple element kernels

__global__ void gather_i32_kernel(const int32_t *__restrict__ in,
                                  const int32_t *__restrict__ idx,
                                  int32_t *__restrict__ out, int64_t n) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = __ldg(in + __ldg(idx + k));
}

int gather_i32(const int32_t *in, const int32_t *idx, int32_t *out, int64_t n,
               cudaStream_t s) {
  if (n <= 0) return CPFIT_OK;
  gather_i32_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(in, idx, out, n);
  CPFIT_LAUNCH_CHECK("gather_i32");
  return CPFIT_OK;
}

template <typename T>
__global__ void gather_vals_kernel(const T *__restrict__ in, const int32_t *__restrict__ idx,
                                   T *__restrict__ out, int64_t n) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = __ldg(in + __ldg(idx + k));
}

__global__ void iota_kernel(int32_t *out, int64_t n) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = (int32_t)k;
}

struct DelinParams {
  int order;
  uint64_t dims[CPFIT_MAXN];
  int32_t *coords[CPFIT_MAXN];
};

// key -> coordinates, last mode fastest (core.py:93-102)
__global__ void delinearize_kernel(const uint64_t *__restrict__ keys, int64_t n,
                                   DelinParams p) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t rem = keys[e];
#pragma unroll 1
    for (int m = p.order - 1; m >= 0; --m) {
      uint64_t d = p.dims[m];
      uint64_t q = rem / d;
      p.coords[m][e] = (int32_t)(rem - q * d);
      rem = q;
    }
  }
}

// offsets[i] = first position whose (sorted) key >= i, for i in [0, dim]
__global__ void offsets_from_sorted(const int32_t *__restrict__ sorted, int64_t n,
                                    int64_t dim, int64_t *__restrict__ offsets) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t prev = e > 0 ? (int64_t)sorted[e - 1] : -1;
    int64_t cur = e < n ? (int64_t)sorted[e] : dim;
    for (int64_t i = prev + 1; i <= cur; ++i) offsets[i] = e;
  }
}

// ---------------------------------------------------------------------------
// stable LSD radix sort of (key, position) pairs.  The digit width is chosen
// per sort: the fewest passes with digits of at most RS_MAX_DIGIT bits, split
// evenly (17 key bits -> 2 x 9 instead of 3 x 8; 10 -> 1 x 10; 40 -> 4 x 10).

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
#ifndef CPFIT_RS_MAX_DIGIT
#define CPFIT_RS_MAX_DIGIT 10
#endif
constexpr int RS_MAX_DIGIT = CPFIT_RS_MAX_DIGIT;

template <typename K>
__device__ __forceinline__ int radix_digit(K key, int shift, unsigned mask) {
  return (int)((((typename std::make_unsigned<K>::type)key) >> shift) & mask);
}

// per-tile digit histogram -> counts[digit * nblocks + tile]
template <typename K>
__global__ void __launch_bounds__(RS_THREADS)
radix_upsweep(const K *__restrict__ keys, int64_t n, int shift, int nbins, int64_t nblocks,
              int32_t *__restrict__ counts) {
  extern __shared__ int hist[];
  const unsigned mask = (unsigned)nbins - 1u;
  for (int i = threadIdx.x; i < nbins; i += RS_THREADS) hist[i] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * RS_TILE;
  for (int i = threadIdx.x; i < RS_TILE; i += RS_THREADS) {
    int64_t k = base + i;
    if (k < n) atomicAdd(&hist[radix_digit(keys[k], shift, mask)], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < nbins; d += RS_THREADS)
    counts[(int64_t)d * nblocks + blockIdx.x] = hist[d];
}

// vals_in == nullptr means the identity (first pass).  Ranks inside a tile
// follow entry order (warp w's items before warp w+1's, item j before j+1,
// lane order inside an item), so the sort is stable.  The tile is first
// reordered by digit in shared memory, then written out position by position:
// consecutive threads store consecutive addresses inside each digit's run
// (whole 32-byte sectors instead of one 4-byte store per sector).
template <typename K>
__global__ void __launch_bounds__(RS_THREADS)
radix_downsweep(const K *__restrict__ keys_in, const int32_t *__restrict__ vals_in,
                int64_t n, int shift, int nbins, int64_t nblocks,
                const int64_t *__restrict__ offs, K *__restrict__ keys_out,
                int32_t *__restrict__ vals_out) {
  extern __shared__ __align__(16) unsigned char rs_smem[];
  // layout: staged keys [RS_TILE] | staged vals [RS_TILE] | digit starts [nbins + 1]
  //         | per-warp histograms RS_WARPS x (nbins + 1)
  K *skey = reinterpret_cast<K *>(rs_smem);
  int32_t *sval = reinterpret_cast<int32_t *>(skey + RS_TILE);
  int *dstart = reinterpret_cast<int *>(sval + RS_TILE);
  int *whist_all = dstart + (nbins + 1);
  __shared__ int wsum[RS_WARPS];
  const int pitch = nbins + 1;
  const unsigned mask = (unsigned)nbins - 1u;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int *whist = whist_all + w * pitch;
  for (int i = lane; i < pitch; i += 32) whist[i] = 0;
  __syncwarp();
  const int64_t tbase = (int64_t)blockIdx.x * RS_TILE;
  const int64_t wbase = tbase + (int64_t)w * 32 * RS_ITEMS;
  K key[RS_ITEMS];
  int32_t val[RS_ITEMS];
  int32_t rank[RS_ITEMS];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    int64_t k = wbase + j * 32 + lane;
    bool valid = k < n;
    key[j] = valid ? keys_in[k] : 0;
    val[j] = valid ? (vals_in ? vals_in[k] : (int32_t)k) : 0;
  }
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    int64_t k = wbase + j * 32 + lane;
    int d = k < n ? radix_digit(key[j], shift, mask) : nbins;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int pre = whist[d];
    __syncwarp();
    int leader = __ffs(peers) - 1;
    if (lane == leader) whist[d] = pre + __popc(peers);
    __syncwarp();
    rank[j] = pre + __popc(peers & lt);
  }
  __syncthreads();
  // per digit: exclusive scan over warps; the digit's tile total goes to dstart
  for (int d = threadIdx.x; d < nbins; d += RS_THREADS) {
    int run = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww) {
      int c = whist_all[ww * pitch + d];
      whist_all[ww * pitch + d] = run;
      run += c;
    }
    dstart[d] = run;
  }
  __syncthreads();
  // exclusive scan of the digit totals over the block (thread t owns a
  // contiguous group of nbins / RS_THREADS digits, at least one)
  {
    const int per = nbins >= RS_THREADS ? nbins / RS_THREADS : 1;
    const int d0 = threadIdx.x * per;
    int local = 0;
    if (d0 < nbins)
      for (int i = 0; i < per; ++i) local += dstart[d0 + i];
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int up = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += up;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    int wbefore = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww)
      if (ww < w) wbefore += wsum[ww];
    int run = wbefore + incl - local;
    if (d0 < nbins)
      for (int i = 0; i < per; ++i) {
        int c = dstart[d0 + i];
        dstart[d0 + i] = run;
        run += c;
      }
  }
  __syncthreads();
  // stage the tile in digit order
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    int64_t k = wbase + j * 32 + lane;
    if (k < n) {
      int d = radix_digit(key[j], shift, mask);
      int lp = dstart[d] + whist[d] + rank[j];
      skey[lp] = key[j];
      sval[lp] = val[j];
    }
  }
  __syncthreads();
  const int cnt = (int)(n - tbase < RS_TILE ? n - tbase : RS_TILE);
  for (int i = threadIdx.x; i < cnt; i += RS_THREADS) {
    K kk = skey[i];
    int d = radix_digit(kk, shift, mask);
    int64_t pos = offs[(int64_t)d * nblocks + blockIdx.x] + (i - dstart[d]);
    keys_out[pos] = kk;
    vals_out[pos] = sval[i];
  }
}

// Stable LSD sort of positions 0..n-1 by the low `bits` bits of keys
// (int32 mode coordinates or uint64 linearized keys).  Writes the sorted keys
// and the permutation.
template <typename K>
int radix_sort_pairs(const K *keys, int64_t n, int bits, K *sorted_keys, int32_t *perm,
                     cudaStream_t s) {
  const int passes = (bits + RS_MAX_DIGIT - 1) / RS_MAX_DIGIT;
  if (passes == 0 || n <= 1) {
    iota_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(perm, n);
    CPFIT_LAUNCH_CHECK("iota");
    if (n) CPFIT_CUDA(cudaMemcpyAsync(sorted_keys, keys, n * sizeof(K),
                                      cudaMemcpyDeviceToDevice, s));
    return CPFIT_OK;
  }
  const int dbits = (bits + passes - 1) / passes;  // even split, <= RS_MAX_DIGIT
  const int nbins = 1 << dbits;
  const size_t up_smem = (size_t)nbins * sizeof(int);
  const size_t down_smem = (size_t)RS_TILE * (sizeof(K) + sizeof(int32_t)) +
                           (size_t)(RS_WARPS + 1) * (nbins + 1) * sizeof(int);
  static bool attr_set = false;  // > 48 KB of dynamic shared memory needs the opt-in
  if (!attr_set) {
    constexpr size_t worst = (size_t)RS_TILE * (sizeof(K) + sizeof(int32_t)) +
                             (size_t)(RS_WARPS + 1) * ((1 << RS_MAX_DIGIT) + 1) * sizeof(int);
    static_assert(worst <= 200 * 1024, "radix tile does not fit shared memory");
    CPFIT_CUDA(cudaFuncSetAttribute(radix_downsweep<K>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)worst));
    attr_set = true;
  }
  int64_t nblocks = (n + RS_TILE - 1) / RS_TILE;
  Scratch<int32_t> counts(s), v_tmp(s);
  Scratch<K> k_tmp(s);
  Scratch<int64_t> offs(s);
  CPFIT_TRY(counts.alloc((int64_t)nbins * nblocks));
  CPFIT_TRY(offs.alloc((int64_t)nbins * nblocks + 1));
  CPFIT_TRY(k_tmp.alloc(n));
  CPFIT_TRY(v_tmp.alloc(n));
  // ping-pong so that the last pass lands in (sorted_keys, perm)
  K *kb[2];
  int32_t *vb[2];
  if (passes % 2 == 1) {
    kb[0] = sorted_keys; vb[0] = perm; kb[1] = k_tmp.ptr; vb[1] = v_tmp.ptr;
  } else {
    kb[0] = k_tmp.ptr; vb[0] = v_tmp.ptr; kb[1] = sorted_keys; vb[1] = perm;
  }
  const K *kin = keys;
  const int32_t *vin = nullptr;
  for (int p = 0; p < passes; ++p) {
    int shift = dbits * p;
    radix_upsweep<K><<<(unsigned)nblocks, RS_THREADS, up_smem, s>>>(kin, n, shift, nbins,
                                                                     nblocks, counts.ptr);
    CPFIT_LAUNCH_CHECK("radix_upsweep");
    CPFIT_TRY(exclusive_scan<int32_t>(counts.ptr, offs.ptr, (int64_t)nbins * nblocks, s));
    K *ko = kb[p % 2];
    int32_t *vo = vb[p % 2];
    radix_downsweep<K><<<(unsigned)nblocks, RS_THREADS, down_smem, s>>>(
        kin, vin, n, shift, nbins, nblocks, offs.ptr, ko, vo);
    CPFIT_LAUNCH_CHECK("radix_downsweep");
    kin = ko;
    vin = vo;
  }
  return CPFIT_OK;
}
template int radix_sort_pairs<uint64_t>(const uint64_t *, int64_t, int, uint64_t *, int32_t *,
                                        cudaStream_t);
template int radix_sort_pairs<int32_t>(const int32_t *, int64_t, int, int32_t *, int32_t *,
                                       cudaStream_t);

// Stable sort of positions 0..n-1 by keys (non-negative, < dim).
static int radix_sort_positions(const int32_t *keys, int64_t n, int64_t dim,
                                int32_t *sorted_keys, int32_t *perm, cudaStream_t s) {
  int bits = 0;
  while (bits < 31 && ((int64_t)1 << bits) < dim) ++bits;
  return radix_sort_pairs<int32_t>(keys, n, bits, sorted_keys, perm, s);
}

// ---------------------------------------------------------------------------
// task tables: every non-empty slice is cut into ceil(len / L) contiguous
// tasks of near-equal length; slices with more than one task get partial
// slots, combined in task order afterwards (deterministic, no atomics).

__global__ void task_count_kernel(const int64_t *__restrict__ offsets, int64_t dim, int64_t L,
                                  int32_t *__restrict__ nt, int32_t *__restrict__ nslot,
                                  int32_t *__restrict__ split, int *__restrict__ max_t) {
  int mt = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t len = offsets[i + 1] - offsets[i];
    int64_t t = (len + L - 1) / L;
    nt[i] = (int32_t)t;
    nslot[i] = t > 1 ? (int32_t)t : 0;
    split[i] = t > 1 ? 1 : 0;
    mt = t > mt ? (int)t : mt;
  }
  if (mt) atomicMax(max_t, mt);
}

__global__ void task_fill_kernel(const int64_t *__restrict__ offsets, int64_t dim,
                                 const int32_t *__restrict__ nt,
                                 const int64_t *__restrict__ tstart,
                                 const int64_t *__restrict__ sstart,
                                 const int64_t *__restrict__ xstart, int64_t nnz,
                                 int64_t *__restrict__ task_begin, int32_t *__restrict__ task_row,
                                 int32_t *__restrict__ task_slot, int32_t *__restrict__ split_row,
                                 int32_t *__restrict__ split_slot) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = nt[i];
    if (t == 0) continue;
    int64_t len = offsets[i + 1] - offsets[i];
    int64_t t0 = tstart[i];
    for (int64_t j = 0; j < t; ++j) {
      task_begin[t0 + j] = offsets[i] + (j * len) / t;
      task_row[t0 + j] = (int32_t)i;
      task_slot[t0 + j] = t > 1 ? (int32_t)(sstart[i] + j) : -1;
    }
    if (t > 1) {
      int64_t x = xstart[i];
      split_row[x] = (int32_t)i;
      split_slot[x] = (int32_t)sstart[i];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    task_begin[tstart[dim]] = nnz;
    split_slot[xstart[dim]] = (int32_t)sstart[dim];
  }
}

static int build_tasks(CpfitModeLayout &L, int64_t dim, int64_t nnz, int64_t task_size,
                       cudaStream_t s) {
  Scratch<int32_t> nt(s), nslot(s), split(s);
  Scratch<int64_t> tstart(s), sstart(s), xstart(s);
  Scratch<int> maxt(s);
  CPFIT_TRY(maxt.alloc(1));
  CPFIT_CUDA(cudaMemsetAsync(maxt.ptr, 0, sizeof(int), s));
  CPFIT_TRY(nt.alloc(dim));
  CPFIT_TRY(nslot.alloc(dim));
  CPFIT_TRY(split.alloc(dim));
  CPFIT_TRY(tstart.alloc(dim + 1));
  CPFIT_TRY(sstart.alloc(dim + 1));
  CPFIT_TRY(xstart.alloc(dim + 1));
  task_count_kernel<<<grid_for(dim, 256), 256, 0, s>>>(L.offsets, dim, task_size, nt.ptr,
                                                       nslot.ptr, split.ptr, maxt.ptr);
  CPFIT_LAUNCH_CHECK("task_count");
  CPFIT_TRY(exclusive_scan<int32_t>(nt.ptr, tstart.ptr, dim, s));
  CPFIT_TRY(exclusive_scan<int32_t>(nslot.ptr, sstart.ptr, dim, s));
  CPFIT_TRY(exclusive_scan<int32_t>(split.ptr, xstart.ptr, dim, s));
  int64_t tot[3];
  CPFIT_CUDA(cudaMemcpyAsync(&tot[0], tstart.ptr + dim, 8, cudaMemcpyDeviceToHost, s));
  CPFIT_CUDA(cudaMemcpyAsync(&tot[1], sstart.ptr + dim, 8, cudaMemcpyDeviceToHost, s));
  CPFIT_CUDA(cudaMemcpyAsync(&tot[2], xstart.ptr + dim, 8, cudaMemcpyDeviceToHost, s));
  int hmax = 0;
  CPFIT_CUDA(cudaMemcpyAsync(&hmax, maxt.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
  CPFIT_CUDA(cudaStreamSynchronize(s));
  L.max_slots = hmax;
  L.ntasks = tot[0];
  L.nslots = tot[1];
  L.nsplit = tot[2];
  L.task_size = task_size;
  CPFIT_TRY(dalloc(&L.task_begin, L.ntasks + 1, s));
  CPFIT_TRY(dalloc(&L.task_row, L.ntasks > 0 ? L.ntasks : 1, s));
  CPFIT_TRY(dalloc(&L.task_slot, L.ntasks > 0 ? L.ntasks : 1, s));
  CPFIT_TRY(dalloc(&L.split_row, L.nsplit > 0 ? L.nsplit : 1, s));
  CPFIT_TRY(dalloc(&L.split_slot, L.nsplit + 1, s));
  task_fill_kernel<<<grid_for(dim, 256), 256, 0, s>>>(
      L.offsets, dim, nt.ptr, tstart.ptr, sstart.ptr, xstart.ptr, nnz, L.task_begin,
      L.task_row, L.task_slot, L.split_row, L.split_slot);
  CPFIT_LAUNCH_CHECK("task_fill");
  return CPFIT_OK;
}

int ensure_layout(cpfit_pattern *p, int mode, cudaStream_t s) {
  CpfitModeLayout &L = p->modes[mode];
  if (L.built) return CPFIT_OK;
  const int64_t n = p->nnz, dim = p->dims[mode];
  CPFIT_TRY(dalloc(&L.offsets, dim + 1, s));
  if (mode == 0) {
    // keys are sorted, so mode 0 groups are already contiguous: perm = identity
    L.perm = nullptr;
    for (int k = 0; k < p->order; ++k) {
      L.sorted_idx[k] = p->coords[k];
      L.owns_sorted[k] = false;
    }
    if (n > 0) {
      offsets_from_sorted<<<grid_for(n + 1, 256, 4), 256, 0, s>>>(p->coords[0], n, dim,
                                                                  L.offsets);
      CPFIT_LAUNCH_CHECK("offsets_from_sorted");
    } else {
      CPFIT_CUDA(cudaMemsetAsync(L.offsets, 0, (dim + 1) * sizeof(int64_t), s));
    }
  } else {
    int32_t *sorted_keys = nullptr;
    CPFIT_TRY(dalloc(&L.perm, n > 0 ? n : 1, s));
    CPFIT_TRY(dalloc(&sorted_keys, n > 0 ? n : 1, s));
    if (n > 0) {
      CPFIT_TRY(radix_sort_positions(p->coords[mode], n, dim, sorted_keys, L.perm, s));
      offsets_from_sorted<<<grid_for(n + 1, 256, 4), 256, 0, s>>>(sorted_keys, n, dim,
                                                                  L.offsets);
      CPFIT_LAUNCH_CHECK("offsets_from_sorted");
    } else {
      CPFIT_CUDA(cudaMemsetAsync(L.offsets, 0, (dim + 1) * sizeof(int64_t), s));
    }
    L.sorted_idx[mode] = sorted_keys;
    L.owns_sorted[mode] = true;
    for (int k = 0; k < p->order; ++k) {
      if (k == mode) continue;
      CPFIT_TRY(dalloc(&L.sorted_idx[k], n > 0 ? n : 1, s));
      L.owns_sorted[k] = true;
      CPFIT_TRY(gather_i32(p->coords[k], L.perm, L.sorted_idx[k], n, s));
    }
  }
  CPFIT_TRY(build_tasks(L, dim, n, task_size_for(p), s));
  L.built = true;
  return CPFIT_OK;
}

int ensure_coarse_layout(cpfit_pattern *p, int mode, cudaStream_t s) {
  CPFIT_TRY(ensure_layout(p, mode, s));
  CpfitModeLayout &C = p->coarse[mode];
  if (C.built) return CPFIT_OK;
  const CpfitModeLayout &L = p->modes[mode];
  C.perm = L.perm;
  C.offsets = L.offsets;
  for (int k = 0; k < p->order; ++k) {
    C.sorted_idx[k] = L.sorted_idx[k];
    C.owns_sorted[k] = false;
  }
  C.borrowed = true;
  CPFIT_TRY(build_tasks(C, p->dims[mode], p->nnz, coarse_task_size_for(p), s));
  C.built = true;
  return CPFIT_OK;
}

template <typename T>
static int permute_vals(const T *in, const int32_t *perm, T *out, int64_t n, cudaStream_t s) {
  if (n <= 0) return CPFIT_OK;
  gather_vals_kernel<T><<<grid_for(n, 256, 4), 256, 0, s>>>(in, perm, out, n);
  CPFIT_LAUNCH_CHECK("permute_values");
  return CPFIT_OK;
}

}  // namespace cpfit

using namespace cpfit;

extern "C" {

const char *cpfit_version(void) { return "cpfit-b200 0.1.0 (sm_100a)"; }

const char *cpfit_last_error(void) { return g_err; }

static int validate_dims(int order, const int64_t *dims) {
  if (order < 1 || order > CPFIT_MAXN) {
    set_error("order %d outside the supported range [1, %d]", order, CPFIT_MAXN);
    return CPFIT_EINVAL;
  }
  for (int n = 0; n < order; ++n) {
    if (dims[n] < 1 || dims[n] > INT32_MAX) {
      set_error("dimension of mode %d (%lld) outside [1, 2^31-1]", n, (long long)dims[n]);
      return CPFIT_EINVAL;
    }
  }
  return CPFIT_OK;
}

int cpfit_pattern_create(int order, const int64_t *dims, int64_t nnz, const uint64_t *keys,
                         void *stream, cpfit_pattern **out) {
  *out = nullptr;
  CPFIT_TRY(validate_dims(order, dims));
  if (nnz < 0 || nnz > INT32_MAX) {
    set_error("nnz %lld outside [0, 2^31-1]", (long long)nnz);
    return CPFIT_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cpfit_pattern *p = new (std::nothrow) cpfit_pattern();
  if (!p) return CPFIT_ENOMEM;
  p->order = order;
  p->nnz = nnz;
  DelinParams dp;
  dp.order = order;
  for (int n = 0; n < order; ++n) {
    p->dims[n] = dims[n];
    dp.dims[n] = (uint64_t)dims[n];
    int st = dalloc(&p->coords[n], nnz > 0 ? nnz : 1, s);
    if (st) { cpfit_pattern_destroy(p); return st; }
    dp.coords[n] = p->coords[n];
  }
  if (nnz > 0) {
    delinearize_kernel<<<grid_for(nnz, 256, 4), 256, 0, s>>>(keys, nnz, dp);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { cpfit_pattern_destroy(p); return cuda_status(e, "delinearize"); }
  }
  *out = p;
  return CPFIT_OK;
}

int cpfit_pattern_create_coords(int order, const int64_t *dims, int64_t nnz,
                                const int32_t *const *coords, void *stream,
                                cpfit_pattern **out) {
  *out = nullptr;
  CPFIT_TRY(validate_dims(order, dims));
  if (nnz < 0 || nnz > INT32_MAX) {
    set_error("nnz %lld outside [0, 2^31-1]", (long long)nnz);
    return CPFIT_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cpfit_pattern *p = new (std::nothrow) cpfit_pattern();
  if (!p) return CPFIT_ENOMEM;
  p->order = order;
  p->nnz = nnz;
  for (int n = 0; n < order; ++n) {
    p->dims[n] = dims[n];
    int st = dalloc(&p->coords[n], nnz > 0 ? nnz : 1, s);
    if (st) { cpfit_pattern_destroy(p); return st; }
    if (nnz > 0) {
      cudaError_t e = cudaMemcpyAsync(p->coords[n], coords[n], nnz * sizeof(int32_t),
                                      cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) { cpfit_pattern_destroy(p); return cuda_status(e, "copy coords"); }
    }
  }
  *out = p;
  return CPFIT_OK;
}

// Release every device buffer of a pattern.  stream_ordered: cudaFreeAsync on
// `s` (no host or device-wide synchronisation); otherwise a device sync and
// synchronous frees, safe whatever streams used the buffers.
static void pattern_release(cpfit_pattern *p, bool stream_ordered, cudaStream_t s) {
  auto rel = [&](void *q) {
    if (!q) return;
    if (stream_ordered) cudaFreeAsync(q, s);
    else cudaFree(q);
  };
  if (!stream_ordered) cudaDeviceSynchronize();
  for (int m = 0; m < p->order; ++m) {
    CpfitModeLayout &L = p->modes[m];
    rel(L.perm);
    rel(L.offsets);
    for (int k = 0; k < p->order; ++k)
      if (L.owns_sorted[k]) rel(L.sorted_idx[k]);
    rel(L.task_begin);
    rel(L.task_row);
    rel(L.task_slot);
    rel(L.split_row);
    rel(L.split_slot);
    rel(L.identity_perm);
    CpfitModeLayout &C = p->coarse[m];
    rel(C.task_begin);
    rel(C.task_row);
    rel(C.task_slot);
    rel(C.split_row);
    rel(C.split_slot);
  }
  for (int n = 0; n < p->order; ++n) rel(p->coords[n]);
  rel(p->parent);
  delete p;
}

int cpfit_pattern_destroy(cpfit_pattern *p) {
  if (!p) return CPFIT_OK;
  pattern_release(p, false, nullptr);
  return CPFIT_OK;
}

int cpfit_pattern_destroy_async(cpfit_pattern *p, void *stream) {
  if (!p) return CPFIT_OK;
  pattern_release(p, true, (cudaStream_t)stream);
  return CPFIT_OK;
}

int cpfit_pattern_info(const cpfit_pattern *p, int *order, int64_t *nnz) {
  if (!p) { set_error("null pattern"); return CPFIT_EINVAL; }
  if (order) *order = p->order;
  if (nnz) *nnz = p->nnz;
  return CPFIT_OK;
}

int cpfit_pattern_coords(const cpfit_pattern *p, int mode, const int32_t **coords) {
  if (!p || mode < 0 || mode >= p->order) {
    set_error("mode %d out of range", mode);
    return CPFIT_EINVAL;
  }
  *coords = p->coords[mode];
  return CPFIT_OK;
}

int cpfit_pattern_set_task_size(cpfit_pattern *p, int64_t entries) {
  if (!p || entries < 1) { set_error("task size must be >= 1"); return CPFIT_EINVAL; }
  p->task_size = entries;
  return CPFIT_OK;
}

int cpfit_pattern_mode_group(cpfit_pattern *p, int mode, void *stream, const int32_t **perm,
                             const int64_t **offsets) {
  if (!p || mode < 0 || mode >= p->order) {
    set_error("mode %d out of range for order-%d tensor", mode, p ? p->order : 0);
    return CPFIT_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  CPFIT_TRY(ensure_layout(p, mode, s));
  CpfitModeLayout &L = p->modes[mode];
  if (perm) {
    if (L.perm) {
      *perm = L.perm;
    } else {
      if (!L.identity_perm) {
        CPFIT_TRY(dalloc(&L.identity_perm, p->nnz > 0 ? p->nnz : 1, s));
        iota_kernel<<<grid_for(p->nnz, 256, 4), 256, 0, s>>>(L.identity_perm, p->nnz);
        CPFIT_LAUNCH_CHECK("iota");
      }
      *perm = L.identity_perm;
    }
  }
  if (offsets) *offsets = L.offsets;
  return CPFIT_OK;
}

int cpfit_pattern_mode_stats(cpfit_pattern *p, int mode, void *stream, int64_t *ntasks,
                             int64_t *nsplit, int64_t *nslots) {
  if (!p || mode < 0 || mode >= p->order) { set_error("bad mode"); return CPFIT_EINVAL; }
  CPFIT_TRY(ensure_layout(p, mode, (cudaStream_t)stream));
  const CpfitModeLayout &L = p->modes[mode];
  if (ntasks) *ntasks = L.ntasks;
  if (nsplit) *nsplit = L.nsplit;
  if (nslots) *nslots = L.nslots;
  return CPFIT_OK;
}

int cpfit_permute_values(cpfit_pattern *p, int mode, int dtype, const void *vals, void *out,
                         void *stream) {
  if (!p || mode < 0 || mode >= p->order) { set_error("bad mode"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  CPFIT_TRY(ensure_layout(p, mode, s));
  CpfitModeLayout &L = p->modes[mode];
  size_t es = dtype == CPFIT_F64 ? 8 : 4;
  if (!L.perm) {
    if (p->nnz) CPFIT_CUDA(cudaMemcpyAsync(out, vals, p->nnz * es, cudaMemcpyDeviceToDevice, s));
    return CPFIT_OK;
  }
  if (dtype == CPFIT_F64)
    return permute_vals((const double *)vals, L.perm, (double *)out, p->nnz, s);
  if (dtype == CPFIT_F32)
    return permute_vals((const float *)vals, L.perm, (float *)out, p->nnz, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

}  // extern "C"
