// common.cuh -- shared helpers for the sm_100a kernels of cpfit-b200.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/cpfit_b200.h"

#define CPFIT_MAXN 8  // maximum tensor order handled on the device

namespace cpfit {

void set_error(const char *fmt, ...);
int cuda_status(cudaError_t e, const char *what);

#define CPFIT_CUDA(call)                                       \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return ::cpfit::cuda_status(_e, #call); \
  } while (0)

#define CPFIT_LAUNCH_CHECK(what)                               \
  do {                                                         \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return ::cpfit::cuda_status(_e, what); \
  } while (0)

#define CPFIT_TRY(call)          \
  do {                           \
    int _s = (call);             \
    if (_s != CPFIT_OK) return _s; \
  } while (0)

inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    // keep up to CPFIT_POOL_KEEP_GB (default 16) of freed memory mapped in the
    // stream-ordered pool: per-step patterns (SGD samples, their layouts) are
    // then re-used instead of being unmapped at every synchronisation and
    // mapped again (measured: SGD step at cfg 5 16.5 -> 12.3 ms)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      const char *env = getenv("CPFIT_POOL_KEEP_GB");
      uint64_t keep = (uint64_t)(env ? atoi(env) : 16) << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  return sms;
}

// Stream-ordered scratch allocation (the device's default memory pool).
template <typename T>
inline int dalloc(T **p, size_t count, cudaStream_t s) {
  *p = nullptr;
  if (count == 0) return CPFIT_OK;
  cudaError_t e = cudaMallocAsync((void **)p, count * sizeof(T), s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("device allocation of %zu bytes failed: %s", count * sizeof(T),
              cudaGetErrorString(e));
    return CPFIT_ENOMEM;
  }
  return CPFIT_OK;
}

template <typename T>
inline void dfree(T *p, cudaStream_t s) {
  if (p) cudaFreeAsync((void *)p, s);
}

// Per-call scratch comes from a small stream-keyed cache of power-of-two
// blocks (pattern.cu): blocks released on stream s are only handed out again
// on stream s, so reuse is stream-ordered and needs no synchronisation.
// Keeps the per-sweep kernels off the driver's allocate / map / unmap path.
void *scratch_get(size_t bytes, cudaStream_t s, size_t *cap);
void scratch_put(void *p, size_t cap, cudaStream_t s);

// RAII holder for per-call scratch.
template <typename T>
struct Scratch {
  T *ptr = nullptr;
  size_t cap = 0;
  cudaStream_t s = nullptr;
  Scratch() = default;
  explicit Scratch(cudaStream_t st) : s(st) {}
  int alloc(size_t n) {
    if (n == 0) return CPFIT_OK;
    ptr = (T *)scratch_get(n * sizeof(T), s, &cap);
    if (!ptr) {
      set_error("device allocation of %zu bytes failed", n * sizeof(T));
      return CPFIT_ENOMEM;
    }
    return CPFIT_OK;
  }
  ~Scratch() {
    if (ptr) scratch_put(ptr, cap, s);
  }
  Scratch(const Scratch &) = delete;
  Scratch &operator=(const Scratch &) = delete;
};

// ---- vector loads ---------------------------------------------------------
template <typename T, int VEC>
struct VecT;
template <> struct VecT<double, 1> { typedef double type; };
template <> struct VecT<double, 2> { typedef double2 type; };
template <> struct VecT<float, 1> { typedef float type; };
template <> struct VecT<float, 2> { typedef float2 type; };
template <> struct VecT<float, 4> { typedef float4 type; };

template <typename T, int VEC>
__device__ __forceinline__ void load_vec(const T *__restrict__ p, T (&v)[VEC]) {
  typedef typename VecT<T, VEC>::type V;
  V x = __ldg(reinterpret_cast<const V *>(p));
  if constexpr (VEC == 1) {
    v[0] = x;
  } else if constexpr (VEC == 2) {
    v[0] = x.x; v[1] = x.y;
  } else {
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
}

template <typename T, int VEC>
__device__ __forceinline__ void store_vec(T *__restrict__ p, const T (&v)[VEC]) {
  typedef typename VecT<T, VEC>::type V;
  V x;
  if constexpr (VEC == 1) {
    x = v[0];
  } else if constexpr (VEC == 2) {
    x.x = v[0]; x.y = v[1];
  } else {
    x.x = v[0]; x.y = v[1]; x.z = v[2]; x.w = v[3];
  }
  *reinterpret_cast<V *>(p) = x;
}

__device__ __forceinline__ double shfl_xor(double v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}
__device__ __forceinline__ float shfl_xor(float v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

template <typename T>
inline int pick_vec(int rank, const void *const *ptrs, int n) {
  size_t row_bytes = (size_t)rank * sizeof(T);
  int vec = 1;
  if (row_bytes % 16 == 0)
    vec = 16 / (int)sizeof(T);
  else if (row_bytes % 8 == 0 && sizeof(T) == 4)
    vec = 2;
  for (int i = 0; i < n; ++i)
    if (ptrs[i] && ((uintptr_t)ptrs[i] % (vec * sizeof(T)) != 0)) vec = 1;
  return vec;
}

// per-mode column pointers + coordinate arrays passed by value to kernels
struct CpfitCols {
  const double *col[CPFIT_MAXN];
  const int32_t *idx[CPFIT_MAXN];
};

struct CpfitDims {
  int64_t d[CPFIT_MAXN];
};
template <typename C>
struct CpfitCoordPtrs {
  const C *p[CPFIT_MAXN];
};

// ---- elementwise losses (losses.py:41-91) -----------------------------------
// loss 0: least squares  phi = (t - m)^2, dphi = 2 (m - t), d2phi = 2
// loss 1: Poisson log link  phi = exp(m~) - t m, dphi = exp(m~) - t,
//         d2phi = exp(m~), with m~ = min(m, 50) (POISSON_EXP_CLAMP);
// returns whether m was clamped (the reference counts those events).
#define CPFIT_POISSON_CLAMP 50.0
__device__ __forceinline__ bool loss_eval1(int loss, double t, double m, double &phi,
                                           double &d1, double &d2) {
  if (loss == 1) {
    const bool cl = m > CPFIT_POISSON_CLAMP;
    const double e = exp(cl ? CPFIT_POISSON_CLAMP : m);
    phi = __dsub_rn(e, __dmul_rn(t, m));
    d1 = __dsub_rn(e, t);
    d2 = e;
    return cl;
  }
  const double d = __dsub_rn(t, m);
  phi = __dmul_rn(d, d);
  d1 = __dmul_rn(2.0, __dsub_rn(m, t));
  d2 = 2.0;
  return false;
}

// ---- device scan (exclusive, int64 out) -----------------------------------
// out[i] = sum_{j<i} in[j] for i in [0, n]; out has n+1 entries (out[n] = total).
template <typename Tin>
int exclusive_scan(const Tin *in, int64_t *out, int64_t n, cudaStream_t s);

// stable LSD radix sort of positions by the low `bits` bits of uint64 keys
template <typename K>
int radix_sort_pairs(const K *keys, int64_t n, int bits, K *sorted_keys, int32_t *perm,
                     cudaStream_t s);

// gather: out[k] = in[idx[k]]
int gather_i32(const int32_t *in, const int32_t *idx, int32_t *out, int64_t n,
               cudaStream_t s);

inline unsigned grid_for(int64_t work, int threads, int per_thread = 1) {
  int64_t b = (work + (int64_t)threads * per_thread - 1) / ((int64_t)threads * per_thread);
  int64_t cap = (int64_t)num_sms() * 32;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace cpfit

// Opaque pattern handle (C-ABI) -- defined here for the kernel files.
struct CpfitModeLayout {
  bool built = false;
  int32_t *perm = nullptr;        // nnz (mode-sorted position -> entry); null = identity
  int64_t *offsets = nullptr;     // dim + 1
  int32_t *sorted_idx[CPFIT_MAXN] = {nullptr};  // coords of each mode, mode-sorted order
  bool owns_sorted[CPFIT_MAXN] = {false};
  // segmented-work tasks
  int64_t ntasks = 0, nslots = 0, nsplit = 0, task_size = 0;
  int64_t max_slots = 0;          // most tasks of one slice
  int64_t *task_begin = nullptr;  // ntasks + 1
  int32_t *task_row = nullptr;    // ntasks
  int32_t *task_slot = nullptr;   // ntasks (-1 = row owned by one task)
  int32_t *split_row = nullptr;   // nsplit
  int32_t *split_slot = nullptr;  // nsplit + 1
  int32_t *identity_perm = nullptr;  // materialised on request for mode 0
  bool borrowed = false;  // coarse task tables borrow perm / offsets / sorted_idx
};

struct cpfit_pattern {
  int order = 0;
  int64_t dims[CPFIT_MAXN] = {0};
  int64_t nnz = 0;
  int32_t *coords[CPFIT_MAXN] = {nullptr};
  int64_t task_size = 0;  // entries per segmented task; 0 = automatic (task_size_for)
  CpfitModeLayout modes[CPFIT_MAXN];
  int32_t *parent = nullptr;  // sampled patterns: entry -> entry of the source pattern
  // coarse task tables (task_size * CPFIT_COARSE_TASKS) for the Gram kernel:
  // fewer split rows, less partial-Gram traffic
  CpfitModeLayout coarse[CPFIT_MAXN];
};

#define CPFIT_COARSE_TASKS 8

namespace cpfit {
// Task granularity.  Persistent MTTKRP warps (148 SMs x 4 blocks x 8 warps)
// finish within ~1/8 of their work when there are >= 8 tasks per warp; longer
// tasks cost fewer row splits and task prologues.  Automatic size: nnz / (8 x
// warps), rounded up to 32 and clamped to [256, 1024] (cfg 2, 1e7 nnz: 288 --
// MTTKRP 0.189 -> 0.165 ms vs 1024; cfg 3, 1e8 nnz: 1024).  Coarse (Gram)
// tasks: 8192 entries in automatic mode, 8 x an explicit size otherwise.
inline int64_t task_size_for(const cpfit_pattern *p) {
  if (p->task_size > 0) return p->task_size;
  const int64_t warps = (int64_t)num_sms() * 4 * 8;
  int64_t ts = (p->nnz + 8 * warps - 1) / (8 * warps);
  ts = (ts + 31) / 32 * 32;
  return ts < 256 ? 256 : (ts > 1024 ? 1024 : ts);
}
inline int64_t coarse_task_size_for(const cpfit_pattern *p) {
  return p->task_size > 0 ? p->task_size * CPFIT_COARSE_TASKS : 8192;
}
int ensure_layout(cpfit_pattern *p, int mode, cudaStream_t s);
int ensure_coarse_layout(cpfit_pattern *p, int mode, cudaStream_t s);
}
