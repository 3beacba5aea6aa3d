// sparse_kernels.cu -- TTTP and segmented MTTKRP for sm_100a.
//
// Both kernels are gather-bound: per nonzero they stream N int32 indices and
// one value and gather N (TTTP) or N-1 (MTTKRP) factor rows of R values.
// A lane group of LPE lanes owns one nonzero at a time and gathers each
// factor row with 128-bit vector loads (one row = LPE lanes x 16 B, so a
// fp64 R=16 row is one 128 B line fetched by 8 lanes); 32/LPE nonzeros are
// in flight per warp instruction.  Indices and values are loaded coalesced,
// one nonzero per lane, and broadcast to the owning group with shuffles.
//
// TTTP reduces the R products of a nonzero with a shuffle tree inside its
// group.  MTTKRP walks the mode-sorted nonzeros task by task: a task is a
// contiguous run of one output row (long rows are split into several tasks,
// whose partial rows are combined in task order by a fix-up pass), so every
// output element is produced by exactly one warp with a fixed summation
// order: deterministic, no floating-point atomics.
//
// Reference: kernels.tttp (kernels.py:105-149) / _jit.tttp3 (_jit.py:49-59);
// kernels.mttkrp (kernels.py:46-91) / _jit.mttkrp3 (_jit.py:35-47).
#include "common.cuh"

namespace cpfit {

template <typename T>
struct TttpParams {
  int np;       // factors present (absent modes are dropped on the host)
  int rank;
  int64_t nnz;
  const int32_t *idx[CPFIT_MAXN];
  const T *fac[CPFIT_MAXN];
  const T *vals;
  T *out;
  int epi;        // 0: out = vals * acc;  1: out = alpha * acc + beta * vals
  T alpha, beta;
};

template <typename T, int VEC, int LPE, int KV, int NP>
__global__ void __launch_bounds__(256) tttp_kernel(const TttpParams<T> p) {
  constexpr int G = 32 / LPE;                      // nonzeros per warp step
  constexpr int NPM = NP > 0 ? NP : CPFIT_MAXN;    // register slots for indices
  const int np = NP > 0 ? NP : p.np;
  const int lane = threadIdx.x & 31;
  const int q = lane % LPE;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int rank = p.rank;

  for (int64_t base = warp * 32; base < p.nnz; base += nwarps * 32) {
    const int64_t e = base + lane;
    const bool valid = e < p.nnz;
    int32_t my_idx[NPM];
#pragma unroll
    for (int n = 0; n < NPM; ++n)
      my_idx[n] = (n < np && valid) ? __ldg(p.idx[n] + e) : 0;
    const T my_val = valid ? __ldg(p.vals + e) : T(0);
    T result = T(0);
#pragma unroll 4
    for (int s = 0; s < LPE; ++s) {
      const int j = s * G + lane / LPE;  // nonzero (within the 32) owned by my group
      T prod[KV][VEC];
#pragma unroll
      for (int n = 0; n < NPM; ++n) {
        if (n >= np) break;
        const int row = __shfl_sync(0xffffffffu, my_idx[n], j);
        const T *frow = p.fac[n] + (int64_t)row * rank;
#pragma unroll
        for (int k = 0; k < KV; ++k) {
          const int col = (k * LPE + q) * VEC;
          T x[VEC];
          if (col < rank) {
            load_vec<T, VEC>(frow + col, x);
          } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v) x[v] = T(0);
          }
#pragma unroll
          for (int v = 0; v < VEC; ++v) prod[k][v] = (n == 0) ? x[v] : prod[k][v] * x[v];
        }
      }
      T acc = T(0);
#pragma unroll
      for (int k = 0; k < KV; ++k)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc += prod[k][v];
#pragma unroll
      for (int o = LPE / 2; o > 0; o >>= 1) acc += shfl_xor(acc, o);
      const T got = __shfl_sync(0xffffffffu, acc, (lane % G) * LPE);
      if (lane / G == s) result = got;
    }
    if (valid) p.out[e] = p.epi == 0 ? my_val * result : p.alpha * result + p.beta * my_val;
  }
}

template <typename T>
struct MttkrpParams {
  int np;  // other modes
  int rank;
  const int32_t *idx[CPFIT_MAXN];  // mode-sorted coordinates of the other modes
  const T *fac[CPFIT_MAXN];
  const T *vals;          // canonical order if perm != null, else mode-sorted
  const int32_t *perm;    // mode-sorted position -> canonical entry
  const int64_t *task_begin;
  const int32_t *task_row;
  const int32_t *task_slot;
  int64_t ntasks;
  T *out;
  T *partial;
};

template <typename T, int VEC, int LPE, int KV, int NP>
__global__ void __launch_bounds__(256) mttkrp_kernel(const MttkrpParams<T> p) {
  constexpr int G = 32 / LPE;
  constexpr int NPM = NP > 0 ? NP : CPFIT_MAXN;
  const int np = NP > 0 ? NP : p.np;
  const int lane = threadIdx.x & 31;
  const int g = lane / LPE, q = lane % LPE;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int rank = p.rank;

  for (int64_t t = warp; t < p.ntasks; t += nwarps) {
    const int64_t b0 = p.task_begin[t], b1 = p.task_begin[t + 1];
    T acc[KV][VEC];
#pragma unroll
    for (int k = 0; k < KV; ++k)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[k][v] = T(0);

    for (int64_t base = b0; base < b1; base += 32) {
      const int64_t e = base + lane;
      const bool valid = e < b1;
      int32_t my_idx[NPM];
#pragma unroll
      for (int n = 0; n < NPM; ++n)
        my_idx[n] = (n < np && valid) ? __ldg(p.idx[n] + e) : 0;
      T my_val = T(0);
      if (valid) my_val = p.perm ? __ldg(p.vals + __ldg(p.perm + e)) : __ldg(p.vals + e);
      const int cnt = (int)(b1 - base < 32 ? b1 - base : 32);
#pragma unroll 4
      for (int s = 0; s < LPE; ++s) {
        const int j = s * G + g;
        const T v = __shfl_sync(0xffffffffu, my_val, j);
        int rows[NPM];
#pragma unroll
        for (int n = 0; n < NPM; ++n)
          if (n < np) rows[n] = __shfl_sync(0xffffffffu, my_idx[n], j);
        if (j < cnt) {
          T prod[KV][VEC];
#pragma unroll
          for (int n = 0; n < NPM; ++n) {
            if (n >= np) break;
            const T *frow = p.fac[n] + (int64_t)rows[n] * rank;
#pragma unroll
            for (int k = 0; k < KV; ++k) {
              const int col = (k * LPE + q) * VEC;
              T x[VEC];
              if (col < rank) {
                load_vec<T, VEC>(frow + col, x);
              } else {
#pragma unroll
                for (int w = 0; w < VEC; ++w) x[w] = T(0);
              }
#pragma unroll
              for (int w = 0; w < VEC; ++w) prod[k][w] = (n == 0) ? x[w] : prod[k][w] * x[w];
            }
          }
#pragma unroll
          for (int k = 0; k < KV; ++k)
#pragma unroll
            for (int w = 0; w < VEC; ++w) acc[k][w] += prod[k][w] * v;
        }
      }
    }
    // combine the G groups (fixed tree order)
#pragma unroll
    for (int o = LPE; o < 32; o <<= 1)
#pragma unroll
      for (int k = 0; k < KV; ++k)
#pragma unroll
        for (int w = 0; w < VEC; ++w) acc[k][w] += shfl_xor(acc[k][w], o);
    if (g == 0) {
      const int slot = p.task_slot[t];
      T *dst = slot < 0 ? p.out + (int64_t)p.task_row[t] * rank
                        : p.partial + (int64_t)slot * rank;
#pragma unroll
      for (int k = 0; k < KV; ++k) {
        const int col = (k * LPE + q) * VEC;
        if (col < rank) store_vec<T, VEC>(dst + col, acc[k]);
      }
    }
  }
}

// Sum the partial rows of split slices in task order.
template <typename T>
__global__ void combine_partials(const int32_t *__restrict__ split_row,
                                 const int32_t *__restrict__ split_slot, int64_t nsplit,
                                 int rank, const T *__restrict__ partial, T *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < nsplit; s += nwarps) {
    const int64_t row = split_row[s];
    const int64_t a = split_slot[s], b = split_slot[s + 1];
    for (int c = lane; c < rank; c += 32) {
      T acc = partial[a * rank + c];
      for (int64_t k = a + 1; k < b; ++k) acc += partial[k * rank + c];
      out[row * rank + c] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// dispatch

template <typename T, int VEC, int LPE, int KV>
static int launch_tttp_np(const TttpParams<T> &p, cudaStream_t s) {
  const unsigned grid = grid_for((p.nnz + 31) / 32 * 32, 256);
  if (p.np == 3)
    tttp_kernel<T, VEC, LPE, KV, 3><<<grid, 256, 0, s>>>(p);
  else if (p.np == 4)
    tttp_kernel<T, VEC, LPE, KV, 4><<<grid, 256, 0, s>>>(p);
  else
    tttp_kernel<T, VEC, LPE, KV, 0><<<grid, 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("tttp_kernel");
  return CPFIT_OK;
}

template <typename T, int VEC, int LPE, int KV>
static int launch_mttkrp_np(const MttkrpParams<T> &p, cudaStream_t s) {
  int64_t blocks = (p.ntasks + 7) / 8;
  int64_t cap = (int64_t)num_sms() * 8;
  const unsigned grid = (unsigned)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
  if (p.np == 2)
    mttkrp_kernel<T, VEC, LPE, KV, 2><<<grid, 256, 0, s>>>(p);
  else if (p.np == 3)
    mttkrp_kernel<T, VEC, LPE, KV, 3><<<grid, 256, 0, s>>>(p);
  else
    mttkrp_kernel<T, VEC, LPE, KV, 0><<<grid, 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("mttkrp_kernel");
  return CPFIT_OK;
}

// Select <VEC, LPE, KV> for the row tiling and call F<...>::run(p, s).
#define CPFIT_TILING_SWITCH(T, VECV, TIL, LAUNCH, P, S)                                   \
  do {                                                                                     \
    if ((TIL).lpe == 4) return LAUNCH<T, VECV, 4, 1>(P, S);                                \
    if ((TIL).lpe == 8) return LAUNCH<T, VECV, 8, 1>(P, S);                                \
    if ((TIL).lpe == 16) return LAUNCH<T, VECV, 16, 1>(P, S);                              \
    if ((TIL).kv == 1) return LAUNCH<T, VECV, 32, 1>(P, S);                                \
    if ((TIL).kv == 2) return LAUNCH<T, VECV, 32, 2>(P, S);                                \
    return LAUNCH<T, VECV, 32, 4>(P, S);                                                   \
  } while (0)

template <typename T>
static int dispatch_tttp(const TttpParams<T> &p, int vec, cudaStream_t s) {
  RowTiling til = pick_tiling(p.rank, vec, 4);
  if (til.kv < 0) {
    set_error("rank %d too large for the TTTP kernel", p.rank);
    return CPFIT_EINVAL;
  }
  if (til.kv == 3) til.kv = 4;
  if constexpr (sizeof(T) == 8) {
    if (vec == 2) CPFIT_TILING_SWITCH(T, 2, til, launch_tttp_np, p, s);
    CPFIT_TILING_SWITCH(T, 1, til, launch_tttp_np, p, s);
  } else {
    if (vec == 4) CPFIT_TILING_SWITCH(T, 4, til, launch_tttp_np, p, s);
    if (vec == 2) CPFIT_TILING_SWITCH(T, 2, til, launch_tttp_np, p, s);
    CPFIT_TILING_SWITCH(T, 1, til, launch_tttp_np, p, s);
  }
}

template <typename T>
static int dispatch_mttkrp(const MttkrpParams<T> &p, int vec, cudaStream_t s) {
  RowTiling til = pick_tiling(p.rank, vec, 4);
  if (til.kv < 0) {
    set_error("rank %d too large for the MTTKRP kernel", p.rank);
    return CPFIT_EINVAL;
  }
  if (til.kv == 3) til.kv = 4;
  if constexpr (sizeof(T) == 8) {
    if (vec == 2) CPFIT_TILING_SWITCH(T, 2, til, launch_mttkrp_np, p, s);
    CPFIT_TILING_SWITCH(T, 1, til, launch_mttkrp_np, p, s);
  } else {
    if (vec == 4) CPFIT_TILING_SWITCH(T, 4, til, launch_mttkrp_np, p, s);
    if (vec == 2) CPFIT_TILING_SWITCH(T, 2, til, launch_mttkrp_np, p, s);
    CPFIT_TILING_SWITCH(T, 1, til, launch_mttkrp_np, p, s);
  }
}

template <typename T>
static int run_tttp(cpfit_pattern *pt, int rank, const void *vals, const void *const *factors,
                    void *out, cudaStream_t s, int epi = 0, double alpha = 0.0,
                    double beta = 0.0) {
  TttpParams<T> p{};
  p.epi = epi;
  p.alpha = (T)alpha;
  p.beta = (T)beta;
  p.rank = rank;
  p.nnz = pt->nnz;
  p.vals = (const T *)vals;
  p.out = (T *)out;
  int np = 0;
  const void *ptrs[CPFIT_MAXN];
  for (int n = 0; n < pt->order; ++n) {
    if (!factors[n]) continue;
    p.idx[np] = pt->coords[n];
    p.fac[np] = (const T *)factors[n];
    ptrs[np] = factors[n];
    ++np;
  }
  if (np == 0) {
    set_error("at least one factor matrix must be provided");
    return CPFIT_EINVAL;
  }
  p.np = np;
  if (pt->nnz == 0) return CPFIT_OK;
  return dispatch_tttp<T>(p, pick_vec<T>(rank, ptrs, np), s);
}

template <typename T>
static int run_mttkrp(cpfit_pattern *pt, int mode, int rank, const void *vals, int vals_sorted,
                      const void *const *factors, void *out, cudaStream_t s) {
  const int64_t dim = pt->dims[mode];
  CPFIT_CUDA(cudaMemsetAsync(out, 0, (size_t)dim * rank * sizeof(T), s));
  if (pt->nnz == 0) return CPFIT_OK;
  CPFIT_TRY(ensure_layout(pt, mode, s));
  CpfitModeLayout &L = pt->modes[mode];
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
  Scratch<T> partial(s);
  if (L.nslots > 0) CPFIT_TRY(partial.alloc((size_t)L.nslots * rank));
  p.partial = partial.ptr;
  if (np == 0) {
    // order-1 tensor: out[i] = sum of values in row i (empty product = 1)
    set_error("mttkrp needs an order >= 2 tensor");
    return CPFIT_EINVAL;
  }
  CPFIT_TRY(dispatch_mttkrp<T>(p, pick_vec<T>(rank, ptrs, np), s));
  if (L.nsplit > 0) {
    combine_partials<T><<<grid_for(L.nsplit * 32, 256), 256, 0, s>>>(
        L.split_row, L.split_slot, L.nsplit, rank, partial.ptr, (T *)out);
    CPFIT_LAUNCH_CHECK("combine_partials");
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

}  // extern "C"
