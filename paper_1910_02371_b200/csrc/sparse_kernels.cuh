// sparse_kernels.cuh -- TTTP and segmented MTTKRP for sm_100a (templates;
// instantiated per dtype in tttp_f64.cu, tttp_f32.cu, mttkrp_f64.cu,
// mttkrp_f32.cu so nvcc compiles them in parallel).
//
// Both kernels are gather-bound: per nonzero they stream N int32 indices and
// one value and gather N (TTTP) or N-1 (MTTKRP) factor rows of R values.
// A lane group of LPE lanes owns one nonzero at a time and gathers each
// factor row with 128-bit vector loads (one row = LPE lanes x 16 B, so a
// fp64 R=16 row is one 128 B line fetched by 8 lanes); 32/LPE nonzeros are
// in flight per warp instruction.  Indices and values are loaded coalesced,
// one nonzero per lane, and broadcast to the owning group with shuffles.
//
// TTTP finishes the group sums with one transposed butterfly per batch.  MTTKRP walks the mode-sorted nonzeros task by task: a task is a
// contiguous run of one output row (long rows are split into several tasks,
// whose partial rows are combined in task order by a fix-up pass), so every
// output element is produced by exactly one warp with a fixed summation
// order: deterministic, no floating-point atomics.
//
// Reference: kernels.tttp (kernels.py:105-149) / _jit.tttp3 (_jit.py:49-59);
// kernels.mttkrp (kernels.py:46-91) / _jit.mttkrp3 (_jit.py:35-47).
#pragma once
#include "common.cuh"

// Min resident 256-thread blocks per SM (register cap) and the fp64 MTTKRP
// lane tiling, tuned on B200 with tools/tiling_sweep.py (profiles/r1_tuning.md).
#ifndef CPFIT_TTTP_MINB
#define CPFIT_TTTP_MINB 2
#endif
#ifndef CPFIT_MTTKRP_MINB
#define CPFIT_MTTKRP_MINB 4  // fp64 (cfg 2: 0.196 -> 0.188 ms vs 3)
#endif
#ifndef CPFIT_MTTKRP_MINB_F32
#define CPFIT_MTTKRP_MINB_F32 3  // fp32 (cfg 5 SGD samples: 4 cost ~1 ms per step)
#endif
#ifndef CPFIT_TTTP_MINB_F32
#define CPFIT_TTTP_MINB_F32 4  // fp32 (cfg 5-like 2e7 nnz: 1.078 -> 0.865 ms with U0 = 2)
#endif
#ifndef CPFIT_TTTP_U0
#define CPFIT_TTTP_U0 4  // TTTP sub-iterations in flight when the mode-0 row is hoisted
#endif
#ifndef CPFIT_TTTP_U0_F32
#define CPFIT_TTTP_U0_F32 2
#endif
#ifndef CPFIT_MTTKRP_U
#define CPFIT_MTTKRP_U 4  // sub-iterations of gathers in flight per MTTKRP round (fp32)
#endif
#ifndef CPFIT_MTTKRP_U64
// fp64: 2 (cfg 2 0.1657 -> 0.1615 ms, cfg 3-like mode 0 0.766 -> 0.706 ms; 8 is 3-13 %
// slower, 1 is 12 % slower; fp32 prefers 4: profiles/r2_tuning.md)
#define CPFIT_MTTKRP_U64 2
#endif
#ifndef CPFIT_MTTKRP_KVT64
#define CPFIT_MTTKRP_KVT64 1
#endif

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
  int epi;        // 0: out = vals * acc;  1: out = alpha * acc + beta * vals;
                  // 2: loss derivatives at m = acc, t = vals: out = dphi, out2 = d2phi
  T alpha, beta;
  int loss;                       // epi 2: loss id (common.cuh loss_eval1)
  T *out2;                        // epi 2: d2phi
  unsigned long long *clamped;    // epi 2: count of clamped model values (nullable)
};

// Gather the factor rows of U consecutive nonzero slots (j = (s0+u)*G + g)
// of the current 32-entry batch into registers.  Every load of the U entries
// is issued before any is consumed (memory-level parallelism, no branches in
// between).  `fq[n]` is the lane's base pointer (factor n + q*VEC), so a row
// address is one 32-bit multiply + one wide add; column offsets are
// immediates.  FULL: the tiling covers the rank exactly (no column predicate).
// N0 = first mode gathered (1: the mode-0 row is uniform over the batch and
// already in registers, see tttp_kernel).
template <typename T, int VEC, int LPE, int KV, int NPM, int U, bool FULL, int N0 = 0>
__device__ __forceinline__ void gather_rows(const T *const (&fq)[NPM],
                                            const int32_t (&my_idx)[NPM], int np,
                                            unsigned rank, int s0, int g, int q,
                                            T (&x)[U][NPM][KV][VEC]) {
  constexpr int G = 32 / LPE;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int j = (s0 + u) * G + g;
#pragma unroll
    for (int n = N0; n < NPM; ++n) {
      if (n >= np) break;
      const unsigned row = (unsigned)__shfl_sync(0xffffffffu, my_idx[n], j);
      const T *frow = reinterpret_cast<const T *>(reinterpret_cast<const char *>(fq[n]) +
                                                  (unsigned long long)row * (rank * (unsigned)sizeof(T)));
#pragma unroll
      for (int k = 0; k < KV; ++k) {
        if (FULL || (unsigned)((k * LPE + q) * VEC) < rank) {
          load_vec<T, VEC>(frow + k * LPE * VEC, x[u][n][k]);
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) x[u][n][k][v] = T(0);
        }
      }
    }
  }
}

// Generic-order variant (any number of present modes): multiplies each row
// into a running product instead of keeping every row in registers.
template <typename T, int VEC, int LPE, int KV, int NPM>
__device__ __forceinline__ void gather_product(const T *const (&fq)[NPM],
                                               const int32_t (&my_idx)[NPM], int np,
                                               unsigned rank, int s, int g, int q,
                                               T (&prod)[KV][VEC]) {
  constexpr int G = 32 / LPE;
  const int j = s * G + g;
#pragma unroll 1
  for (int n = 0; n < np; ++n) {
    int32_t mine = my_idx[0];
#pragma unroll
    for (int m = 1; m < NPM; ++m)
      if (m == n) mine = my_idx[m];
    const unsigned row = (unsigned)__shfl_sync(0xffffffffu, mine, j);
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      T x[VEC];
      if ((unsigned)((k * LPE + q) * VEC) < rank) {
        const T *base = nullptr;
#pragma unroll
        for (int m = 0; m < NPM; ++m)
          if (m == n) base = fq[m];
        load_vec<T, VEC>(base + (size_t)row * rank + k * LPE * VEC, x);
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) x[v] = T(0);
      }
#pragma unroll
      for (int v = 0; v < VEC; ++v) prod[k][v] = n == 0 ? x[v] : prod[k][v] * x[v];
    }
  }
}

// TTTP: warp = 32 consecutive nonzeros, G = 32/LPE groups of LPE lanes.
// Sub-iteration s gathers the rows of nonzero j = s*G + g into group g; every
// lane accumulates its column slice's partial product-sum for each of the LPE
// nonzeros its group visits (part[s]).  One transposed (reduce-scatter)
// butterfly over the group then leaves lane q with the full sum of nonzero
// q*G + g: LPE-1 shuffles per LPE nonzeros instead of log2(LPE)+1 per
// nonzero.  Values and outputs are accessed in that permuted but coalesced
// order.
template <typename T, int VEC, int LPE, int KV, int NP, bool FULL>
__global__ void __launch_bounds__(256, sizeof(T) == 8 ? CPFIT_TTTP_MINB : CPFIT_TTTP_MINB_F32)
    tttp_kernel(const TttpParams<T> p) {
  constexpr int G = 32 / LPE;                      // nonzeros per warp step
  constexpr int NPM = NP > 0 ? NP : CPFIT_MAXN;    // register slots for indices
  constexpr int U = NP > 0 ? (LPE < 4 ? LPE : 4) : 1;
  const int np = NP > 0 ? NP : p.np;
  const int lane = threadIdx.x & 31;
  const int g = lane / LPE, q = lane % LPE;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t stride = (((int64_t)gridDim.x * blockDim.x) >> 5) * 32;
  const unsigned rank = (unsigned)p.rank;
  const T *fq[NPM];
#pragma unroll
  for (int n = 0; n < NPM; ++n) fq[n] = n < np ? p.fac[n] + q * VEC : nullptr;
  const int my_slot = q * G + g;  // the nonzero of the batch this lane finishes

  int32_t my_idx[NPM];
  int64_t base = warp * 32;
  {
    const int64_t e = base + lane;
    const bool ok = e < p.nnz;
#pragma unroll
    for (int n = 0; n < NPM; ++n) my_idx[n] = (n < np && ok) ? __ldg(p.idx[n] + e) : 0;
  }
  for (; base < p.nnz; base += stride) {
    // prefetch the next batch's indices (software pipelining)
    int32_t nx_idx[NPM];
    {
      const int64_t e = base + stride + lane;
      const bool ok = e < p.nnz;
#pragma unroll
      for (int n = 0; n < NPM; ++n) nx_idx[n] = (n < np && ok) ? __ldg(p.idx[n] + e) : 0;
    }
    const int64_t eo = base + my_slot;
    const bool out_ok = eo < p.nnz;
    const T my_val = out_ok ? __ldg(p.vals + eo) : T(0);
    T part[LPE];
    if constexpr (NP > 0) {
      // canonical (key-sorted) order: the mode-0 index is constant over runs of
      // nnz / I_0 entries (cfg 2: ~1000, cfg 5: ~10^4), so most batches share
      // one mode-0 row.  Then it is gathered once per batch into registers and
      // only the other NP-1 rows per nonzero (same products, same order).
      const int32_t i0 = __shfl_sync(0xffffffffu, my_idx[0], 0);
      const bool uni0 = NP > 1 && __all_sync(0xffffffffu, my_idx[0] == i0);
      if (uni0) {
        T r0[KV][VEC];
        {
          const T *frow = reinterpret_cast<const T *>(
              reinterpret_cast<const char *>(fq[0]) +
              (unsigned long long)(unsigned)i0 * (rank * (unsigned)sizeof(T)));
#pragma unroll
          for (int k = 0; k < KV; ++k) {
            if (FULL || (unsigned)((k * LPE + q) * VEC) < rank) {
              load_vec<T, VEC>(frow + k * LPE * VEC, r0[k]);
            } else {
#pragma unroll
              for (int v = 0; v < VEC; ++v) r0[k][v] = T(0);
            }
          }
        }
        constexpr int U0M = sizeof(T) == 8 ? CPFIT_TTTP_U0 : CPFIT_TTTP_U0_F32;
        constexpr int U0S = U * U0M / 4 < 1 ? 1 : U * U0M / 4;
        constexpr int U0 = U0S <= LPE ? U0S : LPE;
#pragma unroll
        for (int s0 = 0; s0 < LPE; s0 += U0) {
          T x[U0][NPM][KV][VEC];
          gather_rows<T, VEC, LPE, KV, NPM, U0, FULL, 1>(fq, my_idx, np, rank, s0, g, q, x);
#pragma unroll
          for (int u = 0; u < U0; ++u) {
            T acc = T(0);
#pragma unroll
            for (int k = 0; k < KV; ++k)
#pragma unroll
              for (int v = 0; v < VEC; ++v) {
                T prod = r0[k][v];
#pragma unroll
                for (int n = 1; n < NPM; ++n) prod = prod * x[u][n][k][v];
                acc += prod;
              }
            part[s0 + u] = acc;
          }
        }
      } else {
#pragma unroll
        for (int s0 = 0; s0 < LPE; s0 += U) {
          T x[U][NPM][KV][VEC];
          gather_rows<T, VEC, LPE, KV, NPM, U, FULL>(fq, my_idx, np, rank, s0, g, q, x);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            T acc = T(0);
#pragma unroll
            for (int k = 0; k < KV; ++k)
#pragma unroll
              for (int v = 0; v < VEC; ++v) {
                T prod = x[u][0][k][v];
#pragma unroll
                for (int n = 1; n < NPM; ++n) prod = prod * x[u][n][k][v];
                acc += prod;
              }
            part[s0 + u] = acc;
          }
        }
      }
    } else {
#pragma unroll
      for (int s = 0; s < LPE; ++s) {
        T prod[KV][VEC];
        gather_product<T, VEC, LPE, KV, NPM>(fq, my_idx, np, rank, s, g, q, prod);
        T acc = T(0);
#pragma unroll
        for (int k = 0; k < KV; ++k)
#pragma unroll
          for (int v = 0; v < VEC; ++v) acc += prod[k][v];
        part[s] = acc;
      }
    }
    // reduce-scatter over the LPE lanes of the group: lane q ends with the
    // total of nonzero s = q (fixed butterfly order: deterministic)
#pragma unroll
    for (int half = LPE / 2; half > 0; half >>= 1) {
      const bool upper = (q & half) != 0;
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const T keep = upper ? part[half + i] : part[i];
        const T send = upper ? part[i] : part[half + i];
        part[i] = keep + shfl_xor(send, half);
      }
    }
    if (p.epi < 2) {
      if (out_ok)
        p.out[eo] = p.epi == 0 ? my_val * part[0] : p.alpha * part[0] + p.beta * my_val;
    } else {
      // fused loss epilogue (generalized losses, losses.py:117-123)
      double phi, d1, d2;
      const bool cl = out_ok && loss_eval1(p.loss, (double)my_val, (double)part[0], phi, d1, d2);
      if (out_ok) {
        p.out[eo] = (T)d1;
        p.out2[eo] = (T)d2;
      }
      const unsigned nc = __ballot_sync(0xffffffffu, cl);
      if (nc && lane == 0 && p.clamped) atomicAdd(p.clamped, (unsigned long long)__popc(nc));
    }
#pragma unroll
    for (int n = 0; n < NPM; ++n) my_idx[n] = nx_idx[n];
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
  // Gram-free normal-equations product (MV kernels): out_i = sum_e w_e h_e (h_e . x_i)
  const T *xvec;               // I_mode x rank
  const int32_t *row_active;   // nullable: rows with 0 are skipped (their output is 0)
};

// One batch of up to 32 entries: coalesced indices (row 0 and value 0 past
// the end, so padded slots contribute exactly nothing) and values.
template <typename T, int NPM>
__device__ __forceinline__ void mttkrp_load_batch(const MttkrpParams<T> &p, int np, int64_t e,
                                                  int64_t end, int32_t (&ix)[NPM], T &v) {
  const bool ok = e < end;
#pragma unroll
  for (int n = 0; n < NPM; ++n) ix[n] = (n < np && ok) ? __ldg(p.idx[n] + e) : 0;
  v = T(0);
  if (ok) v = !p.vals ? T(1) : p.perm ? __ldg(p.vals + __ldg(p.perm + e)) : __ldg(p.vals + e);
}

// MV: the entry weight is w_e (h_e . x_row) with x_row the task row's slice of
// p.xvec -- the per-row normal-equations product G_i x_i of implicit-CG ALS,
// without materialising G ("ALS with implicit CG").
template <typename T, int VEC, int LPE, int KV, int NP, bool FULL, bool MV = false>
__global__ void __launch_bounds__(256, sizeof(T) == 8 ? CPFIT_MTTKRP_MINB : CPFIT_MTTKRP_MINB_F32)
    mttkrp_kernel(const MttkrpParams<T> p) {
  constexpr int G = 32 / LPE;
  constexpr int NPM = NP > 0 ? NP : CPFIT_MAXN;
  constexpr int UT = sizeof(T) == 8 ? CPFIT_MTTKRP_U64 : CPFIT_MTTKRP_U;
  constexpr int U = NP > 0 ? (LPE < UT ? LPE : UT) : 1;
  const int np = NP > 0 ? NP : p.np;
  const int lane = threadIdx.x & 31;
  const int g = lane / LPE, q = lane % LPE;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned rank = (unsigned)p.rank;
  const T *fq[NPM];
#pragma unroll
  for (int n = 0; n < NPM; ++n) fq[n] = n < np ? p.fac[n] + q * VEC : nullptr;

  // persistent warps: boundaries of the next task are fetched one task ahead
  int64_t nb0 = warp < p.ntasks ? p.task_begin[warp] : 0;
  int64_t nb1 = warp < p.ntasks ? p.task_begin[warp + 1] : 0;
  for (int64_t t = warp; t < p.ntasks; t += nwarps) {
    const int64_t b0 = nb0;
    int64_t b1 = nb1;
    if (t + nwarps < p.ntasks) {
      nb0 = p.task_begin[t + nwarps];
      nb1 = p.task_begin[t + nwarps + 1];
    }
    T xr[MV ? KV : 1][MV ? VEC : 1];
    if constexpr (MV) {
      const int64_t row = p.task_row[t];
      if (p.row_active && !p.row_active[row]) b1 = b0;  // converged row: contributes 0
#pragma unroll
      for (int k = 0; k < KV; ++k) {
        const int col = (k * LPE + q) * VEC;
        if (FULL || col < (int)rank) {
          load_vec<T, VEC>(p.xvec + row * rank + col, xr[k]);
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) xr[k][v] = T(0);
        }
      }
    }
    T acc[KV][VEC];
#pragma unroll
    for (int k = 0; k < KV; ++k)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[k][v] = T(0);

    int32_t my_idx[NPM];
    T my_val;
    mttkrp_load_batch<T, NPM>(p, np, b0 + lane, b1, my_idx, my_val);
    for (int64_t base = b0; base < b1; base += 32) {
      int32_t nx_idx[NPM];
      T nx_val;
      mttkrp_load_batch<T, NPM>(p, np, base + 32 + lane, b1, nx_idx, nx_val);
      const int cnt = (int)(b1 - base < 32 ? b1 - base : 32);
#pragma unroll
      for (int s0 = 0; s0 < LPE; s0 += U) {
        if (s0 * G >= cnt) break;  // warp-uniform: the rest of the batch is empty
        if constexpr (NP > 0) {
          T x[U][NPM][KV][VEC];
          gather_rows<T, VEC, LPE, KV, NPM, U, FULL>(fq, my_idx, np, rank, s0, g, q, x);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            T v = __shfl_sync(0xffffffffu, my_val, (s0 + u) * G + g);
            if constexpr (MV) {
              T d = T(0);
#pragma unroll
              for (int k = 0; k < KV; ++k)
#pragma unroll
                for (int w = 0; w < VEC; ++w) {
                  T prod = x[u][0][k][w];
#pragma unroll
                  for (int n = 1; n < NPM; ++n) prod = prod * x[u][n][k][w];
                  x[u][0][k][w] = prod;
                  d += prod * xr[k][w];
                }
#pragma unroll
              for (int o = LPE / 2; o > 0; o >>= 1) d += shfl_xor(d, o);
              v *= d;
#pragma unroll
              for (int k = 0; k < KV; ++k)
#pragma unroll
                for (int w = 0; w < VEC; ++w) acc[k][w] += x[u][0][k][w] * v;
            } else {
#pragma unroll
              for (int k = 0; k < KV; ++k)
#pragma unroll
                for (int w = 0; w < VEC; ++w) {
                  T prod = x[u][0][k][w];
#pragma unroll
                  for (int n = 1; n < NPM; ++n) prod = prod * x[u][n][k][w];
                  acc[k][w] += prod * v;
                }
            }
          }
        } else {
          T prod[KV][VEC];
          gather_product<T, VEC, LPE, KV, NPM>(fq, my_idx, np, rank, s0, g, q, prod);
          T v = __shfl_sync(0xffffffffu, my_val, s0 * G + g);
          if constexpr (MV) {
            T d = T(0);
#pragma unroll
            for (int k = 0; k < KV; ++k)
#pragma unroll
              for (int w = 0; w < VEC; ++w) d += prod[k][w] * xr[k][w];
#pragma unroll
            for (int o = LPE / 2; o > 0; o >>= 1) d += shfl_xor(d, o);
            v *= d;
          }
#pragma unroll
          for (int k = 0; k < KV; ++k)
#pragma unroll
            for (int w = 0; w < VEC; ++w) acc[k][w] += prod[k][w] * v;
        }
      }
#pragma unroll
      for (int n = 0; n < NPM; ++n) my_idx[n] = nx_idx[n];
      my_val = nx_val;
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
        if (FULL || col < (int)rank) store_vec<T, VEC>(dst + col, acc[k]);
      }
    }
  }
}

// Sum the partial rows of split slices in a fixed order (deterministic).
// Rows with few slots: warp per row, slots summed in task order (lane =
// column).  Rows with many slots (Zipf heads: thousands): block per row,
// warp w takes slots a + w, a + w + 8, ..., then the 8 warp sums are added in
// warp order.  Each kernel skips the other's rows.
constexpr int COMBINE_LONG = 64;

template <typename T>
__global__ void combine_partials(const int32_t *__restrict__ split_row,
                                 const int32_t *__restrict__ split_slot, int64_t nsplit,
                                 int rank, const T *__restrict__ partial, T *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < nsplit; s += nwarps) {
    const int64_t a = split_slot[s], b = split_slot[s + 1];
    if (b - a > COMBINE_LONG) continue;
    const int64_t row = split_row[s];
    for (int c = lane; c < rank; c += 32) {
      T acc = partial[a * rank + c];
      for (int64_t k = a + 1; k < b; ++k) acc += partial[k * rank + c];
      out[row * rank + c] = acc;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) combine_partials_long(
    const int32_t *__restrict__ split_row, const int32_t *__restrict__ split_slot,
    int64_t nsplit, int rank, const T *__restrict__ partial, T *__restrict__ out) {
  __shared__ T red[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t s = blockIdx.x; s < nsplit; s += gridDim.x) {
    const int64_t a = split_slot[s], b = split_slot[s + 1];
    if (b - a <= COMBINE_LONG) continue;  // block-uniform
    const int64_t row = split_row[s];
    for (int c0 = 0; c0 < rank; c0 += 32) {
      const int c = c0 + lane;
      T acc = T(0);
      if (c < rank)
        for (int64_t k = a + w; k < b; k += 8) acc += partial[k * rank + c];
      red[w][lane] = acc;
      __syncthreads();
      if (w == 0 && c < rank) {
        T tot = red[0][lane];
#pragma unroll
        for (int j = 1; j < 8; ++j) tot += red[j][lane];
        out[row * rank + c] = tot;
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// launch + lane-tiling dispatch (instantiated per dtype in tttp_f64.cu, ...)

template <typename T, int VEC, int LPE, int KV>
static int launch_tttp_np(const TttpParams<T> &p, cudaStream_t s) {
  const unsigned grid = grid_for((p.nnz + 31) / 32 * 32, 256);
  const bool full = p.rank == LPE * VEC * KV;
  constexpr bool HOT = (sizeof(T) == 8 && VEC == 2) || (sizeof(T) == 4 && VEC == 4);
  if constexpr (HOT) {
    if (p.np == 3 && full) {
      tttp_kernel<T, VEC, LPE, KV, 3, true><<<grid, 256, 0, s>>>(p);
      CPFIT_LAUNCH_CHECK("tttp_kernel");
      return CPFIT_OK;
    }
    if (p.np == 4 && full) {
      tttp_kernel<T, VEC, LPE, KV, 4, true><<<grid, 256, 0, s>>>(p);
      CPFIT_LAUNCH_CHECK("tttp_kernel");
      return CPFIT_OK;
    }
    if (p.np == 3) {  // ranks the lane tiling does not cover exactly (e.g. R = 10)
      tttp_kernel<T, VEC, LPE, KV, 3, false><<<grid, 256, 0, s>>>(p);
      CPFIT_LAUNCH_CHECK("tttp_kernel");
      return CPFIT_OK;
    }
  }
  tttp_kernel<T, VEC, LPE, KV, 0, false><<<grid, 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("tttp_kernel");
  return CPFIT_OK;
}

template <typename T, int VEC, int LPE, int KV, bool MV = false>
static int launch_mttkrp_np(const MttkrpParams<T> &p, cudaStream_t s) {
  // persistent grid: exactly the resident capacity (no partial waves)
  int64_t blocks = (p.ntasks + 7) / 8;
  const int64_t cap =
      (int64_t)num_sms() * (sizeof(T) == 8 ? CPFIT_MTTKRP_MINB : CPFIT_MTTKRP_MINB_F32);
  const unsigned grid = (unsigned)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
  const bool full = p.rank == LPE * VEC * KV;
  constexpr bool HOT = (sizeof(T) == 8 && VEC == 2) || (sizeof(T) == 4 && VEC == 4);
  if constexpr (HOT) {
    if (p.np == 2 && full) {
      mttkrp_kernel<T, VEC, LPE, KV, 2, true, MV><<<grid, 256, 0, s>>>(p);
      CPFIT_LAUNCH_CHECK("mttkrp_kernel");
      return CPFIT_OK;
    }
    if (p.np == 3 && full) {
      mttkrp_kernel<T, VEC, LPE, KV, 3, true, MV><<<grid, 256, 0, s>>>(p);
      CPFIT_LAUNCH_CHECK("mttkrp_kernel");
      return CPFIT_OK;
    }
    if (p.np == 2) {  // ranks the lane tiling does not cover exactly (e.g. R = 10)
      mttkrp_kernel<T, VEC, LPE, KV, 2, false, MV><<<grid, 256, 0, s>>>(p);
      CPFIT_LAUNCH_CHECK("mttkrp_kernel");
      return CPFIT_OK;
    }
  }
  mttkrp_kernel<T, VEC, LPE, KV, 0, false, MV><<<grid, 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("mttkrp_kernel");
  return CPFIT_OK;
}

// Tiling policies (tools/tiling_sweep.py, profiles/r1_tuning.md):
//  TTTP   -- 8 lanes per nonzero (LPE = 8, fewer when the row is narrower),
//            KV = ceil(nv / 8) vectors per lane.
//  MTTKRP -- CPFIT_MTTKRP_KVT64 vectors per lane for fp64, 1 for fp32.
// (lpe, kv) pairs outside the instantiated set fall back to LPE = 32.
template <typename F>
static int tttp_tiling_dispatch(int nv, F &&f) {
  if (nv <= 1) return f.template operator()<1, 1>();
  if (nv <= 2) return f.template operator()<2, 1>();
  if (nv <= 4) return f.template operator()<4, 1>();
  if (nv <= 8) return f.template operator()<8, 1>();
  if (nv <= 16) return f.template operator()<8, 2>();
  if (nv <= 32) return f.template operator()<8, 4>();
  if (nv <= 64) return f.template operator()<8, 8>();
  if (nv <= 128) return f.template operator()<16, 8>();
  if (nv <= 256) return f.template operator()<32, 8>();
  set_error("rank too large for the TTTP kernel (%d vectors per row)", nv);
  return CPFIT_EINVAL;
}

template <int KVT, typename F>
static int mttkrp_tiling_dispatch(int nv, F &&f) {
  if constexpr (KVT == 2) {
    if (nv <= 1) return f.template operator()<1, 1>();
    if (nv <= 2) return f.template operator()<1, 2>();
    if (nv <= 4) return f.template operator()<2, 2>();
    if (nv <= 8) return f.template operator()<4, 2>();
    if (nv <= 16) return f.template operator()<8, 2>();
    if (nv <= 32) return f.template operator()<16, 2>();
  } else {
    if (nv <= 1) return f.template operator()<1, 1>();
    if (nv <= 2) return f.template operator()<2, 1>();
    if (nv <= 4) return f.template operator()<4, 1>();
    if (nv <= 8) return f.template operator()<8, 1>();
    if (nv <= 16) return f.template operator()<16, 1>();
    if (nv <= 32) return f.template operator()<32, 1>();
  }
  if (nv <= 64) return f.template operator()<32, 2>();
  if (nv <= 128) return f.template operator()<32, 4>();
  if (nv <= 256) return f.template operator()<32, 8>();
  set_error("rank too large for the MTTKRP kernel (%d vectors per row)", nv);
  return CPFIT_EINVAL;
}

template <typename T>
int dispatch_tttp(const TttpParams<T> &p, int vec, cudaStream_t s) {
  const int nv = (p.rank + vec - 1) / vec;
  if constexpr (sizeof(T) == 8) {
    if (vec == 2)
      return tttp_tiling_dispatch(nv, [&]<int L, int K>() { return launch_tttp_np<T, 2, L, K>(p, s); });
    return tttp_tiling_dispatch(nv, [&]<int L, int K>() { return launch_tttp_np<T, 1, L, K>(p, s); });
  } else {
    if (vec == 4)
      return tttp_tiling_dispatch(nv, [&]<int L, int K>() { return launch_tttp_np<T, 4, L, K>(p, s); });
    if (vec == 2)
      return tttp_tiling_dispatch(nv, [&]<int L, int K>() { return launch_tttp_np<T, 2, L, K>(p, s); });
    return tttp_tiling_dispatch(nv, [&]<int L, int K>() { return launch_tttp_np<T, 1, L, K>(p, s); });
  }
}

template <typename T>
int dispatch_mttkrp(const MttkrpParams<T> &p, int vec, cudaStream_t s) {
  const int nv = (p.rank + vec - 1) / vec;
  constexpr int KVT = sizeof(T) == 8 ? CPFIT_MTTKRP_KVT64 : 1;
  if constexpr (sizeof(T) == 8) {
    if (vec == 2)
      return mttkrp_tiling_dispatch<KVT>(nv, [&]<int L, int K>() { return launch_mttkrp_np<T, 2, L, K>(p, s); });
    return mttkrp_tiling_dispatch<KVT>(nv, [&]<int L, int K>() { return launch_mttkrp_np<T, 1, L, K>(p, s); });
  } else {
    if (vec == 4)
      return mttkrp_tiling_dispatch<KVT>(nv, [&]<int L, int K>() { return launch_mttkrp_np<T, 4, L, K>(p, s); });
    if (vec == 2)
      return mttkrp_tiling_dispatch<KVT>(nv, [&]<int L, int K>() { return launch_mttkrp_np<T, 2, L, K>(p, s); });
    return mttkrp_tiling_dispatch<KVT>(nv, [&]<int L, int K>() { return launch_mttkrp_np<T, 1, L, K>(p, s); });
  }
}

// Gram-free matvec variants (instantiated in gram_matvec_f64.cu / _f32.cu)
template <typename T>
int dispatch_mttkrp_mv(const MttkrpParams<T> &p, int vec, cudaStream_t s) {
  const int nv = (p.rank + vec - 1) / vec;
  constexpr int KVT = sizeof(T) == 8 ? CPFIT_MTTKRP_KVT64 : 1;
  if constexpr (sizeof(T) == 8) {
    if (vec == 2)
      return mttkrp_tiling_dispatch<KVT>(nv, [&]<int L, int K>() { return launch_mttkrp_np<T, 2, L, K, true>(p, s); });
    return mttkrp_tiling_dispatch<KVT>(nv, [&]<int L, int K>() { return launch_mttkrp_np<T, 1, L, K, true>(p, s); });
  } else {
    if (vec == 4)
      return mttkrp_tiling_dispatch<KVT>(nv, [&]<int L, int K>() { return launch_mttkrp_np<T, 4, L, K, true>(p, s); });
    if (vec == 2)
      return mttkrp_tiling_dispatch<KVT>(nv, [&]<int L, int K>() { return launch_mttkrp_np<T, 2, L, K, true>(p, s); });
    return mttkrp_tiling_dispatch<KVT>(nv, [&]<int L, int K>() { return launch_mttkrp_np<T, 1, L, K, true>(p, s); });
  }
}

template <typename T>
int dispatch_tttp(const TttpParams<T> &p, int vec, cudaStream_t s);
template <typename T>
int dispatch_mttkrp(const MttkrpParams<T> &p, int vec, cudaStream_t s);
template <typename T>
int dispatch_mttkrp_mv(const MttkrpParams<T> &p, int vec, cudaStream_t s);

}  // namespace cpfit
