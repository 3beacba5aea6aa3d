// gram_solve.cu -- per-row normal-equation blocks (Gram) and the batched
// small-SPD solve of ALS completion, for sm_100a.
//
// Gram: G_i = sum_{e in row i} (sqrt(w_e) h_e)(sqrt(w_e) h_e)^T with
// h_e = prod_{k != mode} A_k[i_k(e), :] -- exactly the reference's staged
// rank-k update (kernels.py:195-205).  One warp per mode-sorted task stages
// 32 Hadamard rows at a time in shared memory (lane groups gather the factor
// rows with vector loads, several nonzeros per warp instruction, loads for
// U slots issued before use) and accumulates G with FP64 tensor-core MMAs
// (mma.sync m8n8k4 f64 -> DMMA; tcgen05 has no f64 kind), computing only the
// upper-triangular 8x8 tiles (G is symmetric) and mirroring on store.  Long
// rows are split into tasks whose partial Grams are summed in task order
// (deterministic; no floating-point atomics).
//
// Solve: for R <= 32 one warp per row keeps G + reg I in registers (lane j
// owns column j) and runs a right-looking Cholesky whose column broadcasts
// (warp-uniform shared-memory loads, one __syncwarp per step) also drive the
// forward substitution, then back-substitutes with one shuffle per step.  Rows whose Cholesky
// meets a non-positive pivot (and every row when R > 32) go through a
// shared-memory kernel with a partial-pivoting LU fallback that reports
// "singular" exactly when LAPACK gesv (np.linalg.solve, kernels.py:259)
// would: on an exact zero pivot.  Empty rows follow kernels.py:245-257
// (x = rhs/reg, or identity when reg == 0 with an error for a nonzero rhs).
// The first offending row is found with an integer atomicMin.
#include <cfloat>

#include "common.cuh"

namespace cpfit {

__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

template <typename T>
struct GramParams {
  int np;
  int rank;
  const int32_t *idx[CPFIT_MAXN];  // mode-sorted coordinates of the other modes
  const T *fac[CPFIT_MAXN];
  const T *weights;       // nullable (unit weights)
  const int32_t *wperm;   // non-null: weights in canonical order, gather by perm
  const int64_t *task_begin;
  const int32_t *task_row;
  const int32_t *task_slot;
  int64_t ntasks;
  T *gram;      // dims[mode] x R x R
  T *partial;   // nslots x pstride (R x R, then R rhs values when vals != null)
  int64_t pstride;
  // fused right-hand side (ALS): rhs_i = sum_{e in row i} vals_e h_e, i.e. the
  // MTTKRP of the data computed from the same staged Hadamard rows
  const T *vals;          // nullable: no rhs
  const int32_t *vperm;   // non-null: vals in canonical order, gather by perm
  T *rhs;                 // dims[mode] x R
  const double *sqrt_w;   // fragment kernel: sqrt(weights) in sorted order (nullable)
};

constexpr int GRAM_WARPS = 4;
constexpr int GRAM_CHUNK = 32;  // Hadamard rows staged per MMA sweep

template <int RT>
constexpr int gram_ld() {
  // +4 doubles: consecutive rows 32 B (8 banks) apart, so the four rows an
  // MMA operand load touches per half-warp (lane = 4 gq + tq reads row tq,
  // column gq) land on disjoint banks (+8 gave 2-way conflicts)
  return RT * 8 + 4;
}

constexpr int pow2_at_least(int x) {
  int p = 1;
  while (p < x && p < 32) p *= 2;
  return p;
}

template <typename T, int RT, int VEC, int NPT>
__global__ void __launch_bounds__(GRAM_WARPS * 32)
gram_kernel(const GramParams<T> p) {
  constexpr int RP = RT * 8;
  constexpr int LD = gram_ld<RT>();
  constexpr int NT = RT * (RT + 1) / 2;           // upper-triangular tiles
  constexpr int NV = RP / VEC;                    // vectors per padded row
  constexpr int LPE = pow2_at_least(NV);          // lanes per staged entry
  constexpr int KV = (NV + LPE - 1) / LPE;
  constexpr int G = 32 / LPE;                     // entries per warp instruction
  constexpr int U = LPE < 4 ? LPE : 4;            // sub-iterations batched
  constexpr int NPM = NPT > 0 ? NPT : CPFIT_MAXN;
  extern __shared__ double gsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int g = lane / LPE, q = lane % LPE;
  double *H = gsm + (size_t)wib * GRAM_CHUNK * LD;
  const int rank = p.rank;
  const int np = NPT > 0 ? NPT : p.np;
  const int64_t warp = (int64_t)blockIdx.x * GRAM_WARPS + wib;
  const int64_t nwarps = (int64_t)gridDim.x * GRAM_WARPS;
  const int gq = lane >> 2, tq = lane & 3;

  for (int64_t t = warp; t < p.ntasks; t += nwarps) {
    const int64_t b0 = p.task_begin[t], b1 = p.task_begin[t + 1];
    double acc[NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i) acc[i][0] = acc[i][1] = 0.0;
    double racc[KV][VEC];  // rhs columns (k*LPE+q)*VEC+v over this group's slots
#pragma unroll
    for (int k = 0; k < KV; ++k)
#pragma unroll
      for (int v = 0; v < VEC; ++v) racc[k][v] = 0.0;

    for (int64_t base = b0; base < b1; base += GRAM_CHUNK) {
      const int cnt = (int)(b1 - base < GRAM_CHUNK ? b1 - base : GRAM_CHUNK);
      // coalesced index / weight loads, one entry per lane
      const int64_t e = base + lane;
      int32_t my_idx[NPM];
#pragma unroll
      for (int n = 0; n < NPM; ++n) my_idx[n] = (n < np && lane < cnt) ? __ldg(p.idx[n] + e) : 0;
      double my_sw = 0.0;  // padded slots stage zero rows
      double my_v = 0.0;
      if (lane < cnt) {
        my_sw = 1.0;
        if (p.weights) {
          T w = p.wperm ? __ldg(p.weights + __ldg(p.wperm + e)) : __ldg(p.weights + e);
          my_sw = sqrt((double)w);
        }
        if (p.vals) my_v = (double)(p.vperm ? __ldg(p.vals + __ldg(p.vperm + e)) : __ldg(p.vals + e));
      }
      // stage sqrt(w) * h rows: group g handles slot j = s*G + g
#pragma unroll
      for (int s0 = 0; s0 < LPE; s0 += U) {
        T x[U][NPM][KV][VEC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = (s0 + u) * G + g;
#pragma unroll
          for (int n = 0; n < NPM; ++n) {
            if (n >= np) break;
            const unsigned row = (unsigned)__shfl_sync(0xffffffffu, my_idx[n], j);
            const T *frow = p.fac[n] + (size_t)row * (unsigned)rank;
#pragma unroll
            for (int k = 0; k < KV; ++k) {
              const int col = (k * LPE + q) * VEC;
              if (col < rank) {
                load_vec<T, VEC>(frow + col, x[u][n][k]);
              } else {
#pragma unroll
                for (int v = 0; v < VEC; ++v) x[u][n][k][v] = T(0);
              }
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = (s0 + u) * G + g;
          const double sw = __shfl_sync(0xffffffffu, my_sw, j);
          const double tv = __shfl_sync(0xffffffffu, my_v, j);
#pragma unroll
          for (int k = 0; k < KV; ++k) {
            const int col = (k * LPE + q) * VEC;
            double h[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
              double prod = (double)x[u][0][k][v];
#pragma unroll
              for (int n = 1; n < NPM; ++n)
                if (n < np) prod *= (double)x[u][n][k][v];
              h[v] = prod * sw;
              racc[k][v] = fma(tv, prod, racc[k][v]);
            }
            if (col < RP) {
              if constexpr (VEC == 2) {
                *reinterpret_cast<double2 *>(H + j * LD + col) = make_double2(h[0], h[1]);
              } else {
                H[j * LD + col] = h[0];
              }
            }
          }
        }
      }
      __syncwarp();
      const int kend = (cnt + 3) & ~3;
      for (int kk = 0; kk < kend; kk += 4) {
        double f[RT];
#pragma unroll
        for (int i = 0; i < RT; ++i) f[i] = H[(kk + tq) * LD + 8 * i + gq];
        int tile = 0;
#pragma unroll
        for (int i = 0; i < RT; ++i)
#pragma unroll
          for (int jt = i; jt < RT; ++jt) {
            dmma_8x8x4(acc[tile][0], acc[tile][1], f[i], f[jt]);
            ++tile;
          }
      }
      __syncwarp();
    }
    // store G (tiles and their mirror images)
    const int slot = p.task_slot[t];
    T *dst = slot < 0 ? p.gram + (int64_t)p.task_row[t] * rank * rank
                      : p.partial + (int64_t)slot * p.pstride;
    if (p.vals) {
      // fold the G groups' rhs partials (fixed xor tree), group 0 stores
#pragma unroll
      for (int o = LPE; o < 32; o <<= 1)
#pragma unroll
        for (int k = 0; k < KV; ++k)
#pragma unroll
          for (int v = 0; v < VEC; ++v) racc[k][v] += __shfl_xor_sync(0xffffffffu, racc[k][v], o);
      T *rdst = slot < 0 ? p.rhs + (int64_t)p.task_row[t] * rank : dst + rank * rank;
      if (g == 0) {
#pragma unroll
        for (int k = 0; k < KV; ++k)
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const int col = (k * LPE + q) * VEC + v;
            if (col < rank) rdst[col] = (T)racc[k][v];
          }
      }
    }
    if constexpr (RP <= GRAM_CHUNK) {
      // transpose through the staging buffer, then write whole rows coalesced
      int tile = 0;
#pragma unroll
      for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int jt = i; jt < RT; ++jt) {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int r = 8 * i + gq, c = 8 * jt + 2 * tq + v;
            H[r * LD + c] = acc[tile][v];
            H[c * LD + r] = acc[tile][v];
          }
          ++tile;
        }
      __syncwarp();
      const int total = rank * rank;
      for (int k = lane; k < total; k += 32) {
        const int r = k / rank, c = k - r * rank;
        dst[k] = (T)H[r * LD + c];
      }
      __syncwarp();
    } else {
      int tile = 0;
#pragma unroll
      for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int jt = i; jt < RT; ++jt) {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int r = 8 * i + gq, c = 8 * jt + 2 * tq + v;
            if (r < rank && c < rank) {
              dst[(int64_t)r * rank + c] = (T)acc[tile][v];
              if (i != jt) dst[(int64_t)c * rank + r] = (T)acc[tile][v];
            }
          }
          ++tile;
        }
    }
  }
}

// Register-fragment Gram kernel (fp64, fixed number of other modes, R <= 32):
// no shared-memory staging.  The DMMA m8n8k4 operand of lane (gq, tq) for
// column block i and k-step kk is H[kk + tq][8 i + gq] -- one element of the
// Hadamard row of entry kk + tq -- so every lane gathers exactly the factor
// elements its own fragments need (8 lanes with the same tq read 64
// contiguous bytes of one row) and multiplies them in registers.  Stream and
// gather loads run one stage (U k-steps) ahead of the MMAs, indices two
// stages ahead, so each warp overlaps its own gather latency with its tensor
// work.  Tile set as gram_kernel (upper-triangular 8x8 tiles); the per-tile
// accumulation order over k is the same, so results agree with gram_kernel
// to rounding of the (identical) products.
// k-steps (of 4 entries) per stage and the stage schedule (1: one buffer,
// operands before the next loads; 0: the earlier ping-pong buffers).  Measured at
// cfg 3 (ALS sweep, ms): ping-pong U=2 22.96; one buffer U=2 22.44, U=3 21.02,
// U=4 (202 registers) 22.5; schedules without intra-warp overlap or with the
// index loads after the MMAs 22.3-22.6 (profiles/r2_tuning.md).
#ifndef CPFIT_GRAM_FRAG_U
#define CPFIT_GRAM_FRAG_U 3
#endif
#ifndef CPFIT_GRAM_ORDER
#define CPFIT_GRAM_ORDER 1
#endif
constexpr int GRAM_FRAG_WARPS = 4;

template <int RT, int NPT, int U>
struct GramFragStage {
  double x[U][NPT][RT];
  double sw[U], tv[U];
};

template <int RT, int NPT, int U>
__device__ __forceinline__ void gram_frag_idx(const GramParams<double> &p, int64_t kb,
                                              int64_t b1, int tq, int32_t (&ix)[U][NPT]) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t e = kb + 4 * u + tq;
#pragma unroll
    for (int n = 0; n < NPT; ++n) ix[u][n] = e < b1 ? __ldg(p.idx[n] + e) : -1;
  }
}

template <int RT, int NPT, int U>
__device__ __forceinline__ void gram_frag_load(const GramParams<double> &p, int64_t kb,
                                               int64_t b1, int gq, int tq,
                                               const int32_t (&ix)[U][NPT],
                                               GramFragStage<RT, NPT, U> &st) {
  const int rank = p.rank;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t e = kb + 4 * u + tq;
    const bool ok = e < b1;
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      const double *row = p.fac[n] + (size_t)(unsigned)(ok ? ix[u][n] : 0) * (unsigned)rank;
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int col = 8 * i + gq;
        st.x[u][n][i] = (ok && col < rank) ? __ldg(row + col) : 0.0;
      }
    }
    double sw = 0.0, tv = 0.0;
    if (ok) {
      sw = 1.0;
      if (p.sqrt_w) sw = __ldg(p.sqrt_w + e);  // sqrt(w) precomputed in sorted order
      else if (p.weights) sw = sqrt(p.wperm ? __ldg(p.weights + __ldg(p.wperm + e)) : __ldg(p.weights + e));
      if (p.vals) tv = p.vperm ? __ldg(p.vals + __ldg(p.vperm + e)) : __ldg(p.vals + e);
    }
    st.sw[u] = sw;
    st.tv[u] = tv;
  }
}

// Full-stage variants (every entry of the stage inside the task, rank == 8 RT,
// values / sqrt(w) in sorted order): no per-entry bounds or column predicates
// and no zero fills -- the generic loaders spend ~30 % of the kernel's issued
// instructions on them (ncu r2: ISETP / CS2R / UISETP / BRA, 80 of 283 per
// 8-entry stage).  Same loads, same values, same order.
template <int RT, int NPT, int U>
__device__ __forceinline__ void gram_frag_idx_full(const GramParams<double> &p, int64_t kb,
                                                   int tq, int32_t (&ix)[U][NPT]) {
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int n = 0; n < NPT; ++n) ix[u][n] = __ldg(p.idx[n] + kb + 4 * u + tq);
}

template <int RT, int NPT, int U, bool WEIGHTED, bool RHS>
__device__ __forceinline__ void gram_frag_load_full(const GramParams<double> &p, int64_t kb,
                                                    int gq, int tq, const int32_t (&ix)[U][NPT],
                                                    GramFragStage<RT, NPT, U> &st) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      const double *row = p.fac[n] + (size_t)(unsigned)ix[u][n] * (unsigned)(8 * RT) + gq;
#pragma unroll
      for (int i = 0; i < RT; ++i) st.x[u][n][i] = __ldg(row + 8 * i);
    }
    const int64_t e = kb + 4 * u + tq;
    st.sw[u] = WEIGHTED ? __ldg(p.sqrt_w + e) : 1.0;
    st.tv[u] = RHS ? __ldg(p.vals + e) : 0.0;
  }
}

template <int RT, int NPT, int U, bool FULLR = false, bool WEIGHTED = false, bool RHS = false>
__global__ void __launch_bounds__(GRAM_FRAG_WARPS * 32)
gram_frag_kernel(const GramParams<double> p) {
  constexpr int NT = RT * (RT + 1) / 2;
  constexpr int KS = 4 * U;  // entries per stage
  const int lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int rank = p.rank;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < p.ntasks; t += nwarps) {
    const int64_t b0 = p.task_begin[t], b1 = p.task_begin[t + 1];
    double acc[NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i) acc[i][0] = acc[i][1] = 0.0;
    double racc[RT];
#pragma unroll
    for (int i = 0; i < RT; ++i) racc[i] = 0.0;
    int32_t ix_next[U][NPT];
    // stage loaders: the predicate-free variants when the whole stage lies
    // inside the task (warp-uniform test), the generic ones at the tail
    auto load_idx = [&](int64_t ks, int32_t(&ix)[U][NPT]) {
      if (FULLR && ks + KS <= b1) gram_frag_idx_full<RT, NPT, U>(p, ks, tq, ix);
      else gram_frag_idx<RT, NPT, U>(p, ks, b1, tq, ix);
    };
    auto load_rows = [&](int64_t ks, const int32_t(&ix)[U][NPT], GramFragStage<RT, NPT, U> &st) {
      if (FULLR && ks + KS <= b1) gram_frag_load_full<RT, NPT, U, WEIGHTED, RHS>(p, ks, gq, tq, ix, st);
      else gram_frag_load<RT, NPT, U>(p, ks, b1, gq, tq, ix, st);
    };
    // Hadamard rows of a stage -> MMA operands f (and the fused rhs)
    auto hadamard = [&](const GramFragStage<RT, NPT, U> &st, double (&f)[U][RT]) {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < RT; ++i) {
          double prod = st.x[u][0][i];
#pragma unroll
          for (int n = 1; n < NPT; ++n) prod *= st.x[u][n][i];
          f[u][i] = prod * st.sw[u];
          racc[i] = fma(st.tv[u], prod, racc[i]);
        }
    };
    auto dmma_stage = [&](const double (&f)[U][RT], int64_t kb) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (kb + 4 * u < b1) {
          int tile = 0;
#pragma unroll
          for (int i = 0; i < RT; ++i)
#pragma unroll
            for (int jt = i; jt < RT; ++jt) {
              dmma_8x8x4(acc[tile][0], acc[tile][1], f[u][i], f[u][jt]);
              ++tile;
            }
        }
    };
#if CPFIT_GRAM_ORDER == 1
    // One stage buffer.  A stage is first consumed into its MMA operands (the
    // only wait on gathered rows, with nothing younger in flight), THEN the
    // next stage's gathers and the indices after it are issued into the same
    // registers, then the MMAs run under them.  In the ping-pong order below
    // ptxas put the freshly issued stream / gather loads on the scoreboard the
    // first Hadamard multiply waits on in one of the two loop copies (ncu:
    // 26 % of the kernel's samples on that DMUL against 3 % in the other copy).
    GramFragStage<RT, NPT, U> sa;
    {
      int32_t ix0[U][NPT];
      load_idx(b0, ix0);
      load_idx(b0 + KS, ix_next);
      load_rows(b0, ix0, sa);
    }
    for (int64_t kb = b0; kb < b1; kb += KS) {
      double f[U][RT];
      hadamard(sa, f);
      load_rows(kb + KS, ix_next, sa);
      load_idx(kb + 2 * KS, ix_next);
      dmma_stage(f, kb);
    }
#else
    // two stage buffers used alternately (no register copies between stages):
    // the next stage's gathers (indices loaded one stage earlier) and the
    // indices of the stage after it are issued before this stage's MMAs
    GramFragStage<RT, NPT, U> sa, sb;
    {
      int32_t ix0[U][NPT];
      load_idx(b0, ix0);
      load_idx(b0 + KS, ix_next);
      load_rows(b0, ix0, sa);
    }
    for (int64_t kb = b0; kb < b1;) {
      double f[U][RT];
      load_rows(kb + KS, ix_next, sb);
      load_idx(kb + 2 * KS, ix_next);
      hadamard(sa, f);
      dmma_stage(f, kb);
      kb += KS;
      if (kb >= b1) break;
      load_rows(kb + KS, ix_next, sa);
      load_idx(kb + 2 * KS, ix_next);
      hadamard(sb, f);
      dmma_stage(f, kb);
      kb += KS;
    }
#endif
    const int slot = p.task_slot[t];
    double *dst = slot < 0 ? p.gram + (int64_t)p.task_row[t] * rank * rank
                           : p.partial + (int64_t)slot * p.pstride;
    if (p.vals) {
      // entries of this task were split over tq: fixed xor tree over tq
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        racc[i] += __shfl_xor_sync(0xffffffffu, racc[i], 1);
        racc[i] += __shfl_xor_sync(0xffffffffu, racc[i], 2);
      }
      double *rdst = slot < 0 ? p.rhs + (int64_t)p.task_row[t] * rank : dst + rank * rank;
      if (tq == 0) {
#pragma unroll
        for (int i = 0; i < RT; ++i)
          if (8 * i + gq < rank) rdst[8 * i + gq] = racc[i];
      }
    }
    // accumulator fragment (tile (i, jt), element v) = G[8 i + gq][8 jt + 2 tq + v]
    int tile = 0;
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int jt = i; jt < RT; ++jt) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int r = 8 * i + gq, c = 8 * jt + 2 * tq + v;
          if (r < rank && c < rank) {
            dst[(int64_t)r * rank + c] = acc[tile][v];
            if (i != jt) dst[(int64_t)c * rank + r] = acc[tile][v];
          }
        }
        ++tile;
      }
  }
}

template <typename T>
__global__ void combine_gram_partials(const int32_t *__restrict__ split_row,
                                      const int32_t *__restrict__ split_slot, int64_t nsplit,
                                      int64_t rr, int64_t pstride,
                                      const T *__restrict__ partial, T *__restrict__ gram,
                                      T *__restrict__ rhs, int rank) {
  for (int64_t s = blockIdx.x; s < nsplit; s += gridDim.x) {
    const int64_t row = split_row[s];
    const int64_t a = split_slot[s], b = split_slot[s + 1];
    // columns are spread over gridDim.y blocks so that a long row is not one block's work
    for (int64_t c = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; c < pstride;
         c += (int64_t)gridDim.y * blockDim.x) {
      // eight interleaved running sums (slot k -> sum k mod 8), added by a fixed
      // tree: a Zipf head row has ~1000 partial blocks, and one running sum made
      // every thread wait for 1000 dependent loads (cfg 3 mode 1: 0.54 ms)
      double acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.0;
      int64_t k = a;
      for (; k + 8 <= b; k += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += (double)partial[(k + j) * pstride + c];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (k + j < b) acc[j] += (double)partial[(k + j) * pstride + c];
      const double tot = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
      if (c < rr) gram[row * rr + c] = (T)tot;
      else rhs[row * rank + (c - rr)] = (T)tot;
    }
  }
}

// zero G (and rhs) of the rows without entries: warp per row
template <typename T>
__global__ void zero_empty_rows(int64_t dim, const int64_t *__restrict__ offsets, int64_t rr,
                                T *__restrict__ gram, T *__restrict__ rhs, int rank) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < dim; i += nwarps) {
    if (offsets[i + 1] != offsets[i]) continue;
    for (int64_t c = lane; c < rr; c += 32) gram[i * rr + c] = T(0);
    if (rhs)
      for (int c = lane; c < rank; c += 32) rhs[i * rank + c] = T(0);
  }
}

// sqrt(w) of every entry in mode-sorted order (the fragment Gram kernel's
// per-entry scale; computed once instead of on the 8 lanes sharing an entry)
template <typename T>
__global__ void sqrt_weights_kernel(int64_t n, const T *__restrict__ w,
                                    const int32_t *__restrict__ wperm,
                                    double *__restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = sqrt((double)(wperm ? w[wperm[e]] : w[e]));
}

template <typename T>
__global__ void check_weights_kernel(const T *__restrict__ w, int64_t n, int *flag) {
  int bad = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    bad |= (w[k] < T(0));
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}

template <int RT, int NPT, bool FULLR, bool WEIGHTED, bool RHS>
static int launch_gram_frag_v(const GramParams<double> &p, cudaStream_t s) {
  constexpr int U = CPFIT_GRAM_FRAG_U;
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, gram_frag_kernel<RT, NPT, U, FULLR, WEIGHTED, RHS>, GRAM_FRAG_WARPS * 32, 0);
    if (per_sm < 1) per_sm = 1;
  }
  int64_t blocks = (p.ntasks + GRAM_FRAG_WARPS - 1) / GRAM_FRAG_WARPS;
  int64_t cap = (int64_t)num_sms() * per_sm;
  unsigned grid = (unsigned)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
  gram_frag_kernel<RT, NPT, U, FULLR, WEIGHTED, RHS><<<grid, GRAM_FRAG_WARPS * 32, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("gram_frag_kernel");
  return CPFIT_OK;
}

static bool gram_fast_enabled() {
  static int on = -1;
  if (on < 0) {
    const char *env = getenv("CPFIT_GRAM_FAST");
    on = env ? atoi(env) : 1;
  }
  return on != 0;
}

template <int RT, int NPT>
static int launch_gram_frag(const GramParams<double> &p, cudaStream_t s) {
  // predicate-free full stages: rank == 8 RT, values in sorted order (the ALS
  // sweep and the precomputed-sqrt(w) weighted Grams); everything else keeps
  // the generic loaders
  const bool fast = gram_fast_enabled() && p.rank == 8 * RT && !p.vperm && !p.wperm &&
                    (!p.weights || p.sqrt_w);
  if (fast) {
    const bool w = p.sqrt_w != nullptr, r = p.vals != nullptr;
    if (w && r) return launch_gram_frag_v<RT, NPT, true, true, true>(p, s);
    if (w) return launch_gram_frag_v<RT, NPT, true, true, false>(p, s);
    if (r) return launch_gram_frag_v<RT, NPT, true, false, true>(p, s);
    return launch_gram_frag_v<RT, NPT, true, false, false>(p, s);
  }
  return launch_gram_frag_v<RT, NPT, false, false, false>(p, s);
}

static bool gram_frag_enabled() {
  static int on = -1;
  if (on < 0) {
    const char *env = getenv("CPFIT_GRAM_FRAG");
    on = env ? atoi(env) : 1;
  }
  return on != 0;
}

template <typename T, int RT, int VEC, int NPT>
static int launch_gram_v(const GramParams<T> &p, cudaStream_t s) {
  if constexpr (sizeof(T) == 8 && (NPT == 2 || NPT == 3) && RT <= 4) {
    // weighted Grams (solve_factor, Gauss-Newton, generalized losses) reach
    // the fragment kernel with sqrt(w) precomputed per entry (run_gram): it
    // would otherwise recompute it on the 8 lanes sharing an entry
    if (gram_frag_enabled() && (!p.weights || p.sqrt_w))
      return launch_gram_frag<RT, NPT>(reinterpret_cast<const GramParams<double> &>(p), s);
  }
  constexpr int LD = gram_ld<RT>();
  const size_t smem = (size_t)GRAM_WARPS * GRAM_CHUNK * LD * sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gram_kernel<T, RT, VEC, NPT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  // persistent grid: exactly the resident capacity
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gram_kernel<T, RT, VEC, NPT>,
                                                  GRAM_WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
  }
  int64_t blocks = (p.ntasks + GRAM_WARPS - 1) / GRAM_WARPS;
  int64_t cap = (int64_t)num_sms() * per_sm;
  unsigned grid = (unsigned)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
  gram_kernel<T, RT, VEC, NPT><<<grid, GRAM_WARPS * 32, smem, s>>>(p);
  CPFIT_LAUNCH_CHECK("gram_kernel");
  return CPFIT_OK;
}

template <typename T, int RT>
static int launch_gram_rt(const GramParams<T> &p, cudaStream_t s) {
  bool vec2 = (p.rank % 2 == 0);
  for (int n = 0; n < p.np; ++n)
    if ((uintptr_t)p.fac[n] % (2 * sizeof(T))) vec2 = false;
  if (vec2) {
    if (p.np == 2) return launch_gram_v<T, RT, 2, 2>(p, s);
    return launch_gram_v<T, RT, 2, 0>(p, s);
  }
  if (p.np == 2) return launch_gram_v<T, RT, 1, 2>(p, s);
  return launch_gram_v<T, RT, 1, 0>(p, s);
}

template <typename T>
static int launch_gram(const GramParams<T> &p, cudaStream_t s) {
  switch ((p.rank + 7) / 8) {
    case 1: return launch_gram_rt<T, 1>(p, s);
    case 2: return launch_gram_rt<T, 2>(p, s);
    case 3: return launch_gram_rt<T, 3>(p, s);
    case 4: return launch_gram_rt<T, 4>(p, s);
    case 5: return launch_gram_rt<T, 5>(p, s);
    case 6: return launch_gram_rt<T, 6>(p, s);
    case 7: return launch_gram_rt<T, 7>(p, s);
    case 8: return launch_gram_rt<T, 8>(p, s);
  }
  set_error("rank %d > 64 is not supported by the Gram kernel", p.rank);
  return CPFIT_EINVAL;
}

// Runs the Gram assembly into `gram` (dims[mode] x R x R, zero rows for
// empty slices).  Weights: nullptr = unit mask.
template <typename T>
static int run_gram(cpfit_pattern *pt, int mode, int rank, const T *weights,
                    int weights_sorted, const void *const *factors, T *gram, cudaStream_t s,
                    const T *vals = nullptr, int vals_sorted = 0, T *rhs = nullptr) {
  const int64_t dim = pt->dims[mode];
  const int64_t rr = (int64_t)rank * rank;
  if (weights && pt->nnz > 0) {
    Scratch<int> flag(s);
    CPFIT_TRY(flag.alloc(1));
    CPFIT_CUDA(cudaMemsetAsync(flag.ptr, 0, sizeof(int), s));
    check_weights_kernel<T><<<grid_for(pt->nnz, 256, 8), 256, 0, s>>>(weights, pt->nnz, flag.ptr);
    CPFIT_LAUNCH_CHECK("check_weights");
    int h = 0;
    CPFIT_CUDA(cudaMemcpyAsync(&h, flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
    CPFIT_CUDA(cudaStreamSynchronize(s));
    if (h) {
      set_error("weights must be nonnegative for normal-equation assembly");
      return CPFIT_ENEGWEIGHT;
    }
  }
  if (pt->nnz == 0) {
    CPFIT_CUDA(cudaMemsetAsync(gram, 0, (size_t)dim * rr * sizeof(T), s));
    if (vals) CPFIT_CUDA(cudaMemsetAsync(rhs, 0, (size_t)dim * rank * sizeof(T), s));
    return CPFIT_OK;
  }
  CPFIT_TRY(ensure_coarse_layout(pt, mode, s));
  CpfitModeLayout &L = pt->coarse[mode];
  // every non-empty row is written by the Gram kernel (or its partial-slot
  // combine); only empty rows need zeros -- no full memset of dim * R^2
  zero_empty_rows<T><<<grid_for(dim * 32, 256), 256, 0, s>>>(dim, L.offsets, rr, gram,
                                                             vals ? rhs : nullptr, rank);
  CPFIT_LAUNCH_CHECK("zero_empty_rows");
  GramParams<T> p{};
  p.rank = rank;
  int np = 0;
  for (int n = 0; n < pt->order; ++n) {
    if (n == mode) continue;
    if (!factors[n]) {
      set_error("factor[%d] is required but missing", n);
      return CPFIT_EINVAL;
    }
    p.idx[np] = L.sorted_idx[n];
    p.fac[np] = (const T *)factors[n];
    ++np;
  }
  if (np == 0) {
    set_error("at least one factor matrix must be provided");
    return CPFIT_EINVAL;
  }
  p.np = np;
  p.weights = weights;
  p.wperm = (weights && !weights_sorted) ? L.perm : nullptr;
  p.task_begin = L.task_begin;
  p.task_row = L.task_row;
  p.task_slot = L.task_slot;
  p.ntasks = L.ntasks;
  p.gram = gram;
  p.vals = vals;
  p.vperm = (vals && !vals_sorted) ? L.perm : nullptr;
  p.rhs = rhs;
  p.pstride = rr + (vals ? rank : 0);
  Scratch<T> partial(s);
  if (L.nslots > 0) CPFIT_TRY(partial.alloc((size_t)L.nslots * p.pstride));
  p.partial = partial.ptr;
  Scratch<double> sqw(s);
  if (sizeof(T) == 8 && weights && np == 2 && rank <= 32 &&
      gram_frag_enabled()) {
    CPFIT_TRY(sqw.alloc(pt->nnz));
    sqrt_weights_kernel<T><<<grid_for(pt->nnz, 256, 4), 256, 0, s>>>(
        pt->nnz, weights, p.wperm, sqw.ptr);
    CPFIT_LAUNCH_CHECK("sqrt_weights");
    p.sqrt_w = sqw.ptr;
    // sqrt_w is in mode-sorted order and supersedes (weights, wperm): with the
    // permutation cleared the predicate-free full-stage kernel is eligible
    p.wperm = nullptr;
  }
  CPFIT_TRY(launch_gram<T>(p, s));
  if (L.nsplit > 0) {
    dim3 grid((unsigned)(L.nsplit < 65535 ? L.nsplit : 65535),
              (unsigned)((p.pstride + 255) / 256));
    combine_gram_partials<T><<<grid, 256, 0, s>>>(L.split_row, L.split_slot, L.nsplit, rr,
                                                  p.pstride, partial.ptr, gram, rhs, rank);
    CPFIT_LAUNCH_CHECK("combine_gram_partials");
  }
  return CPFIT_OK;
}

// ---------------------------------------------------------------------------
// batched solve

template <typename T>
struct SolveParams {
  int rank;
  int64_t dim;
  const T *gram;
  const T *rhs;
  const int64_t *offsets;
  double reg;
  T *x;
  unsigned long long *bad;  // [0] first empty row with nonzero rhs, [1] first singular row
  const int32_t *rows;      // smem kernel: explicit row list (null: rows 0..dim-1)
  int64_t nrows;
  int64_t gstride;          // elements between consecutive rows' G (0: one shared G)
  int32_t *retry;           // register kernel: rows whose Cholesky failed
  unsigned long long *nretry;
};

// Empty row (kernels.py:245-257): reg*I system (x = rhs/reg) or identity when
// reg == 0 (error for a nonzero rhs).
template <typename T>
__device__ __forceinline__ void solve_empty_row(const SolveParams<T> &p, int64_t row) {
  const int lane = threadIdx.x & 31;
  const int R = p.rank;
  bool nz = false;
  for (int i = lane; i < R; i += 32) {
    const double b = (double)p.rhs[row * R + i];
    if (p.reg == 0.0) {
      nz |= (b != 0.0);
      p.x[row * R + i] = (T)b;
    } else {
      p.x[row * R + i] = (T)(b / p.reg);
    }
  }
  if (__any_sync(0xffffffffu, nz) && lane == 0) atomicMin(&p.bad[0], (unsigned long long)row);
}

// Column broadcast through shared memory (1) or shuffles (0); measured at
// cfg 3 mode 0 (480k systems, R = 32): shuffles 2.79 ms (96 registers), smem
// 2.73 ms (132 registers), smem held to 96 registers (5 blocks/SM, a few
// spilled values) 2.47 ms -- profiles/r1_tuning.md.
#ifndef CPFIT_CHOL_SMEM
#define CPFIT_CHOL_SMEM 1
#endif
#ifndef CPFIT_SOLVE_MINB
#define CPFIT_SOLVE_MINB 5
#endif
// Register-resident warp Cholesky solve for R <= RMAX <= 32.  Lane j holds
// column j of (G + reg I) in a[] (G is symmetric: column j is loaded as row
// entries G[i][j] -- coalesced across lanes) and b_j of the right-hand side
// (then y_j, then x_j).  Step k broadcasts the UNSCALED column k (one shuffle
// per element); the scaling by 1/L[k][k] is folded into the per-lane scalar
// s_j = A[j][k] / d of the trailing update, so each element costs two
// shuffles and one FMA.  Column j stays unscaled on lane j, and lane j's own
// a[k] is A[j][k] -- row j of L times L[k][k] -- so the forward and back
// substitutions need one broadcast and one FMA per step:
//   y_k = b_k / L_kk,  b_j -= (A[j][k] / L_kk) y_k            (j > k)
//   x_k = z_k / L_kk,  z_j -= (A[k][j] / L_jj) x_k            (j < k)
// Registers: the column (2 R) and a handful of scalars.
template <typename T, int RMAX>
__device__ __forceinline__ void chol_factor_solve(const T *__restrict__ Gr,
                                                  const T *__restrict__ rh, int R, double reg,
                                                  double &mine_out, bool &ok_out) {
  // The R x R system is embedded in an RMAX x RMAX one padded with the
  // identity (block diagonal: same solution), so every loop below is
  // guard-free and every shuffle is warp-uniform.
  const int lane = threadIdx.x & 31;
  double a[RMAX];
#pragma unroll
  for (int i = 0; i < RMAX; ++i) {
    const bool in = i < R && lane < R;
    a[i] = in ? (double)__ldg(Gr + i * R + lane) + (i == lane ? reg : 0.0)
              : (i == lane ? 1.0 : 0.0);
  }
  double bj = lane < R ? (double)__ldg(rh + lane) : 0.0;
  bool ok = true;
  double my_inv = 1.0;  // 1 / L[lane][lane]
#if CPFIT_CHOL_SMEM
  // Step k needs A[i][k] (i > k) on every lane; by symmetry of the Schur
  // complement that is lane i's own a[k]: every lane stores one value and
  // the column is read back as warp-uniform (broadcast) LDS.128 pairs
  // instead of two SHFL per element.  Buffers alternate by k parity.
  __shared__ __align__(16) double col_buf[4][2][32];
  __shared__ double rhs_buf[4][2];
  double(&cb)[2][32] = col_buf[(threadIdx.x >> 5) & 3];
  double(&rb)[2] = rhs_buf[(threadIdx.x >> 5) & 3];
#endif
#pragma unroll
  for (int k = 0; k < RMAX; ++k) {
#if CPFIT_CHOL_SMEM
    double *c = cb[k & 1];
    c[lane] = a[k];
    if (lane == k) rb[k & 1] = bj;
    __syncwarp();
    const double d = c[k];
#else
    const double d = __shfl_sync(0xffffffffu, a[k], k);
#endif
    ok = ok && (d > 0.0) && (d < DBL_MAX);
    const double inv = rsqrt(d);  // MUFU.RSQ64H + Newton: ~1 ulp, no sqrt/div slow paths on the chain
#if CPFIT_CHOL_SMEM
    const double yk = rb[k & 1] * inv;
#else
    const double yk = __shfl_sync(0xffffffffu, bj, k) * inv;
#endif
    const bool right = lane > k;
    const double ljk = a[k] * inv;                      // L[j][k] on lanes j > k
    const double sj = right ? ljk * inv : 0.0;          // A[j][k] / d
    bj = right ? fma(-ljk, yk, bj) : (lane == k ? yk : bj);
    if (lane == k) my_inv = inv;
#pragma unroll
    for (int i = k + 1; i < RMAX; ++i) {
#if CPFIT_CHOL_SMEM
      const double ci = c[i];  // A[k][i] = A[i][k] (unscaled)
#else
      const double ci = __shfl_sync(0xffffffffu, a[i], k);  // A[i][k] (unscaled)
#endif
      a[i] = fma(-ci, sj, a[i]);  // trailing update of column lane
    }
  }
  // back substitution L^T x = y (garbage when !ok, not stored)
#pragma unroll
  for (int kk = 0; kk < RMAX; ++kk) {
    const int k = RMAX - 1 - kk;
    const double xk = __shfl_sync(0xffffffffu, bj * my_inv, k);
    if (lane == k) bj = xk;
    if (lane < k) bj = fma(-(a[k] * my_inv), xk, bj);
  }
  mine_out = bj;
  ok_out = __all_sync(0xffffffffu, ok);
}

// One warp per row and no grid-stride loop (inside a loop ptxas keeps the
// fully unrolled register arrays on the stack); the Cholesky runs
// unconditionally so its shuffles sit in convergent code (no divergence
// fallback paths), results are used only for active, non-empty rows.
template <typename T, int RMAX>
__device__ __forceinline__ void chol_factor_solve(const T *__restrict__ Gr,
                                                  const T *__restrict__ rh, int R, double reg,
                                                  double &mine, bool &ok);

template <typename T, int RMAX>
__global__ void __launch_bounds__(128, CPFIT_SOLVE_MINB) solve_reg_kernel(const SolveParams<T> p) {
  const int lane = threadIdx.x & 31;
  const int R = p.rank;
  const int64_t wrow = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const bool active = wrow < p.dim;
  const int64_t row = active ? wrow : p.dim - 1;
  const bool empty = p.offsets ? p.offsets[row + 1] == p.offsets[row] : false;
  double mine;
  bool ok;
  chol_factor_solve<T, RMAX>(p.gram + row * p.gstride, p.rhs + row * (int64_t)R, R, p.reg,
                             mine, ok);
  if (!active) return;
  if (empty) {
    solve_empty_row(p, row);
  } else if (ok) {
    if (lane < R) p.x[row * (int64_t)R + lane] = (T)mine;
  } else if (lane == 0) {
    const unsigned long long slot = atomicAdd(p.nretry, 1ull);
    p.retry[slot] = (int32_t)row;
  }
}

// Partial-pivot LU of the R x R system in smem (row-major, leading dim ld),
// right-hand side b[] distributed (element i held by lane i % 32, slot i / 32).
// Returns false on an exact zero pivot (LAPACK dgetrf info > 0).
template <int KB>
__device__ bool warp_lu_solve(double *A, int ld, int R, double (&b)[KB]) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < R; ++k) {
    // pivot: max |A[i][k]|, lowest index on ties (idamax)
    double best = -1.0;
    int bi = R;
    for (int i = k + lane; i < R; i += 32) {
      double v = fabs(A[i * ld + k]);
      if (v > best) { best = v; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const int piv = bi < R ? bi : k;  // all-NaN column: keep k, as idamax would
    if (A[piv * ld + k] == 0.0) return false;
    if (piv != k) {
      for (int j = lane; j < R; j += 32) {
        double t = A[k * ld + j];
        A[k * ld + j] = A[piv * ld + j];
        A[piv * ld + j] = t;
      }
      // swap b[k] and b[piv]
      double bk = 0.0, bp = 0.0;
#pragma unroll
      for (int s = 0; s < KB; ++s) {
        bk = (k / 32 == s) ? __shfl_sync(0xffffffffu, b[s], k % 32) : bk;
        bp = (piv / 32 == s) ? __shfl_sync(0xffffffffu, b[s], piv % 32) : bp;
      }
#pragma unroll
      for (int s = 0; s < KB; ++s) {
        if (s * 32 + lane == k) b[s] = bp;
        if (s * 32 + lane == piv) b[s] = bk;
      }
    }
    __syncwarp();
    const double akk = A[k * ld + k];
    double bk = 0.0;
#pragma unroll
    for (int s = 0; s < KB; ++s)
      bk = (k / 32 == s) ? __shfl_sync(0xffffffffu, b[s], k % 32) : bk;
    // multipliers and rhs update
#pragma unroll
    for (int s = 0; s < KB; ++s) {
      int i = s * 32 + lane;
      if (i > k && i < R) {
        double l = A[i * ld + k] / akk;
        A[i * ld + k] = l;
        b[s] -= l * bk;
      }
    }
    __syncwarp();
    const int n = R - k - 1;
    for (int q = lane; q < n * n; q += 32) {
      int i = k + 1 + q / n, j = k + 1 + q % n;
      A[i * ld + j] -= A[i * ld + k] * A[k * ld + j];
    }
    __syncwarp();
  }
  // back substitution U x = b
  for (int k = R - 1; k >= 0; --k) {
    double bk = 0.0;
#pragma unroll
    for (int s = 0; s < KB; ++s)
      bk = (k / 32 == s) ? __shfl_sync(0xffffffffu, b[s], k % 32) : bk;
    const double xk = bk / A[k * ld + k];
#pragma unroll
    for (int s = 0; s < KB; ++s) {
      int i = s * 32 + lane;
      if (i == k) b[s] = xk;
      else if (i < k) b[s] -= A[i * ld + k] * xk;
    }
  }
  return true;
}

template <typename T, int KB>
__global__ void solve_kernel(const SolveParams<T> p, int warps_per_block) {
  extern __shared__ double ssm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int R = p.rank, ld = R + 1;
  double *A = ssm + (size_t)wib * R * ld;
  const int64_t warp = (int64_t)blockIdx.x * warps_per_block + wib;
  const int64_t nwarps = (int64_t)gridDim.x * warps_per_block;

  const int64_t nrows = p.rows ? p.nrows : p.dim;
  for (int64_t it = warp; it < nrows; it += nwarps) {
    const int64_t row = p.rows ? (int64_t)p.rows[it] : it;
    const bool empty = p.offsets ? p.offsets[row + 1] == p.offsets[row] : false;
    const T *rhs = p.rhs + row * R;
    T *xo = p.x + row * R;
    double b[KB];
#pragma unroll
    for (int s = 0; s < KB; ++s) {
      int i = s * 32 + lane;
      b[s] = i < R ? (double)rhs[i] : 0.0;
    }
    if (empty) {
      // kernels.py:245-257: reg*I system (x = rhs/reg) or identity when reg == 0
      bool nz = false;
#pragma unroll
      for (int s = 0; s < KB; ++s) {
        int i = s * 32 + lane;
        if (i < R) {
          if (p.reg == 0.0) {
            nz |= (b[s] != 0.0);
            xo[i] = (T)b[s];
          } else {
            xo[i] = (T)(b[s] / p.reg);
          }
        }
      }
      if (__any_sync(0xffffffffu, nz) && lane == 0) atomicMin(&p.bad[0], (unsigned long long)row);
      continue;
    }
    const T *G = p.gram + row * p.gstride;
    for (int q = lane; q < R * R; q += 32) {
      int i = q / R, j = q % R;
      A[i * ld + j] = (double)G[q] + (i == j ? p.reg : 0.0);
    }
    __syncwarp();
    // Cholesky (lower, in place)
    bool ok = true;
    for (int k = 0; k < R; ++k) {
      const double d = A[k * ld + k];
      if (!(d > 0.0) || !(d < DBL_MAX)) { ok = false; break; }
      const double l = sqrt(d);
      __syncwarp();
      for (int i = k + 1 + lane; i < R; i += 32) A[i * ld + k] /= l;
      if (lane == 0) A[k * ld + k] = l;
      __syncwarp();
      const int n = R - k - 1;
      for (int q = lane; q < n * n; q += 32) {
        int i = k + 1 + q / n, j = k + 1 + q % n;
        if (j <= i) A[i * ld + j] -= A[i * ld + k] * A[j * ld + k];
      }
      __syncwarp();
    }
    if (ok) {
      // forward L y = b
      for (int k = 0; k < R; ++k) {
        double bk = 0.0;
#pragma unroll
        for (int s = 0; s < KB; ++s)
          bk = (k / 32 == s) ? __shfl_sync(0xffffffffu, b[s], k % 32) : bk;
        const double yk = bk / A[k * ld + k];
#pragma unroll
        for (int s = 0; s < KB; ++s) {
          int i = s * 32 + lane;
          if (i == k) b[s] = yk;
          else if (i > k && i < R) b[s] -= A[i * ld + k] * yk;
        }
      }
      // backward L^T x = y
      for (int k = R - 1; k >= 0; --k) {
        double bk = 0.0;
#pragma unroll
        for (int s = 0; s < KB; ++s)
          bk = (k / 32 == s) ? __shfl_sync(0xffffffffu, b[s], k % 32) : bk;
        const double xk = bk / A[k * ld + k];
#pragma unroll
        for (int s = 0; s < KB; ++s) {
          int i = s * 32 + lane;
          if (i == k) b[s] = xk;
          else if (i < k) b[s] -= A[k * ld + i] * xk;
        }
      }
    } else {
      // not numerically positive definite: LU with partial pivoting decides
      __syncwarp();
      for (int q = lane; q < R * R; q += 32) {
        int i = q / R, j = q % R;
        A[i * ld + j] = (double)G[q] + (i == j ? p.reg : 0.0);
      }
#pragma unroll
      for (int s = 0; s < KB; ++s) {
        int i = s * 32 + lane;
        b[s] = i < R ? (double)rhs[i] : 0.0;
      }
      __syncwarp();
      if (!warp_lu_solve<KB>(A, ld, R, b)) {
        if (lane == 0) atomicMin(&p.bad[1], (unsigned long long)row);
      }
    }
#pragma unroll
    for (int s = 0; s < KB; ++s) {
      int i = s * 32 + lane;
      if (i < R) xo[i] = (T)b[s];
    }
    __syncwarp();
  }
}

template <typename T>
static int launch_solve_smem(const SolveParams<T> &p, int rank, int64_t nrows, cudaStream_t s) {
  const size_t per_warp = (size_t)rank * (rank + 1) * sizeof(double);
  int wpb = (int)(49152 / per_warp);
  if (wpb > 8) wpb = 8;
  if (wpb < 1) wpb = 1;
  const size_t smem = per_warp * wpb;
  int64_t blocks = (nrows + wpb - 1) / wpb;
  int64_t cap = (int64_t)num_sms() * 16;
  unsigned grid = (unsigned)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
  const int kb = (rank + 31) / 32;
#define CPFIT_SOLVE_CASE(K)                                                              \
  case K: {                                                                              \
    cudaFuncSetAttribute(solve_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)smem);                                                     \
    solve_kernel<T, K><<<grid, wpb * 32, smem, s>>>(p, wpb);                             \
    break;                                                                               \
  }
  switch (kb) {
    CPFIT_SOLVE_CASE(1)
    CPFIT_SOLVE_CASE(2)
    CPFIT_SOLVE_CASE(3)
    CPFIT_SOLVE_CASE(4)
    default:
      set_error("rank %d > 128 is not supported by the solve kernel", rank);
      return CPFIT_EINVAL;
  }
#undef CPFIT_SOLVE_CASE
  CPFIT_LAUNCH_CHECK("solve_kernel");
  return CPFIT_OK;
}

// ---- one shared SPD matrix for every row (dense CP-ALS: G = Hadamard of the
// other factors' Gramians, every entry observed) --------------------------------
// (G + reg I)^-1 once: right-looking Cholesky in shared memory by one CTA, then
// thread j solves L L^T x = e_j in place in column j of Ainv.  *bad = 1 when a
// pivot is not positive (the caller then takes the per-row path, whose
// LU fallback carries the reference's singular-row semantics).
template <typename T>
__global__ void shared_spd_inverse(int R, const T *__restrict__ G, double reg,
                                   double *__restrict__ Ainv, int *__restrict__ bad) {
  extern __shared__ double Ls[];
  __shared__ int fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < R * R; e += nt) {
    const int i = e / R, j = e % R;
    Ls[e] = (double)G[e] + (i == j ? reg : 0.0);
  }
  if (tid == 0) fail = 0;
  __syncthreads();
  for (int k = 0; k < R; ++k) {
    if (tid == 0) {
      const double d = Ls[k * R + k];
      if (!(d > 0.0) || !isfinite(d)) fail = 1;
      else Ls[k * R + k] = sqrt(d);
    }
    __syncthreads();
    if (fail) break;
    const double piv = Ls[k * R + k];
    for (int i = k + 1 + tid; i < R; i += nt) Ls[i * R + k] /= piv;
    __syncthreads();
    const int w = R - k - 1;
    for (int e = tid; e < w * w; e += nt) {
      const int i = k + 1 + e / w, j = k + 1 + e % w;
      if (j <= i) Ls[i * R + j] -= Ls[i * R + k] * Ls[j * R + k];
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) *bad = 1;
    return;
  }
  double *Y = Ls + R * R;  // column j of the inverse, solved in shared memory by thread j
  for (int j = tid; j < R; j += nt) {
    for (int i = 0; i < R; ++i) {  // L y = e_j
      double acc = (i == j) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) acc -= Ls[i * R + k] * Y[k * R + j];
      Y[i * R + j] = acc / Ls[i * R + i];
    }
    for (int i = R - 1; i >= 0; --i) {  // L^T x = y, in place
      double acc = Y[i * R + j];
      for (int k = i + 1; k < R; ++k) acc -= Ls[k * R + i] * Y[k * R + j];
      Y[i * R + j] = acc / Ls[i * R + i];
    }
  }
  __syncthreads();
  for (int e = tid; e < R * R; e += nt) Ainv[e] = Y[e];
}

// x[i, r] = sum_k rhs[i, k] Ainv[k, r]
template <typename T>
__global__ void shared_spd_apply(int64_t n, int R, const T *__restrict__ rhs,
                                 const double *__restrict__ Ainv, T *__restrict__ x) {
  const int64_t total = n * R;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = o / R;
    const int r = (int)(o - i * R);
    const T *b = rhs + i * R;
    double acc = 0.0;
    for (int k = 0; k < R; ++k) acc += (double)b[k] * Ainv[k * R + r];
    x[o] = (T)acc;
  }
}

// returns 1 when the shared path solved everything, 0 to fall back
template <typename T>
static int solve_shared_spd(int64_t n, int R, const T *gram, const T *rhs, double reg, T *x,
                            cudaStream_t s, int *status) {
  *status = CPFIT_OK;
  if (R > 112 || n < 2) return 0;  // L and the inverse both live in shared memory
  const size_t shm = 2 * (size_t)R * R * sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(shared_spd_inverse<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * 112 * 112 * (int)sizeof(double));
    configured = true;
  }
  Scratch<double> inv(s);
  Scratch<int> bad(s);
  if ((*status = inv.alloc((size_t)R * R)) != CPFIT_OK) return 1;
  if ((*status = bad.alloc(1)) != CPFIT_OK) return 1;
  cudaMemsetAsync(bad.ptr, 0, sizeof(int), s);
  const int threads = R * R >= 256 ? 256 : 64;
  shared_spd_inverse<T><<<1, threads, shm, s>>>(R, gram, reg, inv.ptr, bad.ptr);
  int h = 0;
  cudaMemcpyAsync(&h, bad.ptr, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    *status = cuda_status(e, "shared_spd_inverse");
    return 1;
  }
  if (h) return 0;
  shared_spd_apply<T><<<grid_for(n * R, 256), 256, 0, s>>>(n, R, rhs, inv.ptr, x);
  e = cudaGetLastError();
  if (e != cudaSuccess) *status = cuda_status(e, "shared_spd_apply");
  return 1;
}

template <typename T>
static int run_solve_rows(int mode, int64_t dim, const int64_t *offsets, int rank, const T *gram,
                          int64_t gstride, const T *rhs, double reg, T *x, int64_t *bad_row,
                          cudaStream_t s) {
  Scratch<unsigned long long> bad(s);
  CPFIT_TRY(bad.alloc(3));
  CPFIT_CUDA(cudaMemsetAsync(bad.ptr, 0xff, 2 * sizeof(unsigned long long), s));
  CPFIT_CUDA(cudaMemsetAsync(bad.ptr + 2, 0, sizeof(unsigned long long), s));
  SolveParams<T> p{};
  p.rank = rank;
  p.dim = dim;
  p.gram = gram;
  p.rhs = rhs;
  p.offsets = offsets;
  p.gstride = gstride;
  p.reg = reg;
  p.x = x;
  p.bad = bad.ptr;
  Scratch<int32_t> retry(s);
  unsigned long long h[3] = {~0ull, ~0ull, 0};
  if (rank <= 32) {
    CPFIT_TRY(retry.alloc(dim > 0 ? dim : 1));
    p.retry = retry.ptr;
    p.nretry = bad.ptr + 2;
    const unsigned grid = (unsigned)((dim + 3) / 4 > 0 ? (dim + 3) / 4 : 1);
    if (rank <= 8)
      solve_reg_kernel<T, 8><<<grid, 128, 0, s>>>(p);
    else if (rank <= 16)
      solve_reg_kernel<T, 16><<<grid, 128, 0, s>>>(p);
    else
      solve_reg_kernel<T, 32><<<grid, 128, 0, s>>>(p);
    CPFIT_LAUNCH_CHECK("solve_reg_kernel");
    CPFIT_CUDA(cudaMemcpyAsync(h, bad.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
    CPFIT_CUDA(cudaStreamSynchronize(s));
    if (h[2] > 0) {  // rows that are not numerically SPD: Cholesky/LU smem path
      p.rows = retry.ptr;
      p.nrows = (int64_t)h[2];
      CPFIT_TRY(launch_solve_smem<T>(p, rank, p.nrows, s));
    }
  } else {
    CPFIT_TRY(launch_solve_smem<T>(p, rank, dim, s));
  }
  if (rank > 32 || h[2] > 0) {
    CPFIT_CUDA(cudaMemcpyAsync(h, bad.ptr, 2 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s));
    CPFIT_CUDA(cudaStreamSynchronize(s));
  }
  if (h[0] != ~0ull) {
    *bad_row = (int64_t)h[0];
    set_error("mode %d row %lld: no incident entries and reg=0 but right-hand side is nonzero",
              mode, (long long)h[0]);
    return CPFIT_EEMPTYROW;
  }
  if (h[1] != ~0ull) {
    *bad_row = (int64_t)h[1];
    set_error("mode %d row %lld: singular normal equations (reg=%g)", mode, (long long)h[1],
              reg);
    return CPFIT_ESINGULAR;
  }
  return CPFIT_OK;
}

template <typename T>
static int run_solve(cpfit_pattern *pt, int mode, int rank, const T *gram, const T *rhs,
                     double reg, T *x, int64_t *bad_row, cudaStream_t s) {
  return run_solve_rows<T>(mode, pt->dims[mode], pt->modes[mode].offsets, rank, gram,
                           (int64_t)rank * rank, rhs, reg, x, bad_row, s);
}

template <typename T>
static int run_solve_factor(cpfit_pattern *pt, int mode, int rank, const void *weights,
                            int weights_sorted, const void *const *factors, const void *rhs,
                            double reg, void *x_out, void *gram_out, int64_t *bad_row,
                            cudaStream_t s) {
  const int64_t dim = pt->dims[mode];
  Scratch<T> gtmp(s);
  T *gram = (T *)gram_out;
  if (!gram) {
    CPFIT_TRY(gtmp.alloc((size_t)dim * rank * rank));
    gram = gtmp.ptr;
  }
  // Gram first, then the regularisation check: the reference's error order
  // (kernels.py:235-243)
  CPFIT_TRY(run_gram<T>(pt, mode, rank, (const T *)weights, weights_sorted, factors, gram, s));
  if (reg < 0.0) {
    set_error("regularization must be >= 0");
    return CPFIT_EINVAL;
  }
  CPFIT_TRY(ensure_layout(pt, mode, s));
  int64_t dummy = -1;
  return run_solve<T>(pt, mode, rank, gram, (const T *)rhs, reg, (T *)x_out,
                      bad_row ? bad_row : &dummy, s);
}

// One ALS mode update (optim.py:214-228 with kernels.py:222-265): the
// right-hand side (MTTKRP of the data) is accumulated by the Gram kernel from
// the same staged Hadamard rows, so the factor rows are gathered once.
template <typename T>
static int run_als_update(cpfit_pattern *pt, int mode, int rank, const void *vals,
                          int vals_sorted, const void *const *factors, double reg, void *x_out,
                          void *gram_out, void *rhs_out, int64_t *bad_row, cudaStream_t s) {
  const int64_t dim = pt->dims[mode];
  Scratch<T> gtmp(s), rtmp(s);
  T *gram = (T *)gram_out, *rhs = (T *)rhs_out;
  if (!gram) {
    CPFIT_TRY(gtmp.alloc((size_t)dim * rank * rank));
    gram = gtmp.ptr;
  }
  if (!rhs) {
    CPFIT_TRY(rtmp.alloc((size_t)dim * rank));
    rhs = rtmp.ptr;
  }
  CPFIT_TRY(run_gram<T>(pt, mode, rank, nullptr, 0, factors, gram, s, (const T *)vals,
                        vals_sorted, rhs));
  if (reg < 0.0) {
    set_error("regularization must be >= 0");
    return CPFIT_EINVAL;
  }
  CPFIT_TRY(ensure_layout(pt, mode, s));
  int64_t dummy = -1;
  return run_solve<T>(pt, mode, rank, gram, rhs, reg, (T *)x_out, bad_row ? bad_row : &dummy, s);
}

}  // namespace cpfit

using namespace cpfit;

extern "C" {

int cpfit_gram(cpfit_pattern *p, int mode, int dtype, int rank, const void *weights,
               int weights_sorted, const void *const *factors, void *gram_out, void *stream) {
  if (!p || mode < 0 || mode >= p->order) {
    set_error("mode %d out of range for order-%d tensor", mode, p ? p->order : 0);
    return CPFIT_EINVAL;
  }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    return run_gram<double>(p, mode, rank, (const double *)weights, weights_sorted, factors,
                            (double *)gram_out, s);
  if (dtype == CPFIT_F32)
    return run_gram<float>(p, mode, rank, (const float *)weights, weights_sorted, factors,
                           (float *)gram_out, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_solve_rows(int dtype, int rank, int64_t nrows, const void *gram, int64_t gram_stride,
                     const void *rhs, double reg, void *x_out, int64_t *bad_row, void *stream) {
  if (rank < 1 || nrows < 0 || gram_stride < 0) {
    set_error("invalid solve_rows arguments");
    return CPFIT_EINVAL;
  }
  if (reg < 0.0) {
    set_error("regularization must be >= 0");
    return CPFIT_EINVAL;
  }
  if (nrows == 0) return CPFIT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t dummy = -1;
  if (gram_stride == 0 && (dtype == CPFIT_F64 || dtype == CPFIT_F32)) {
    // one shared G: factor and invert it once (falls through when not SPD)
    int st = CPFIT_OK;
    const int done =
        dtype == CPFIT_F64
            ? solve_shared_spd<double>(nrows, rank, (const double *)gram, (const double *)rhs, reg,
                                       (double *)x_out, s, &st)
            : solve_shared_spd<float>(nrows, rank, (const float *)gram, (const float *)rhs, reg,
                                      (float *)x_out, s, &st);
    if (done) return st;
  }
  if (dtype == CPFIT_F64)
    return run_solve_rows<double>(-1, nrows, nullptr, rank, (const double *)gram, gram_stride,
                                  (const double *)rhs, reg, (double *)x_out,
                                  bad_row ? bad_row : &dummy, s);
  if (dtype == CPFIT_F32)
    return run_solve_rows<float>(-1, nrows, nullptr, rank, (const float *)gram, gram_stride,
                                 (const float *)rhs, reg, (float *)x_out,
                                 bad_row ? bad_row : &dummy, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_solve_factor(cpfit_pattern *p, int mode, int dtype, int rank, const void *weights,
                       int weights_sorted, const void *const *factors, const void *rhs,
                       double reg, void *x_out, void *gram_out, int64_t *bad_row,
                       void *stream) {
  if (!p || mode < 0 || mode >= p->order) {
    set_error("mode %d out of range for order-%d tensor", mode, p ? p->order : 0);
    return CPFIT_EINVAL;
  }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    return run_solve_factor<double>(p, mode, rank, weights, weights_sorted, factors, rhs, reg,
                                    x_out, gram_out, bad_row, s);
  if (dtype == CPFIT_F32)
    return run_solve_factor<float>(p, mode, rank, weights, weights_sorted, factors, rhs, reg,
                                   x_out, gram_out, bad_row, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_als_update(cpfit_pattern *p, int mode, int dtype, int rank, const void *vals,
                     int vals_sorted, const void *const *factors, double reg, void *x_out,
                     void *gram_out, void *rhs_out, int64_t *bad_row, void *stream) {
  if (!p || mode < 0 || mode >= p->order) {
    set_error("mode %d out of range for order-%d tensor", mode, p ? p->order : 0);
    return CPFIT_EINVAL;
  }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  if (!vals && p->nnz > 0) { set_error("values are required"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    return run_als_update<double>(p, mode, rank, vals, vals_sorted, factors, reg, x_out,
                                  gram_out, rhs_out, bad_row, s);
  if (dtype == CPFIT_F32)
    return run_als_update<float>(p, mode, rank, vals, vals_sorted, factors, reg, x_out,
                                 gram_out, rhs_out, bad_row, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

}  // extern "C"
