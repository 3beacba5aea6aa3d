// ccd.cu -- CCD++ column updates for sm_100a (least squares, optim.py:235-268).
//
// The reference updates, for every rank-one column r and every mode in turn,
//   partial_e = prod_{p != mode} col_p[i_p(e)]
//   rho_e     = resid_e + partial_e * col_mode[i(e)]
//   num_i = sum_{e in row i} rho_e partial_e,  den_i = sum partial_e^2
//   new_i = num_i / (den_i + reg)  (old value kept when den_i + reg <= 0)
//   resid_e = rho_e - partial_e * new[i(e)]
// Within one column r, rho is the same tensor for every mode in exact
// arithmetic: rho_{n+1} = rho_n - partial_n new_n + partial_{n+1} old_{n+1},
// and both products are the rank-one term with the current columns.  So the
// device keeps rho itself ("rhat", the residual with column r added back, in
// canonical entry order) for the whole column and skips the per-mode residual
// pass: per (r, mode) one segmented pass computes (num, den); between columns
// one pass folds rhat_{r+1} = (rhat_r - prod new_r) + prod col_{r+1}, fused
// into the mode-0 pass of column r+1 (mode 0 is in canonical order).  The two
// products use the reference's multiplication orders at those points (sub:
// ascending modes, as for the last mode; add: partial over p != 0, then col_0),
// so only the intermediate rho values differ from the reference, by rounding.
//
// Pass layout: warp per task of the mode-sorted task table (no atomics, fixed
// summation order); split rows leave (num, den) partials combined in task
// order.  Modes other than 0 read rhat through the mode permutation.
#include <cstring>

#include "common.cuh"

namespace cpfit {

struct CcdParams {
  int order, mode;
  int64_t nnz, dim;
  double *cols[CPFIT_MAXN];          // column r of every mode (cols[mode] updated in place)
  const double *sub[CPFIT_MAXN];     // fold: previous column (nullable as a whole)
  const int32_t *sidx[CPFIT_MAXN];   // mode-sorted coordinates (all modes)
  const int32_t *coords[CPFIT_MAXN];
  const int32_t *perm;               // sorted position -> entry (null: identity)
  const int64_t *task_begin;
  const int32_t *task_row;
  const int32_t *task_slot;
  int64_t ntasks;
  double *slots;                     // 2 * nslots (num, den)
  double *rhat;
  double reg;
  int fold, has_sub;
  double *numden;  // non-null: emit (num, den) per row, [num(I_n), den(I_n)], cols untouched
};

__device__ __forceinline__ double ccd_partial_sorted(const CcdParams &p, int64_t e) {
  double part = 1.0;
#pragma unroll
  for (int q = 0; q < CPFIT_MAXN; ++q) {
    if (q >= p.order) break;
    if (q == p.mode) continue;
    part = __dmul_rn(part, __ldg(p.cols[q] + __ldg(p.sidx[q] + e)));
  }
  return part;
}

// Pass A: warp per task, U entries per lane in flight.  FOLD (mode 0,
// identity order): rhat is first rebuilt for this column and written back.
template <bool FOLD>
__global__ void __launch_bounds__(256) ccd_rows_kernel(const CcdParams p) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < p.ntasks; t += nwarps) {
    const int64_t b0 = p.task_begin[t], b1 = p.task_begin[t + 1];
    const int64_t row = p.task_row[t];
    const double oc = p.cols[p.mode][row];
    const double s0 = (FOLD && p.has_sub) ? p.sub[0][row] : 0.0;
    double num = 0.0, den = 0.0;
    for (int64_t e0 = b0 + lane; e0 < b1; e0 += 32 * U) {
      double part[U], rh[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = e0 + 32 * u;
        part[u] = 0.0;
        rh[u] = 0.0;
        if (e < b1) {
          part[u] = ccd_partial_sorted(p, e);
          if constexpr (FOLD) {
            rh[u] = p.rhat[e];
          } else {
            const int64_t ent = p.perm ? __ldg(p.perm + e) : e;
            rh[u] = __ldg(p.rhat + ent);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = e0 + 32 * u;
        if (e < b1) {
          if constexpr (FOLD) {
            double r = rh[u];
            if (p.has_sub) {
              double s = s0;
#pragma unroll
              for (int q = 1; q < CPFIT_MAXN; ++q) {
                if (q >= p.order) break;
                s = __dmul_rn(s, __ldg(p.sub[q] + __ldg(p.sidx[q] + e)));
              }
              r = __dsub_rn(r, s);
            }
            r = __dadd_rn(r, __dmul_rn(part[u], oc));
            p.rhat[e] = r;
            rh[u] = r;
          }
          num += __dmul_rn(rh[u], part[u]);
          den += __dmul_rn(part[u], part[u]);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      num += __shfl_xor_sync(0xffffffffu, num, o);
      den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    const int slot = p.task_slot[t];
    if (lane == 0) {
      if (slot >= 0) {
        p.slots[2 * (int64_t)slot] = num;
        p.slots[2 * (int64_t)slot + 1] = den;
      } else if (p.numden) {
        p.numden[row] = num;
        p.numden[p.dim + row] = den;
      } else {
        const double dr = den + p.reg;
        p.cols[p.mode][row] = dr > 0.0 ? num / dr : oc;
      }
    }
  }
}

// Split rows: warp per row, slots summed lane-strided then by a fixed xor
// tree (deterministic), new value finalised (or (num, den) emitted).
__global__ void ccd_combine(const CcdParams p, const int32_t *__restrict__ split_row,
                            const int32_t *__restrict__ split_slot, int64_t nsplit) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < nsplit; s += nwarps) {
    const int64_t row = split_row[s];
    double num = 0.0, den = 0.0;
    for (int64_t k = split_slot[s] + lane; k < split_slot[s + 1]; k += 32) {
      num += p.slots[2 * k];
      den += p.slots[2 * k + 1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      num += __shfl_xor_sync(0xffffffffu, num, o);
      den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    if (lane == 0 && p.numden) {
      p.numden[row] = num;
      p.numden[p.dim + row] = den;
    } else if (lane == 0) {
      const double dr = den + p.reg;
      if (dr > 0.0) p.cols[p.mode][row] = num / dr;
    }
  }
}

// Distributed CCD++: new values from the all-reduced (num, den) of every row.
__global__ void ccd_finalize_kernel(int64_t dim, const double *__restrict__ numden, double reg,
                                    double *__restrict__ col) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double dr = numden[dim + i] + reg;
    if (dr > 0.0) col[i] = numden[i] / dr;
  }
}

__global__ void ccd_empty_rows(int64_t dim, const int64_t *__restrict__ offsets, double reg,
                               double *__restrict__ col) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim;
       i += (int64_t)gridDim.x * blockDim.x)
    if (offsets[i + 1] == offsets[i]) col[i] = 0.0 / reg;
}

// Canonical-order fold: rhat = (rhat - prod sub) + prod add (either side
// optional), products in the reference's orders (see the file comment).
__global__ void ccd_fold_kernel(int order, int64_t nnz, const CcdParams p, int has_add) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    int32_t ix[CPFIT_MAXN];
#pragma unroll
    for (int q = 0; q < CPFIT_MAXN; ++q)
      if (q < order) ix[q] = __ldg(p.coords[q] + e);
    double r = p.rhat[e];
    if (p.has_sub) {
      double s = __ldg(p.sub[0] + ix[0]);
#pragma unroll
      for (int q = 1; q < CPFIT_MAXN; ++q) {
        if (q >= order) break;
        s = __dmul_rn(s, __ldg(p.sub[q] + ix[q]));
      }
      r = __dsub_rn(r, s);
    }
    if (has_add) {
      double a = 1.0;
#pragma unroll
      for (int q = 1; q < CPFIT_MAXN; ++q) {
        if (q >= order) break;
        a = __dmul_rn(a, __ldg(p.cols[q] + ix[q]));
      }
      r = __dadd_rn(r, __dmul_rn(a, __ldg(p.cols[0] + ix[0])));
    }
    p.rhat[e] = r;
  }
}


// ---------------------------------------------------------------------------
// Flat segmented pass (mode-sorted order, no task table).  Warp w walks a fixed
// contiguous chunk [c0, c1) of the sorted entries 32 at a time; rows are
// contiguous, so a segmented warp scan (fixed shuffle tree) gives each row's
// step sum, carried across steps in entry order.  Rows wholly inside the chunk
// are finalised by the warp; a row that starts before the chunk leaves its
// partial in pf[c], one that continues past it in pl[c]; ccd_flat_fixup sums
// those in chunk order.  FOLD (identity order, mode 0): rhat re-formed first.
#ifndef CCD_FLAT_U
#define CCD_FLAT_U 2
#endif
#ifndef CCD_FLAT_STEPS
#define CCD_FLAT_STEPS 8
#endif
constexpr int CCD_FLAT_CHUNK = 32 * CCD_FLAT_U * CCD_FLAT_STEPS;  // entries per warp chunk

__device__ __forceinline__ void ccd_emit(const CcdParams &p, int64_t c, int32_t row,
                                         double num, double den, int32_t first_row,
                                         bool first_cont, int32_t last_row, bool last_cont,
                                         double2 *pf, double2 *pl) {
  if (row == first_row && first_cont) {
    pf[c] = make_double2(num, den);
  } else if (row == last_row && last_cont) {
    pl[c] = make_double2(num, den);
  } else if (p.numden) {
    p.numden[row] = num;
    p.numden[p.dim + row] = den;
  } else {
    const double dr = den + p.reg;
    if (dr > 0.0) p.cols[p.mode][row] = num / dr;
  }
}

template <int NO, int U>
struct CcdBatch {
  int32_t row[U], ix[U][NO], pe[U];
  double rh[U];
};

// Stream loads of one batch (U warp steps of 32 entries) of chunk c.
template <int NO, int U, bool FOLD>
__device__ __forceinline__ void ccd_load_batch(const CcdParams &p, int64_t c, int b, int lane,
                                               CcdBatch<NO, U> &B) {
  const int64_t c0 = c * CCD_FLAT_CHUNK;
  const int64_t c1 = min(c0 + (int64_t)CCD_FLAT_CHUNK, p.nnz);
  const int32_t *__restrict__ key = p.sidx[p.mode];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t e = c0 + (int64_t)b * 32 * U + 32 * u + lane;
    const bool ok = e < c1;
    B.row[u] = ok ? __ldg(key + e) : -2;
#pragma unroll
    for (int q = 0; q < NO; ++q) B.ix[u][q] = (ok && q != p.mode) ? __ldg(p.sidx[q] + e) : 0;
    if constexpr (FOLD) {
      B.rh[u] = ok ? __ldg(p.rhat + e) : 0.0;
      B.pe[u] = 0;
    } else {
      B.pe[u] = ok ? (p.perm ? __ldg(p.perm + e) : (int32_t)e) : 0;
      B.rh[u] = 0.0;
    }
  }
}

template <int NO, bool FOLD>
__global__ void __launch_bounds__(256) ccd_flat_kernel(const CcdParams p, int64_t nchunks,
                                                       double2 *__restrict__ pf,
                                                       double2 *__restrict__ pl) {
  constexpr int U = CCD_FLAT_U, S = CCD_FLAT_STEPS;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int32_t *__restrict__ key = p.sidx[p.mode];
  const double *__restrict__ mycol = p.cols[p.mode];
  const int mode = p.mode;
  int64_t c = warp;
  int bi = 0;
  CcdBatch<NO, U> cur;
  if (c < nchunks) ccd_load_batch<NO, U, FOLD>(p, c, 0, lane, cur);
  int32_t first_row = 0, last_row = 0, carry_row = -1;
  bool first_cont = false, last_cont = false;
  double cnum = 0.0, cden = 0.0;
  while (c < nchunks) {
    const int64_t c0 = c * CCD_FLAT_CHUNK;
    const int64_t c1 = min(c0 + (int64_t)CCD_FLAT_CHUNK, p.nnz);
    if (bi == 0) {
      first_row = __ldg(key + c0);
      last_row = __ldg(key + c1 - 1);
      first_cont = c0 > 0 && __ldg(key + c0 - 1) == first_row;
      last_cont = c1 < p.nnz && __ldg(key + c1) == last_row;
      carry_row = -1;
      cnum = cden = 0.0;
    }
    // software pipeline: the next batch's stream loads are in flight while
    // this batch gathers, multiplies and scans
    int64_t nc = c;
    int nb = bi + 1;
    if (nb == S) {
      nb = 0;
      nc = c + nwarps;
    }
    CcdBatch<NO, U> nxt;
    if (nc < nchunks) ccd_load_batch<NO, U, FOLD>(p, nc, nb, lane, nxt);
    // gathers (factor columns, rhat through the permutation)
    double g[U][NO], sv[U][NO], own[U], rh[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int q = 0; q < NO; ++q) {
        g[u][q] = q != mode ? __ldg(p.cols[q] + cur.ix[u][q]) : 1.0;
        if constexpr (FOLD)
          sv[u][q] = (p.has_sub && q != mode) ? __ldg(p.sub[q] + cur.ix[u][q]) : 1.0;
      }
      if constexpr (FOLD) {
        own[u] = cur.row[u] >= 0 ? mycol[cur.row[u]] : 0.0;
        if (p.has_sub) sv[u][0] = cur.row[u] >= 0 ? __ldg(p.sub[0] + cur.row[u]) : 0.0;
        rh[u] = cur.rh[u];
      } else {
        rh[u] = cur.row[u] >= 0 ? __ldg(p.rhat + cur.pe[u]) : 0.0;
      }
    }
    // products (reference orders), fold write-back, weights
    double w1[U], w2[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double part = 1.0;
#pragma unroll
      for (int q = 0; q < NO; ++q)
        if (q != mode) part = __dmul_rn(part, g[u][q]);
      if constexpr (FOLD) {  // mode 0
        double r = rh[u];
        if (p.has_sub) {
          double sp = sv[u][0];
#pragma unroll
          for (int q = 1; q < NO; ++q) sp = __dmul_rn(sp, sv[u][q]);
          r = __dsub_rn(r, sp);
        }
        r = __dadd_rn(r, __dmul_rn(part, own[u]));
        const int64_t e = c0 + (int64_t)bi * 32 * U + 32 * u + lane;
        if (cur.row[u] >= 0) p.rhat[e] = r;
        rh[u] = r;
      }
      w1[u] = cur.row[u] >= 0 ? __dmul_rn(rh[u], part) : 0.0;
      w2[u] = cur.row[u] >= 0 ? __dmul_rn(part, part) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t r = cur.row[u];
      double a = w1[u], b = w2[u];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double ua = __shfl_up_sync(0xffffffffu, a, d);
        const double ub = __shfl_up_sync(0xffffffffu, b, d);
        const int32_t ur = __shfl_up_sync(0xffffffffu, r, d);
        if (lane >= d && ur == r) {
          a = ua + a;
          b = ub + b;
        }
      }
      const int32_t next = __shfl_down_sync(0xffffffffu, r, 1);
      const int32_t r0 = __shfl_sync(0xffffffffu, r, 0);
      if (lane == 0 && carry_row >= 0 && r0 != carry_row)  // carried row ended last step
        ccd_emit(p, c, carry_row, cnum, cden, first_row, first_cont, last_row, last_cont, pf, pl);
      if (r == r0 && r == carry_row) {  // first segment continues the carry
        a = cnum + a;
        b = cden + b;
      }
      const bool tail = lane == 31 || next != r;
      if (tail && lane < 31 && r >= 0)
        ccd_emit(p, c, r, a, b, first_row, first_cont, last_row, last_cont, pf, pl);
      carry_row = __shfl_sync(0xffffffffu, r, 31);  // padded lanes leave -2 (nothing carried)
      cnum = __shfl_sync(0xffffffffu, a, 31);
      cden = __shfl_sync(0xffffffffu, b, 31);
    }
    if (nb == 0) {  // chunk done: flush the carry
      if (lane == 0 && carry_row >= 0)
        ccd_emit(p, c, carry_row, cnum, cden, first_row, first_cont, last_row, last_cont, pf, pl);
    }
    cur = nxt;
    c = nc;
    bi = nb;
  }
}

// Rows spanning chunks: pl[first chunk] + pf[later chunks], in chunk order
// (warp per row; lane-strided then fixed xor tree).  Empty rows: new = 0 / reg.
__global__ void ccd_flat_fixup(const CcdParams p, const int64_t *__restrict__ offsets,
                               const double2 *__restrict__ pf, const double2 *__restrict__ pl) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < p.dim; i += nwarps) {
    const int64_t s = offsets[i], e = offsets[i + 1];
    if (e == s) {
      if (lane == 0 && !p.numden && p.reg > 0.0) p.cols[p.mode][i] = 0.0 / p.reg;
      continue;
    }
    const int64_t cs = s / CCD_FLAT_CHUNK, ce = (e - 1) / CCD_FLAT_CHUNK;
    if (cs == ce) continue;
    double num = 0.0, den = 0.0;
    for (int64_t c = cs + 1 + lane; c <= ce; c += 32) {
      const double2 v = pf[c];
      num += v.x;
      den += v.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      num += __shfl_xor_sync(0xffffffffu, num, o);
      den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    if (lane == 0) {
      const double2 f = pl[cs];
      num = f.x + num;
      den = f.y + den;
      if (p.numden) {
        p.numden[i] = num;
        p.numden[p.dim + i] = den;
      } else {
        const double dr = den + p.reg;
        if (dr > 0.0) p.cols[p.mode][i] = num / dr;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Privatised canonical pass for modes with few rows (dims[mode] * 16 B per
// warp fits shared memory): entries read in canonical order (coalesced rhat,
// no permutation), every warp accumulates (num, den) into its own
// shared-memory row array -- lanes of a step that hit the same row add in
// lane order, one rank per round (match_any), so the order is fixed -- then the
// CTA sums its warps in order into cta_part[block], and ccd_priv_finish sums
// the CTAs in order.  Deterministic, no atomics.
constexpr int CCD_PRIV_U = 16;

template <int NO, int MODE>
__global__ void __launch_bounds__(256) ccd_priv_kernel(const CcdParams p, int64_t per_cta,
                                                       double2 *__restrict__ cta_part) {
  extern __shared__ double2 acc[];  // [warps][dim]
  constexpr int U = CCD_PRIV_U;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int64_t dim = p.dim;
  for (int64_t k = threadIdx.x; k < (int64_t)nw * dim; k += blockDim.x)
    acc[k] = make_double2(0.0, 0.0);
  __syncthreads();
  double2 *my = acc + (int64_t)wid * dim;
  const int64_t b0 = (int64_t)blockIdx.x * per_cta;
  const int64_t b1 = min(b0 + per_cta, p.nnz);
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = b0 + (int64_t)wid * 32 * U; base < b1; base += (int64_t)nw * 32 * U) {
    int32_t row[U];
    double w1[U], w2[U];
    int32_t ix[U][NO];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + 32 * u + lane;
#pragma unroll
      for (int q = 0; q < NO; ++q) ix[u][q] = e < b1 ? __ldg(p.coords[q] + e) : 0;
      w1[u] = e < b1 ? __ldg(p.rhat + e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + 32 * u + lane;
      double part = 1.0;
      int32_t r = -1;
#pragma unroll
      for (int q = 0; q < NO; ++q) {
        if (q == MODE) {
          r = ix[u][q];
        } else {
          part = __dmul_rn(part, __ldg(p.cols[q] + ix[u][q]));
        }
      }
      row[u] = e < b1 ? r : -1 - lane;  // padded lanes: distinct dummy keys
      w1[u] = e < b1 ? __dmul_rn(w1[u], part) : 0.0;
      w2[u] = e < b1 ? __dmul_rn(part, part) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned peers = __match_any_sync(0xffffffffu, row[u]);
      const int rk = __popc(peers & lt);
      const int rounds = __reduce_max_sync(0xffffffffu, rk);
      for (int j = 0; j <= rounds; ++j) {
        if (rk == j && row[u] >= 0) {
          double2 v = my[row[u]];
          v.x += w1[u];
          v.y += w2[u];
          my[row[u]] = v;
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  for (int64_t k = threadIdx.x; k < dim; k += blockDim.x) {
    double2 s = acc[k];
    for (int w = 1; w < nw; ++w) {
      const double2 v = acc[(int64_t)w * dim + k];
      s.x += v.x;
      s.y += v.y;
    }
    cta_part[(int64_t)blockIdx.x * dim + k] = s;
  }
}

__global__ void ccd_priv_finish(const CcdParams p, const double2 *__restrict__ cta_part,
                                int nblocks) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.dim;
       i += (int64_t)gridDim.x * blockDim.x) {
    double num = 0.0, den = 0.0;
    for (int b = 0; b < nblocks; ++b) {
      const double2 v = cta_part[(int64_t)b * p.dim + i];
      num += v.x;
      den += v.y;
    }
    if (p.numden) {
      p.numden[i] = num;
      p.numden[p.dim + i] = den;
    } else {
      const double dr = den + p.reg;
      if (dr > 0.0) p.cols[p.mode][i] = num / dr;
    }
  }
}

}  // namespace cpfit

using namespace cpfit;

static unsigned ccd_task_grid(int64_t ntasks) {
  int64_t blocks = (ntasks + 7) / 8;
  int64_t cap = (int64_t)num_sms() * 8;
  return (unsigned)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

// Pass selection (CPFIT_CCD_PATH=task|flat|priv overrides, for tuning):
// the flat segmented pass for orders 2..5 (fold fused in identity order,
// rhat through the permutation otherwise), the task-table pass beyond.
enum { CCD_PATH_TASK = 0, CCD_PATH_FLAT = 1, CCD_PATH_PRIV = 2 };
constexpr size_t CCD_PRIV_SMEM = 200 * 1024;

static int ccd_priv_warps(int64_t dim) {
  int64_t nw = (int64_t)CCD_PRIV_SMEM / (dim * (int64_t)sizeof(double2));
  return (int)(nw > 8 ? 8 : nw);
}

static int ccd_path(cpfit_pattern *pt, int mode, int fold) {
  const char *env = getenv("CPFIT_CCD_PATH");
  const int64_t dim = pt->dims[mode];
  const bool priv_ok = !fold && pt->order >= 2 && pt->order <= 4 && ccd_priv_warps(dim) >= 4;
  if (env) {
    if (!strcmp(env, "task")) return CCD_PATH_TASK;
    if (!strcmp(env, "priv") && priv_ok) return CCD_PATH_PRIV;
    return pt->order >= 2 && pt->order <= 5 ? CCD_PATH_FLAT : CCD_PATH_TASK;
  }
  // measured at cfg 3 (mode 2, 2,182 rows): flat-through-permutation 1.87 ms,
  // privatised 2.3 ms (five warps per SM hold the accumulators: latency-bound),
  // so the privatised pass is opt-in
  return pt->order >= 2 && pt->order <= 5 ? CCD_PATH_FLAT : CCD_PATH_TASK;
}

static int64_t ccd_priv_per_cta(int64_t nnz) {
  const int64_t nblocks = num_sms();
  int64_t per_cta = (nnz + nblocks - 1) / nblocks;
  return (per_cta + 32 * CCD_PRIV_U - 1) / (32 * CCD_PRIV_U) * (32 * CCD_PRIV_U);
}

template <int NO, int MODE>
static int ccd_priv_launch1(const CcdParams &p, int64_t per_cta, double2 *part, int nw,
                            size_t smem, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    CPFIT_CUDA(cudaFuncSetAttribute(ccd_priv_kernel<NO, MODE>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)CCD_PRIV_SMEM));
    attr_set = true;
  }
  ccd_priv_kernel<NO, MODE><<<num_sms(), nw * 32, smem, s>>>(p, per_cta, part);
  CPFIT_LAUNCH_CHECK("ccd_priv");
  return CPFIT_OK;
}

static int ccd_priv_launch(int order, int mode, const CcdParams &p, int64_t per_cta,
                           double2 *part, int nw, size_t smem, cudaStream_t s) {
#define CCD_PRIV_CASE(NO, M) \
  if (order == NO && mode == M) return ccd_priv_launch1<NO, M>(p, per_cta, part, nw, smem, s);
  CCD_PRIV_CASE(2, 0) CCD_PRIV_CASE(2, 1)
  CCD_PRIV_CASE(3, 0) CCD_PRIV_CASE(3, 1) CCD_PRIV_CASE(3, 2)
  CCD_PRIV_CASE(4, 0) CCD_PRIV_CASE(4, 1) CCD_PRIV_CASE(4, 2) CCD_PRIV_CASE(4, 3)
#undef CCD_PRIV_CASE
  set_error("privatised CCD pass: order %d mode %d not instantiated", order, mode);
  return CPFIT_EINVAL;
}

extern "C" {

int cpfit_ccd_step(cpfit_pattern *pt, int mode, double *const *cols, double *rhat,
                   int fold, const double *const *fold_sub, double reg, double *numden,
                   void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!pt || mode < 0 || mode >= pt->order) {
    set_error("mode %d out of range", mode);
    return CPFIT_EINVAL;
  }
  if (!cols || (pt->nnz > 0 && !rhat)) {
    set_error("cols and rhat are required");
    return CPFIT_EINVAL;
  }
  for (int q = 0; q < pt->order; ++q)
    if (!cols[q] || (fold_sub && !fold_sub[q])) {
      set_error("column of mode %d is null", q);
      return CPFIT_EINVAL;
    }
  CPFIT_TRY(ensure_layout(pt, mode, s));
  CpfitModeLayout &L = pt->modes[mode];
  if (fold && L.perm) {
    set_error("fused fold needs the identity (canonical) order: mode 0 only");
    return CPFIT_EINVAL;
  }
  CcdParams p{};
  p.order = pt->order;
  p.mode = mode;
  p.nnz = pt->nnz;
  p.dim = pt->dims[mode];
  for (int q = 0; q < pt->order; ++q) {
    p.cols[q] = cols[q];
    p.sub[q] = fold_sub ? fold_sub[q] : nullptr;
    p.sidx[q] = L.sorted_idx[q];
    p.coords[q] = pt->coords[q];
  }
  p.perm = L.perm;
  p.task_begin = L.task_begin;
  p.task_row = L.task_row;
  p.task_slot = L.task_slot;
  p.ntasks = L.ntasks;
  p.rhat = rhat;
  p.reg = reg;
  p.fold = fold;
  p.has_sub = fold_sub != nullptr;
  p.numden = numden;
  if (numden) CPFIT_CUDA(cudaMemsetAsync(numden, 0, 2 * (size_t)p.dim * sizeof(double), s));
  if (pt->nnz == 0) {
    if (!numden && reg > 0.0) {
      ccd_empty_rows<<<grid_for(p.dim, 256), 256, 0, s>>>(p.dim, L.offsets, reg, cols[mode]);
      CPFIT_LAUNCH_CHECK("ccd_empty_rows");
    }
    return CPFIT_OK;
  }
  const int path = ccd_path(pt, mode, fold);
  if (path == CCD_PATH_PRIV) {
    // few rows: canonical order, per-warp shared-memory accumulators
    const int nw = ccd_priv_warps(p.dim);
    const size_t smem = (size_t)nw * p.dim * sizeof(double2);
    const int64_t per_cta = ccd_priv_per_cta(pt->nnz);
    Scratch<double2> part(s);
    CPFIT_TRY(part.alloc((size_t)num_sms() * p.dim));
    CPFIT_TRY(ccd_priv_launch(pt->order, mode, p, per_cta, part.ptr, nw, smem, s));
    ccd_priv_finish<<<grid_for(p.dim, 128), 128, 0, s>>>(p, part.ptr, num_sms());
    CPFIT_LAUNCH_CHECK("ccd_priv_finish");
    return CPFIT_OK;
  }
  if (path == CCD_PATH_FLAT) {
    const int64_t nchunks = (pt->nnz + CCD_FLAT_CHUNK - 1) / CCD_FLAT_CHUNK;
    Scratch<double2> pf(s), pl(s);
    CPFIT_TRY(pf.alloc(nchunks));
    CPFIT_TRY(pl.alloc(nchunks));
    const unsigned grid = grid_for(nchunks * 32, 256);
#define CCD_FLAT_CASE(NO)                                                      \
  if (pt->order == NO) {                                                       \
    if (fold)                                                                  \
      ccd_flat_kernel<NO, true><<<grid, 256, 0, s>>>(p, nchunks, pf.ptr, pl.ptr);  \
    else                                                                       \
      ccd_flat_kernel<NO, false><<<grid, 256, 0, s>>>(p, nchunks, pf.ptr, pl.ptr); \
  }
    CCD_FLAT_CASE(2) CCD_FLAT_CASE(3) CCD_FLAT_CASE(4) CCD_FLAT_CASE(5)
#undef CCD_FLAT_CASE
    CPFIT_LAUNCH_CHECK("ccd_flat");
    ccd_flat_fixup<<<grid_for(p.dim * 32, 256), 256, 0, s>>>(p, L.offsets, pf.ptr, pl.ptr);
    CPFIT_LAUNCH_CHECK("ccd_flat_fixup");
    return CPFIT_OK;
  }
  Scratch<double> slots(s);
  if (L.nslots > 0) CPFIT_TRY(slots.alloc(2 * L.nslots));
  p.slots = slots.ptr;
  // rows without entries: num = den = 0, so new = 0 / reg when reg > 0
  if (!numden && reg > 0.0) {
    ccd_empty_rows<<<grid_for(p.dim, 256), 256, 0, s>>>(p.dim, L.offsets, reg, cols[mode]);
    CPFIT_LAUNCH_CHECK("ccd_empty_rows");
  }
  if (fold)
    ccd_rows_kernel<true><<<ccd_task_grid(L.ntasks), 256, 0, s>>>(p);
  else
    ccd_rows_kernel<false><<<ccd_task_grid(L.ntasks), 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("ccd_rows");
  if (L.nsplit > 0) {
    ccd_combine<<<grid_for(L.nsplit * 32, 256), 256, 0, s>>>(p, L.split_row, L.split_slot,
                                                            L.nsplit);
    CPFIT_LAUNCH_CHECK("ccd_combine");
  }
  return CPFIT_OK;
}

int cpfit_ccd_fold(cpfit_pattern *pt, const double *const *sub, const double *const *add,
                   double *rhat, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!pt) {
    set_error("null pattern");
    return CPFIT_EINVAL;
  }
  if (pt->nnz == 0 || (!sub && !add)) return CPFIT_OK;
  CcdParams p{};
  p.order = pt->order;
  p.nnz = pt->nnz;
  for (int q = 0; q < pt->order; ++q) {
    if ((sub && !sub[q]) || (add && !add[q])) {
      set_error("column of mode %d is null", q);
      return CPFIT_EINVAL;
    }
    p.sub[q] = sub ? sub[q] : nullptr;
    p.cols[q] = add ? const_cast<double *>(add[q]) : nullptr;
    p.coords[q] = pt->coords[q];
  }
  p.has_sub = sub != nullptr;
  p.rhat = rhat;
  ccd_fold_kernel<<<grid_for(pt->nnz, 256, 4), 256, 0, s>>>(pt->order, pt->nnz, p, add != nullptr);
  CPFIT_LAUNCH_CHECK("ccd_fold");
  return CPFIT_OK;
}

int cpfit_ccd_finalize(int64_t dim, const double *numden, double reg, double *col,
                       void *stream) {
  if (dim <= 0) return CPFIT_OK;
  ccd_finalize_kernel<<<grid_for(dim, 256), 256, 0, (cudaStream_t)stream>>>(dim, numden, reg,
                                                                            col);
  CPFIT_LAUNCH_CHECK("ccd_finalize");
  return CPFIT_OK;
}

}  // extern "C"
