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
// device keeps rho itself ("rhat", the residual with column r added back) for
// the whole column and skips the per-mode residual pass.  Each mode keeps its
// own copy of rhat in its mode-sorted order, so every pass streams it
// coalesced instead of gathering 8 B through the permutation (a 64 B DRAM
// access each on a 0.8 GB array at cfg 3), and each copy is re-formed in its
// own pass at the start of a column: rhat_r = (rhat_{r-1} - prod new_{r-1}) +
// prod old_r, with old_r saved before the sweep touches column r.  The
// products use the reference's multiplication orders (sub: modes ascending,
// as for the last mode; add: partial over p != 0, then col_0) and the same
// operands in every copy, so the copies stay bitwise identical; only the
// intermediate rho values differ from the reference's, by rounding.
//
// Pass layout: the flat segmented pass (fixed chunks of the mode-sorted
// entries per warp, segmented warp scans, chunk-boundary partials combined in
// chunk order: no atomics, deterministic).  A canonical-only rhat read
// through the permutation (rhat_sorted = 0) remains available for memory-lean
// callers; orders beyond 5 use the task-table pass.
#include <cstring>

#include "common.cuh"

namespace cpfit {

struct CcdParams {
  int order, mode;
  int64_t nnz, dim;
  double *cols[CPFIT_MAXN];          // column r of every mode (cols[mode] updated in place)
  const double *sub[CPFIT_MAXN];     // fold: previous column, new values (nullable as a whole)
  const double *add[CPFIT_MAXN];     // fold: this column before the sweep touched it (nullable)
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
  int fold, has_sub, has_add;
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

// Task-table pass (orders beyond the flat kernel's instantiations): warp per
// task, U entries per lane in flight; rhat read at the sorted position (a
// sorted copy) or through the permutation (canonical rhat).
__global__ void __launch_bounds__(256) ccd_rows_kernel(const CcdParams p) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < p.ntasks; t += nwarps) {
    const int64_t b0 = p.task_begin[t], b1 = p.task_begin[t + 1];
    const int64_t row = p.task_row[t];
    const double oc = p.cols[p.mode][row];
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
          rh[u] = __ldg(p.rhat + (p.perm ? __ldg(p.perm + e) : e));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        num += __dmul_rn(rh[u], part[u]);
        den += __dmul_rn(part[u], part[u]);
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

// Elementwise fold of one rhat copy: rhat = (rhat - prod sub) + prod add
// (either side optional), products in the reference's orders (see the file
// comment); p.coords = the copy's coordinate arrays (canonical or sorted).
__global__ void ccd_fold_kernel(int order, int64_t nnz, const CcdParams p) {
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
    if (p.has_add) {
      double a = 1.0;
#pragma unroll
      for (int q = 1; q < CPFIT_MAXN; ++q) {
        if (q >= order) break;
        a = __dmul_rn(a, __ldg(p.add[q] + ix[q]));
      }
      r = __dadd_rn(r, __dmul_rn(a, __ldg(p.add[0] + ix[0])));
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
// those in chunk order.  FOLD: this mode's rhat copy is re-formed first.
#ifndef CCD_FLAT_U
#define CCD_FLAT_U 2
#endif
#ifndef CCD_FLAT_STEPS
#define CCD_FLAT_STEPS 16
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
template <int NO, int U, bool FOLD, int MODE>
__device__ __forceinline__ void ccd_load_batch(const CcdParams &p, int64_t c, int b, int lane,
                                               CcdBatch<NO, U> &B) {
  const int64_t c0 = c * CCD_FLAT_CHUNK;
  const int64_t c1 = min(c0 + (int64_t)CCD_FLAT_CHUNK, p.nnz);
  const int32_t *__restrict__ key = p.sidx[MODE];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t e = c0 + (int64_t)b * 32 * U + 32 * u + lane;
    const bool ok = e < c1;
    B.row[u] = ok ? __ldg(key + e) : -2;
#pragma unroll
    for (int q = 0; q < NO; ++q) B.ix[u][q] = (ok && q != MODE) ? __ldg(p.sidx[q] + e) : 0;
    if constexpr (FOLD) {
      B.rh[u] = ok ? __ldg(p.rhat + e) : 0.0;
      B.pe[u] = 0;
    } else {
      B.pe[u] = ok ? (p.perm ? __ldg(p.perm + e) : (int32_t)e) : 0;
      B.rh[u] = 0.0;
    }
  }
}

// MODE is a template parameter: with a run-time mode every `q == mode` test in
// the unrolled per-mode loops became ISETP / FSEL / constant-bank pointer
// loads (cfg 3 pass 1.14 -> 1.09 ms at R = 4).
// HS / HA: the fold's sub / add sides as template flags too.
template <int NO, bool FOLD, int MODE, bool HS = false, bool HA = false>
__global__ void __launch_bounds__(256) ccd_flat_kernel(const CcdParams p, int64_t nchunks,
                                                       double2 *__restrict__ pf,
                                                       double2 *__restrict__ pl) {
  constexpr int U = CCD_FLAT_U, S = CCD_FLAT_STEPS;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int32_t *__restrict__ key = p.sidx[MODE];
  constexpr int mode = MODE;
  int64_t c = warp;
  int bi = 0;
  CcdBatch<NO, U> cur;
  if (c < nchunks) ccd_load_batch<NO, U, FOLD, MODE>(p, c, 0, lane, cur);
  int32_t first_row = 0, last_row = 0, carry_row = -1;
  bool first_cont = false, last_cont = false;
  double la = 0.0, lb = 0.0;  // this lane's share of the carried row's (num, den)
  while (c < nchunks) {
    const int64_t c0 = c * CCD_FLAT_CHUNK;
    const int64_t c1 = min(c0 + (int64_t)CCD_FLAT_CHUNK, p.nnz);
    if (bi == 0) {
      first_row = __ldg(key + c0);
      last_row = __ldg(key + c1 - 1);
      first_cont = c0 > 0 && __ldg(key + c0 - 1) == first_row;
      last_cont = c1 < p.nnz && __ldg(key + c1) == last_row;
      carry_row = -1;
      la = lb = 0.0;
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
    if (nc < nchunks) ccd_load_batch<NO, U, FOLD, MODE>(p, nc, nb, lane, nxt);
    // gathers (factor columns; rhat through the permutation unless FOLD)
    double g[U][NO], sv[U][NO], av[U][NO], rh[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t rw = cur.row[u] >= 0 ? cur.row[u] : 0;
#pragma unroll
      for (int q = 0; q < NO; ++q) {
        const int32_t iq = q == mode ? rw : cur.ix[u][q];
        g[u][q] = q != mode ? __ldg(p.cols[q] + iq) : 1.0;
        if constexpr (FOLD) {
          sv[u][q] = HS ? __ldg(p.sub[q] + iq) : 0.0;
          // modes after this one are not updated yet in this column: their
          // pre-sweep value is the current one (no second gather)
          av[u][q] = !HA ? 0.0 : (q > mode ? g[u][q] : __ldg(p.add[q] + iq));
        }
      }
      if constexpr (FOLD) {
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
      if constexpr (FOLD) {
        // rhat of this column: (rhat - prod sub) + prod add, the products in
        // the reference's orders (sub: modes ascending; add: partial over
        // p != 0, then col_0) -- identical in every mode's copy
        double r = rh[u];
        if (HS) {
          double sp = sv[u][0];
#pragma unroll
          for (int q = 1; q < NO; ++q) sp = __dmul_rn(sp, sv[u][q]);
          r = __dsub_rn(r, sp);
        }
        if (HA) {
          double ap = 1.0;
#pragma unroll
          for (int q = 1; q < NO; ++q) ap = __dmul_rn(ap, av[u][q]);
          r = __dadd_rn(r, __dmul_rn(ap, av[u][0]));
        }
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
      // fast path: the whole step continues the carried row -- per-lane sums
      if (__all_sync(0xffffffffu, r == carry_row)) {
        la += w1[u];
        lb += w2[u];
        continue;
      }
      // a boundary in this step: lanes of the carried row (a prefix) finish
      // it, its total is the fixed butterfly over the lane sums
      double a = w1[u], b = w2[u];
      int32_t rs = r;
      if (r == carry_row) {
        la += a;
        lb += b;
        a = b = 0.0;
        rs = -3;  // excluded from the scan below
      }
      if (carry_row >= 0) {
        double ta = la, tb = lb;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ta += __shfl_xor_sync(0xffffffffu, ta, o);
          tb += __shfl_xor_sync(0xffffffffu, tb, o);
        }
        if (lane == 0)
          ccd_emit(p, c, carry_row, ta, tb, first_row, first_cont, last_row, last_cont, pf, pl);
      }
      // the remaining rows of the step: segmented scan (fixed shuffle tree)
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double ua = __shfl_up_sync(0xffffffffu, a, d);
        const double ub = __shfl_up_sync(0xffffffffu, b, d);
        const int32_t ur = __shfl_up_sync(0xffffffffu, rs, d);
        if (lane >= d && ur == rs) {
          a = ua + a;
          b = ub + b;
        }
      }
      const int32_t next = __shfl_down_sync(0xffffffffu, rs, 1);
      if (lane < 31 && next != rs && rs >= 0)
        ccd_emit(p, c, rs, a, b, first_row, first_cont, last_row, last_cont, pf, pl);
      // the last segment continues: its step sum seeds lane 31's accumulator
      carry_row = __shfl_sync(0xffffffffu, rs, 31);  // padded lanes leave -2 (nothing carried)
      la = (lane == 31 && carry_row >= 0) ? a : 0.0;
      lb = (lane == 31 && carry_row >= 0) ? b : 0.0;
    }
    if (nb == 0 && carry_row >= 0) {  // chunk done: flush the carried row
      double ta = la, tb = lb;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ta += __shfl_xor_sync(0xffffffffu, ta, o);
        tb += __shfl_xor_sync(0xffffffffu, tb, o);
      }
      if (lane == 0)
        ccd_emit(p, c, carry_row, ta, tb, first_row, first_cont, last_row, last_cont, pf, pl);
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

}  // namespace cpfit

using namespace cpfit;

static unsigned ccd_task_grid(int64_t ntasks) {
  int64_t blocks = (ntasks + 7) / 8;
  int64_t cap = (int64_t)num_sms() * 8;
  return (unsigned)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

// Pass selection (CPFIT_CCD_PATH=task forces the task-table pass, for tests):
// the flat segmented pass for orders 2..5, the task-table pass beyond.
enum { CCD_PATH_TASK = 0, CCD_PATH_FLAT = 1 };

static int ccd_path(cpfit_pattern *pt) {
  const char *env = getenv("CPFIT_CCD_PATH");
  if (env && !strcmp(env, "task")) return CCD_PATH_TASK;
  return pt->order >= 2 && pt->order <= 5 ? CCD_PATH_FLAT : CCD_PATH_TASK;
}

namespace cpfit {
template <int NO, int M>
static int launch_ccd_flat_mode(int mode, bool fold, unsigned grid, cudaStream_t s,
                                const CcdParams &p, int64_t nchunks, double2 *pf, double2 *pl) {
  if constexpr (M < NO) {
    if (mode == M) {
      if (!fold) ccd_flat_kernel<NO, false, M><<<grid, 256, 0, s>>>(p, nchunks, pf, pl);
      else if (p.has_sub && p.has_add)
        ccd_flat_kernel<NO, true, M, true, true><<<grid, 256, 0, s>>>(p, nchunks, pf, pl);
      else if (p.has_sub)
        ccd_flat_kernel<NO, true, M, true, false><<<grid, 256, 0, s>>>(p, nchunks, pf, pl);
      else
        ccd_flat_kernel<NO, true, M, false, true><<<grid, 256, 0, s>>>(p, nchunks, pf, pl);
      return CPFIT_OK;
    }
    return launch_ccd_flat_mode<NO, M + 1>(mode, fold, grid, s, p, nchunks, pf, pl);
  } else {
    set_error("mode %d out of range", mode);
    return CPFIT_EINVAL;
  }
}

static int launch_ccd_flat(int order, int mode, bool fold, unsigned grid, cudaStream_t s,
                           const CcdParams &p, int64_t nchunks, double2 *pf, double2 *pl) {
  switch (order) {
    case 2: return launch_ccd_flat_mode<2, 0>(mode, fold, grid, s, p, nchunks, pf, pl);
    case 3: return launch_ccd_flat_mode<3, 0>(mode, fold, grid, s, p, nchunks, pf, pl);
    case 4: return launch_ccd_flat_mode<4, 0>(mode, fold, grid, s, p, nchunks, pf, pl);
    case 5: return launch_ccd_flat_mode<5, 0>(mode, fold, grid, s, p, nchunks, pf, pl);
  }
  set_error("order %d has no flat CCD++ kernel", order);
  return CPFIT_EINVAL;
}
}  // namespace cpfit

extern "C" {

int cpfit_ccd_step(cpfit_pattern *pt, int mode, double *const *cols, double *rhat,
                   int rhat_sorted, const double *const *fold_sub,
                   const double *const *fold_add, double reg, double *numden, void *stream) {
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
    if (!cols[q] || (fold_sub && !fold_sub[q]) || (fold_add && !fold_add[q])) {
      set_error("column of mode %d is null", q);
      return CPFIT_EINVAL;
    }
  CPFIT_TRY(ensure_layout(pt, mode, s));
  CpfitModeLayout &L = pt->modes[mode];
  const bool sorted = rhat_sorted || !L.perm;  // identity order: canonical == sorted
  const bool fold = fold_sub || fold_add;
  if (fold && !sorted) {
    set_error("folding needs rhat in the mode-sorted order (rhat_sorted = 1)");
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
    p.add[q] = fold_add ? fold_add[q] : nullptr;
    p.sidx[q] = L.sorted_idx[q];
    p.coords[q] = pt->coords[q];
  }
  p.perm = sorted ? nullptr : L.perm;
  p.task_begin = L.task_begin;
  p.task_row = L.task_row;
  p.task_slot = L.task_slot;
  p.ntasks = L.ntasks;
  p.rhat = rhat;
  p.reg = reg;
  p.fold = fold;
  p.has_sub = fold_sub != nullptr;
  p.has_add = fold_add != nullptr;
  p.numden = numden;
  if (numden) CPFIT_CUDA(cudaMemsetAsync(numden, 0, 2 * (size_t)p.dim * sizeof(double), s));
  if (pt->nnz == 0) {
    if (!numden && reg > 0.0) {
      ccd_empty_rows<<<grid_for(p.dim, 256), 256, 0, s>>>(p.dim, L.offsets, reg, cols[mode]);
      CPFIT_LAUNCH_CHECK("ccd_empty_rows");
    }
    return CPFIT_OK;
  }
  const int path = ccd_path(pt);
  if (path == CCD_PATH_FLAT) {
    const int64_t nchunks = (pt->nnz + CCD_FLAT_CHUNK - 1) / CCD_FLAT_CHUNK;
    Scratch<double2> pf(s), pl(s);
    CPFIT_TRY(pf.alloc(nchunks));
    CPFIT_TRY(pl.alloc(nchunks));
    const unsigned grid = grid_for(nchunks * 32, 256);
    CPFIT_TRY(launch_ccd_flat(pt->order, mode, fold, grid, s, p, nchunks, pf.ptr, pl.ptr));
    CPFIT_LAUNCH_CHECK("ccd_flat");
    ccd_flat_fixup<<<grid_for(p.dim * 32, 256), 256, 0, s>>>(p, L.offsets, pf.ptr, pl.ptr);
    CPFIT_LAUNCH_CHECK("ccd_flat_fixup");
    return CPFIT_OK;
  }
  // task-table pass; a fold is a separate elementwise launch in sorted order
  if (fold) {
    CcdParams f = p;
    for (int q = 0; q < pt->order; ++q) f.coords[q] = L.sorted_idx[q];
    ccd_fold_kernel<<<grid_for(pt->nnz, 256, 4), 256, 0, s>>>(pt->order, pt->nnz, f);
    CPFIT_LAUNCH_CHECK("ccd_fold");
  }
  Scratch<double> slots(s);
  if (L.nslots > 0) CPFIT_TRY(slots.alloc(2 * L.nslots));
  p.slots = slots.ptr;
  // rows without entries: num = den = 0, so new = 0 / reg when reg > 0
  if (!numden && reg > 0.0) {
    ccd_empty_rows<<<grid_for(p.dim, 256), 256, 0, s>>>(p.dim, L.offsets, reg, cols[mode]);
    CPFIT_LAUNCH_CHECK("ccd_empty_rows");
  }
  ccd_rows_kernel<<<ccd_task_grid(L.ntasks), 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("ccd_rows");
  if (L.nsplit > 0) {
    ccd_combine<<<grid_for(L.nsplit * 32, 256), 256, 0, s>>>(p, L.split_row, L.split_slot,
                                                            L.nsplit);
    CPFIT_LAUNCH_CHECK("ccd_combine");
  }
  return CPFIT_OK;
}

int cpfit_ccd_fold(cpfit_pattern *pt, int mode, const double *const *sub,
                   const double *const *add, double *rhat, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!pt || mode < -1 || mode >= pt->order) {
    set_error("bad pattern or mode %d", mode);
    return CPFIT_EINVAL;
  }
  if (pt->nnz == 0 || (!sub && !add)) return CPFIT_OK;
  CcdParams p{};
  p.order = pt->order;
  p.nnz = pt->nnz;
  if (mode >= 0) CPFIT_TRY(ensure_layout(pt, mode, s));
  for (int q = 0; q < pt->order; ++q) {
    if ((sub && !sub[q]) || (add && !add[q])) {
      set_error("column of mode %d is null", q);
      return CPFIT_EINVAL;
    }
    p.sub[q] = sub ? sub[q] : nullptr;
    p.add[q] = add ? add[q] : nullptr;
    p.coords[q] = mode >= 0 ? pt->modes[mode].sorted_idx[q] : pt->coords[q];
  }
  p.has_sub = sub != nullptr;
  p.has_add = add != nullptr;
  p.rhat = rhat;
  ccd_fold_kernel<<<grid_for(pt->nnz, 256, 4), 256, 0, s>>>(pt->order, pt->nnz, p);
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
