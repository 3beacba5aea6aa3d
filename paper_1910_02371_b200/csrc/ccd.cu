// ccd.cu -- CCD++ single-column update for sm_100a.
//
// One (r, mode) step of the least-squares CCD++ sweep (optim.py:249-268):
//   partial_e = prod_{p != mode} col_p[i_p(e)]         (p ascending)
//   rho_e     = resid_e + partial_e * col_mode[i(e)]
//   num_i = sum_{e in row i} rho_e partial_e, den_i = sum partial_e^2
//   new_i = num_i / (den_i + reg) if den_i + reg > 0 else col_mode[i]
//   resid_e = rho_e - partial_e * new[i(e)]
// Pass A walks the mode-sorted tasks (warp per task, no atomics); split rows
// are combined in a fixed order.  Pass B (residual) runs in canonical order
// (coalesced) for modes with a permutation; for mode 0 (identity order) it is
// fused into pass A for rows owned by one task.  rho and resid use explicitly rounded
// (non-contracted) operations so each element follows the reference's
// rounding; only the per-row sums are reassociated.
#include "common.cuh"

namespace cpfit {

struct CcdParams {
  int order, mode;
  int64_t nnz, dim;
  const double *cols[CPFIT_MAXN];   // column r of every mode (contiguous, length I_n)
  const int32_t *sidx[CPFIT_MAXN];  // mode-sorted coordinates (all modes)
  const int32_t *coords[CPFIT_MAXN];
  const int32_t *perm;              // sorted position -> entry (null: identity)
  const int64_t *task_begin;
  const int32_t *task_row;
  const int32_t *task_slot;
  int64_t ntasks;
  const double *old_col;  // col_mode before the update
  double *new_col;
  double *slots;          // 2 * nslots (num, den)
  double *resid;
  double reg;
  double *numden;         // non-null: emit (num, den) per row, [num(I_n), den(I_n)], and stop
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

__global__ void ccd_init_newcol(const CcdParams p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.dim;
       i += (int64_t)gridDim.x * blockDim.x)
    p.new_col[i] = p.reg > 0.0 ? 0.0 / p.reg : p.old_col[i];  // empty rows: num = den = 0
}

// Residual update of the sorted entries [b0, b1) of one row (pass B):
// rho = resid + part * old, resid = rho - part * new (reference rounding).
__device__ __forceinline__ void ccd_update_range(const CcdParams &p, int64_t b0, int64_t b1,
                                                 double oc, double nc) {
  const int lane = threadIdx.x & 31;
  for (int64_t e = b0 + lane; e < b1; e += 32) {
    const double part = ccd_partial_sorted(p, e);
    const int64_t ent = p.perm ? __ldg(p.perm + e) : e;
    const double rho = __dadd_rn(p.resid[ent], __dmul_rn(part, oc));
    p.resid[ent] = __dsub_rn(rho, __dmul_rn(part, nc));
  }
}

// Pass A (+ B for rows owned by one task): warp per task of the coarse table.
// A row that fits one task is finished here -- its new value is known after
// the warp's reduction, so the residual of its entries is updated right away
// while they are still L1/L2-hot; split rows leave (num, den) partials.
__global__ void __launch_bounds__(256) ccd_rows_kernel(const CcdParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < p.ntasks; t += nwarps) {
    const int64_t b0 = p.task_begin[t], b1 = p.task_begin[t + 1];
    const int64_t row = p.task_row[t];
    const double oc = p.old_col[row];
    double num = 0.0, den = 0.0;
    for (int64_t e = b0 + lane; e < b1; e += 32) {
      const double part = ccd_partial_sorted(p, e);
      const int64_t ent = p.perm ? __ldg(p.perm + e) : e;
      const double rho = __dadd_rn(p.resid[ent], __dmul_rn(part, oc));
      num += __dmul_rn(rho, part);
      den += __dmul_rn(part, part);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      num += __shfl_xor_sync(0xffffffffu, num, o);
      den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    const int slot = p.task_slot[t];
    if (slot < 0 && p.numden) {
      if (lane == 0) {
        p.numden[row] = num;
        p.numden[p.dim + row] = den;
      }
    } else if (slot < 0) {
      const double dr = den + p.reg;
      const double nc = dr > 0.0 ? num / dr : oc;
      if (lane == 0) p.new_col[row] = nc;
      // identity order (mode 0): the fused residual pass stays coalesced;
      // through a permutation a separate canonical-order pass is cheaper
      if (!p.perm) ccd_update_range(p, b0, b1, oc, nc);
    } else if (lane == 0) {
      p.slots[2 * (int64_t)slot] = num;
      p.slots[2 * (int64_t)slot + 1] = den;
    }
  }
}

// Split rows: warp per row, slots summed lane-strided then by a fixed xor
// tree (deterministic), new value finalised.
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
      p.new_col[row] = dr > 0.0 ? num / dr : p.old_col[row];
    }
  }
}

// Distributed CCD++: new value from the all-reduced (num, den) of every row.
__global__ void ccd_finalize_kernel(const CcdParams p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.dim;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double dr = p.numden[p.dim + i] + p.reg;
    p.new_col[i] = dr > 0.0 ? p.numden[i] / dr : p.old_col[i];
  }
}

// Pass B in canonical order (modes with a permutation): coalesced.
__global__ void ccd_resid_kernel(const CcdParams p) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p.nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    double part = 1.0;
#pragma unroll
    for (int q = 0; q < CPFIT_MAXN; ++q) {
      if (q >= p.order) break;
      if (q == p.mode) continue;
      part = __dmul_rn(part, __ldg(p.cols[q] + __ldg(p.coords[q] + e)));
    }
    const int32_t i = __ldg(p.coords[p.mode] + e);
    const double rho = __dadd_rn(p.resid[e], __dmul_rn(part, __ldg(p.old_col + i)));
    p.resid[e] = __dsub_rn(rho, __dmul_rn(part, __ldg(p.new_col + i)));
  }
}

// Pass B for the tasks of split rows only, identity order (mode 0).
__global__ void __launch_bounds__(256) ccd_split_resid_kernel(const CcdParams p) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < p.ntasks; t += nwarps) {
    if (p.task_slot[t] < 0) continue;
    const int64_t row = p.task_row[t];
    ccd_update_range(p, p.task_begin[t], p.task_begin[t + 1], p.old_col[row], p.new_col[row]);
  }
}

}  // namespace cpfit

using namespace cpfit;

static unsigned ccd_task_grid(int64_t ntasks) {
  int64_t blocks = (ntasks + 7) / 8;
  int64_t cap = (int64_t)num_sms() * 8;
  return (unsigned)(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

extern "C" {

static int ccd_setup(cpfit_pattern *pt, int mode, const double *const *cols,
                     const double *old_col, double *new_col, double *resid, double reg,
                     cudaStream_t s, CcdParams &p) {
  if (!pt || mode < 0 || mode >= pt->order) {
    set_error("mode %d out of range", mode);
    return CPFIT_EINVAL;
  }
  CPFIT_TRY(ensure_layout(pt, mode, s));
  CpfitModeLayout &L = pt->modes[mode];
  p = CcdParams{};
  p.order = pt->order;
  p.mode = mode;
  p.nnz = pt->nnz;
  p.dim = pt->dims[mode];
  for (int q = 0; q < pt->order; ++q) {
    p.cols[q] = q == mode ? old_col : cols[q];
    p.sidx[q] = L.sorted_idx[q];
    p.coords[q] = pt->coords[q];
  }
  p.perm = L.perm;
  p.task_begin = L.task_begin;
  p.task_row = L.task_row;
  p.task_slot = L.task_slot;
  p.ntasks = L.ntasks;
  p.old_col = old_col;
  p.new_col = new_col;
  p.resid = resid;
  p.reg = reg;
  return CPFIT_OK;
}

// pass A (+ split-row combine): finalises new_col, or fills p.numden
static int ccd_pass_a(cpfit_pattern *pt, CcdParams &p, cudaStream_t s) {
  CpfitModeLayout &L = pt->modes[p.mode];
  Scratch<double> slots(s);
  if (L.nslots > 0) CPFIT_TRY(slots.alloc(2 * L.nslots));
  p.slots = slots.ptr;
  if (p.numden) {
    CPFIT_CUDA(cudaMemsetAsync(p.numden, 0, 2 * (size_t)p.dim * sizeof(double), s));
  } else {
    ccd_init_newcol<<<grid_for(p.dim, 256), 256, 0, s>>>(p);
    CPFIT_LAUNCH_CHECK("ccd_init_newcol");
  }
  if (pt->nnz == 0) return CPFIT_OK;
  ccd_rows_kernel<<<ccd_task_grid(L.ntasks), 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("ccd_rows");
  if (L.nsplit > 0) {
    ccd_combine<<<grid_for(L.nsplit * 32, 256), 256, 0, s>>>(p, L.split_row, L.split_slot,
                                                            L.nsplit);
    CPFIT_LAUNCH_CHECK("ccd_combine");
  }
  return CPFIT_OK;
}

int cpfit_ccd_update(cpfit_pattern *pt, int mode, const double *const *cols,
                     const double *old_col, double *new_col, double *resid, double reg,
                     void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  CcdParams p;
  CPFIT_TRY(ccd_setup(pt, mode, cols, old_col, new_col, resid, reg, s, p));
  CPFIT_TRY(ccd_pass_a(pt, p, s));
  if (pt->nnz == 0) return CPFIT_OK;
  CpfitModeLayout &L = pt->modes[mode];
  if (p.perm) {
    ccd_resid_kernel<<<grid_for(pt->nnz, 256, 4), 256, 0, s>>>(p);
    CPFIT_LAUNCH_CHECK("ccd_resid");
  } else if (L.nsplit > 0) {
    ccd_split_resid_kernel<<<ccd_task_grid(L.ntasks), 256, 0, s>>>(p);
    CPFIT_LAUNCH_CHECK("ccd_split_resid");
  }
  return CPFIT_OK;
}

int cpfit_ccd_numden(cpfit_pattern *pt, int mode, const double *const *cols,
                     const double *old_col, const double *resid, double *numden,
                     void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  CcdParams p;
  CPFIT_TRY(ccd_setup(pt, mode, cols, old_col, nullptr, const_cast<double *>(resid), 0.0, s, p));
  if (!numden) {
    set_error("numden is required");
    return CPFIT_EINVAL;
  }
  p.numden = numden;
  return ccd_pass_a(pt, p, s);
}

int cpfit_ccd_apply(cpfit_pattern *pt, int mode, const double *const *cols,
                    const double *old_col, const double *numden, double reg, double *new_col,
                    double *resid, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  CcdParams p;
  CPFIT_TRY(ccd_setup(pt, mode, cols, old_col, new_col, resid, reg, s, p));
  p.numden = const_cast<double *>(numden);
  ccd_finalize_kernel<<<grid_for(p.dim, 256), 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("ccd_finalize");
  if (pt->nnz == 0) return CPFIT_OK;
  ccd_resid_kernel<<<grid_for(pt->nnz, 256, 4), 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("ccd_resid");
  return CPFIT_OK;
}

}  // extern "C"
