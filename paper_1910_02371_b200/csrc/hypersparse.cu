// hypersparse.cu -- the pairwise-contraction baseline of the paper on the GPU
// (reference hypersparse.py).
//
// The reference keeps a doubly-compressed CSR (CCSR: rows with entries only)
// matricization of the tensor, multiplies it by a dense factor (TTM, giving a
// semi-sparse tensor with one length-R payload per nonzero fiber) and folds
// the remaining factors in pairwise.  These kernels reproduce its arithmetic
// order exactly:
//  * ccsr_spmm: payload[slot] = sum_j v_j * B[col_j] per column in numpy's
//    reduceat order (first product + pairwise sum of the rest);
//  * pairwise_tttp: p_r = ((v * A_first[c, r]) * A_next[c, r]) ... then the
//    row sum over r in numpy's order (np.sum on a contiguous axis: pairwise);
//  * pairwise_mttkrp_fold + segment sums: w_f = payload[f, r] * prod over the
//    remaining non-target modes, summed per target row in fiber order from
//    0.0 (np.bincount) through a stable sort of the fibers by target.
#include "common.cuh"

namespace cpfit {

// numpy pairwise_sum over get(j), j in [a, a + len) (loops_utils.h): blocks
// below 8 summed sequentially from -0.0, up to 128 with eight interleaved
// accumulators, longer ranges split at a multiple of 8 (explicit stack).
template <typename F>
__device__ double np_pairwise_gen(F get, int64_t a, int64_t len) {
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
        for (int64_t j = 0; j < f.len; ++j) res += get(f.a + j);
      } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = get(f.a + j);
        int64_t i = 8;
        const int64_t lim = f.len - (f.len % 8);
        for (; i < lim; i += 8)
#pragma unroll
          for (int j = 0; j < 8; ++j) r[j] += get(f.a + i + j);
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < f.len; ++i) res += get(f.a + i);
      }
      ret = res;
      --sp;
    } else {
      int64_t n2 = f.len / 2;
      n2 -= n2 % 8;
      if (f.state == 0) {
        f.state = 1;
        st[++sp] = {f.a, n2, 0, 0.0};
      } else if (f.state == 1) {
        f.left = ret;
        f.state = 2;
        st[++sp] = {f.a + n2, f.len - n2, 0, 0.0};
      } else {
        ret = f.left + ret;
        --sp;
      }
    }
  }
  return ret;
}

// np.add.reduceat along the entry axis of the (nnz, R) products: per column,
// the first product plus numpy's pairwise sum of the rest.  Thread per
// (nonzero row, column).
__global__ void ccsr_spmm_kernel(int64_t nrows, const int64_t *__restrict__ offs,
                                 const int64_t *__restrict__ cols,
                                 const double *__restrict__ vals,
                                 const double *__restrict__ B, int R,
                                 double *__restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nrows * R;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = k / R;
    const int r = (int)(k - row * R);
    const int64_t s = offs[row], e = offs[row + 1];
    auto prod = [&](int64_t j) { return __dmul_rn(vals[j], B[cols[j] * R + r]); };
    double acc = prod(s);
    if (e - s > 1) acc = acc + np_pairwise_gen(prod, s + 1, e - s - 1);
    out[k] = acc;
  }
}

// one entry per thread; products in a local array (R <= 256)
__global__ void pairwise_tttp_kernel(int64_t nnz, int np, int R, CpfitCols cols,
                                     const double *__restrict__ vals,
                                     double *__restrict__ out) {
  double p[256];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = vals[e];
    const double *f0 = cols.col[0] + (int64_t)cols.idx[0][e] * R;
    for (int r = 0; r < R; ++r) p[r] = __dmul_rn(v, f0[r]);
    for (int n = 1; n < np; ++n) {
      const double *fn = cols.col[n] + (int64_t)cols.idx[n][e] * R;
      for (int r = 0; r < R; ++r) p[r] = __dmul_rn(p[r], fn[r]);
    }
    // np.sum over the contiguous rank axis: numpy's pairwise sum of the row
    // (measured: unlike reduceat, no separate first element).  Non-recursive:
    // a recursive device function would run on the default 1 KB per-thread
    // stack, too small for p[]
    out[e] = np_pairwise_gen([&](int64_t j) { return p[j]; }, 0, R);
  }
}

// w[f, r] = payload[f, r] * prod_{k < nfold} fac_k[idx_k[f], r] (in order)
__global__ void pairwise_fold_kernel(int64_t nf, int R, int nfold, CpfitCols cols,
                                     const double *__restrict__ payload,
                                     double *__restrict__ w) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nf * R;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = k / R;
    const int r = (int)(k - f * R);
    double x = payload[k];
    for (int n = 0; n < nfold; ++n) x = __dmul_rn(x, cols.col[n][(int64_t)cols.idx[n][f] * R + r]);
    w[k] = x;
  }
}

// out[row, r] = 0.0 + sum of w[perm[j], r] over the row's sorted fibers, in
// order (np.bincount); thread per (row, r)
__global__ void segment_sum_kernel(int64_t dim, int R, const int64_t *__restrict__ offs,
                                   const int32_t *__restrict__ perm,
                                   const double *__restrict__ w, double *__restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < dim * R;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = k / R;
    const int r = (int)(k - row * R);
    double acc = 0.0;
    for (int64_t j = offs[row]; j < offs[row + 1]; ++j) acc += w[(int64_t)perm[j] * R + r];
    out[k] = acc;
  }
}

__global__ void target_offsets_kernel(const int32_t *__restrict__ sorted, int64_t n,
                                      int64_t dim, int64_t *__restrict__ offs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = i == 0 ? 0 : (int64_t)sorted[i - 1] + 1;
    const int64_t b = i == n ? dim : (int64_t)sorted[i];
    for (int64_t r = a; r <= b && r <= dim; ++r) offs[r] = i;
  }
}

}  // namespace cpfit

using namespace cpfit;

extern "C" {

int cpfit_ccsr_spmm(int64_t nrows, const int64_t *row_offsets, const int64_t *col_ids,
                    const double *values, const double *dense, int rank, double *payload,
                    void *stream) {
  if (nrows <= 0) return CPFIT_OK;
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  ccsr_spmm_kernel<<<grid_for(nrows * rank, 256), 256, 0, s>>>(nrows, row_offsets, col_ids,
                                                                values, dense, rank, payload);
  CPFIT_LAUNCH_CHECK("ccsr_spmm");
  return CPFIT_OK;
}

int cpfit_pairwise_tttp(int64_t nnz, int nfac, int rank, const int32_t *const *idx,
                        const double *const *factors, const double *values, double *out,
                        void *stream) {
  if (nnz <= 0) return CPFIT_OK;
  if (nfac < 1 || nfac > CPFIT_MAXN) { set_error("1..%d factors", CPFIT_MAXN); return CPFIT_EINVAL; }
  if (rank < 1 || rank > 256) { set_error("pairwise TTTP supports 1 <= R <= 256"); return CPFIT_EINVAL; }
  CpfitCols c{};
  for (int n = 0; n < nfac; ++n) {
    c.col[n] = factors[n];
    c.idx[n] = idx[n];
  }
  cudaStream_t s = (cudaStream_t)stream;
  pairwise_tttp_kernel<<<grid_for(nnz, 128), 128, 0, s>>>(nnz, nfac, rank, c, values, out);
  CPFIT_LAUNCH_CHECK("pairwise_tttp");
  return CPFIT_OK;
}

// MTTKRP tail of the pairwise chain: w = payload * (remaining factors), then
// per target row the fiber-order sum (np.bincount semantics).
int cpfit_pairwise_fold_sum(int64_t nfibers, int rank, int nfold, const int32_t *const *idx,
                            const double *const *factors, const double *payload,
                            const int32_t *target, int64_t dim, double *out, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  if (nfibers <= 0) {
    CPFIT_CUDA(cudaMemsetAsync(out, 0, (size_t)dim * rank * sizeof(double), s));
    return CPFIT_OK;
  }
  if (nfold < 0 || nfold > CPFIT_MAXN) { set_error("bad factor count"); return CPFIT_EINVAL; }
  CpfitCols c{};
  for (int n = 0; n < nfold; ++n) {
    c.col[n] = factors[n];
    c.idx[n] = idx[n];
  }
  Scratch<double> w(s);
  Scratch<int32_t> sorted(s), perm(s);
  Scratch<int64_t> offs(s);
  CPFIT_TRY(w.alloc((size_t)nfibers * rank));
  CPFIT_TRY(sorted.alloc(nfibers));
  CPFIT_TRY(perm.alloc(nfibers));
  CPFIT_TRY(offs.alloc(dim + 1));
  pairwise_fold_kernel<<<grid_for(nfibers * rank, 256, 4), 256, 0, s>>>(nfibers, rank, nfold, c,
                                                                        payload, w.ptr);
  CPFIT_LAUNCH_CHECK("pairwise_fold");
  int bits = 0;
  while (bits < 31 && ((int64_t)1 << bits) < dim) ++bits;
  CPFIT_TRY(radix_sort_pairs<int32_t>(target, nfibers, bits, sorted.ptr, perm.ptr, s));
  target_offsets_kernel<<<grid_for(nfibers + 1, 256), 256, 0, s>>>(sorted.ptr, nfibers, dim,
                                                                   offs.ptr);
  CPFIT_LAUNCH_CHECK("target_offsets");
  segment_sum_kernel<<<grid_for(dim * rank, 256, 4), 256, 0, s>>>(dim, rank, offs.ptr, perm.ptr,
                                                                  w.ptr, out);
  CPFIT_LAUNCH_CHECK("segment_sum");
  return CPFIT_OK;
}

}  // extern "C"
