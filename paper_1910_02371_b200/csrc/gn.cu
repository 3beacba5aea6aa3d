// gn.cu -- kernels of the implicit second-order (Gauss-Newton / Newton) step.
//
// The reference's second-order operator (optim.py:348-464, hessian_matvec /
// _SecondOrderOperator) needs, per CG iteration,
//   z_e = phi2_e * sum_d sum_r X_d[i_d(e), r] * prod_{p != d} A_p[i_p(e), r]
// (the sum of the N TTTPs with one factor slot substituted by its update
// block) followed by one MTTKRP of z per mode.  tttp_subst_kernel computes z
// in ONE pass: every entry gathers its N factor rows and N update rows once
// (2N rows instead of the N^2 of N separate TTTPs) and forms the
// leave-one-out products with prefix / suffix products per column.
// axpby_kernel is the vector update of PCG (optim.py:492-531).
#include <cfloat>

#include "common.cuh"

namespace cpfit {

struct SubstParams {
  int order, rank;
  int64_t nnz;
  const int32_t *idx[CPFIT_MAXN];
  const void *fac[CPFIT_MAXN];
  const void *x[CPFIT_MAXN];
  const void *w;  // nullable: unit weights
  void *out;
};

// LPE lanes per entry (power of two), each owning columns q, q+LPE, ...
template <typename T, int LPE>
__global__ void __launch_bounds__(256) tttp_subst_kernel(const SubstParams p) {
  const int lane = threadIdx.x & 31;
  const int q = lane % LPE;
  constexpr int G = 32 / LPE;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T *__restrict__ const *fac = reinterpret_cast<const T *const *>(p.fac);
  const T *__restrict__ const *xb = reinterpret_cast<const T *const *>(p.x);
  for (int64_t base = warp * G; base < p.nnz; base += nwarps * G) {
    const int64_t e = base + lane / LPE;
    const bool live = e < p.nnz;
    double s = 0.0;
    if (live) {
      uint32_t row[CPFIT_MAXN];
#pragma unroll
      for (int n = 0; n < CPFIT_MAXN; ++n)
        if (n < p.order) row[n] = (uint32_t)__ldg(p.idx[n] + e);
      for (int c = q; c < p.rank; c += LPE) {
        double f[CPFIT_MAXN], xv[CPFIT_MAXN];
#pragma unroll
        for (int n = 0; n < CPFIT_MAXN; ++n) {
          if (n < p.order) {
            const size_t off = (size_t)row[n] * (unsigned)p.rank + c;
            f[n] = (double)__ldg(fac[n] + off);
            xv[n] = (double)__ldg(xb[n] + off);
          }
        }
        // sum_d x_d * prod_{p<d} f_p * prod_{p>d} f_p
        double pre = 1.0, acc = 0.0;
        double suf[CPFIT_MAXN];
        suf[CPFIT_MAXN - 1] = 1.0;
#pragma unroll
        for (int n = CPFIT_MAXN - 1; n > 0; --n)
          suf[n - 1] = (n < p.order) ? suf[n] * f[n] : 1.0;
#pragma unroll
        for (int n = 0; n < CPFIT_MAXN; ++n) {
          if (n < p.order) {
            acc += xv[n] * (pre * suf[n]);
            pre *= f[n];
          }
        }
        s += acc;
      }
    }
#pragma unroll
    for (int o = LPE / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (live && q == 0) {
      const T *w = (const T *)p.w;
      ((T *)p.out)[e] = (T)(w ? (double)w[e] * s : s);
    }
  }
}

// Vectorised variant for R <= LPE * VEC (one VEC-wide column slice per lane):
// a warp takes 32 consecutive entries, loads their indices coalesced (one
// entry per lane) and broadcasts them by shuffle to the G = 32 / LPE lane
// groups; each group gathers one entry's 2N rows with 16-byte loads (two
// sub-iterations' loads in flight), reduces over its LPE lanes, and the
// result lands on lane (entry % 32) for a coalesced store.
template <typename T, int VEC, int LPE, int NP>
__global__ void __launch_bounds__(256) tttp_subst_vec_kernel(const SubstParams p) {
  constexpr int G = 32 / LPE;
  constexpr int NPM = NP > 0 ? NP : CPFIT_MAXN;
  const int np = NP > 0 ? NP : p.order;
  const int lane = threadIdx.x & 31;
  const int g = lane / LPE, q = lane % LPE;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned R = (unsigned)p.rank;
  const int col = q * VEC;
  const bool colok = col < p.rank;
  const T *fac[NPM];
  const T *xb[NPM];
#pragma unroll
  for (int n = 0; n < NPM; ++n) {
    fac[n] = (const T *)p.fac[n < np ? n : 0];
    xb[n] = (const T *)p.x[n < np ? n : 0];
  }
  for (int64_t base = warp * 32; base < p.nnz; base += nwarps * 32) {
    const int cnt = (int)(p.nnz - base < 32 ? p.nnz - base : 32);
    int32_t my_idx[NPM];
#pragma unroll
    for (int n = 0; n < NPM; ++n)
      my_idx[n] = (n < np && lane < cnt) ? __ldg(p.idx[n] + base + lane) : 0;
    double res = 0.0;
#pragma unroll 2
    for (int s = 0; s < LPE; ++s) {
      const int j = s * G + g;
      T f[NPM][VEC], xv[NPM][VEC];
#pragma unroll
      for (int n = 0; n < NPM; ++n) {
        const unsigned row = (unsigned)__shfl_sync(0xffffffffu, my_idx[n], j);
        if (n < np && colok) {
          load_vec<T, VEC>(fac[n] + row * R + col, f[n]);
          load_vec<T, VEC>(xb[n] + row * R + col, xv[n]);
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) f[n][v] = xv[n][v] = T(0);
        }
      }
      double part = 0.0;
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        double sf[NPM];
        sf[NPM - 1] = 1.0;
#pragma unroll
        for (int n = NPM - 1; n > 0; --n) sf[n - 1] = (n < np) ? sf[n] * (double)f[n][v] : 1.0;
        double pre = 1.0;
#pragma unroll
        for (int n = 0; n < NPM; ++n) {
          if (n < np) {
            part += (double)xv[n][v] * (pre * sf[n]);
            pre *= (double)f[n][v];
          }
        }
      }
#pragma unroll
      for (int o = LPE / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      const double mine = __shfl_sync(0xffffffffu, part, (lane % G) * LPE);
      if (lane / G == s) res = mine;
    }
    if (lane < cnt) {
      const T *w = (const T *)p.w;
      ((T *)p.out)[base + lane] = (T)(w ? (double)__ldg(w + base + lane) * res : res);
    }
  }
}

// Block-diagonal preconditioner, inverted once per GN step: warp per row,
// lane j holds column j of A = G + shift I (identity-padded to RMAX), and an
// in-place Gauss-Jordan sweep (no pivoting: A is SPD) leaves A^{-1} in the
// same layout (column broadcasts through shared memory, see below).  Rows meeting a non-positive pivot are counted in *nbad; the
// caller then keeps the pivoted solve (cpfit_solve_rows) for that mode, so
// singular systems still fail exactly like np.linalg.solve.
template <typename T, int RMAX>
__global__ void __launch_bounds__(128, 5) spd_inverse_kernel(int R, int64_t nrows,
                                                          const T *__restrict__ gram,
                                                          int64_t gstride, double shift,
                                                          T *__restrict__ inv,
                                                          unsigned long long *nbad) {
  const int lane = threadIdx.x & 31;
  const int64_t wrow = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const bool active = wrow < nrows;
  const int64_t row = active ? wrow : nrows - 1;
  const T *G = gram + row * gstride;
  double a[RMAX];
#pragma unroll
  for (int i = 0; i < RMAX; ++i) {
    const bool in = i < R && lane < R;
    a[i] = in ? (double)__ldg(G + i * R + lane) + (i == lane ? shift : 0.0)
              : (i == lane ? 1.0 : 0.0);
  }
  bool ok = true;
  // Column k of the partly swept matrix: A[i][k] = A[k][i] for unswept i
  // (i >= k) and -A[k][i] for swept i (i < k) -- the sweep keeps the swept
  // and unswept blocks symmetric and the blocks between them antisymmetric --
  // so every lane stores its own a[k] and the column is read back as
  // warp-uniform shared-memory loads (vectorised pairs) instead of 2 x 32
  // shuffles per step.  Buffers alternate by k parity.
  __shared__ __align__(16) double col_buf[4][2][32];
  double(&cb)[2][32] = col_buf[(threadIdx.x >> 5) & 3];
#pragma unroll
  for (int k = 0; k < RMAX; ++k) {
    double *cs = cb[k & 1];
    cs[lane] = a[k];
    __syncwarp();
    const double piv = cs[k];
    ok = ok && piv > 0.0 && piv < DBL_MAX;
    const double rp = 1.0 / piv;
    double c[RMAX];
#pragma unroll
    for (int i = 0; i < RMAX; ++i) c[i] = i < k ? -cs[i] : cs[i];
    const double rk = a[k] * rp;
#pragma unroll
    for (int i = 0; i < RMAX; ++i) {
      if (lane == k)
        a[i] = (i == k) ? rp : -c[i] * rp;
      else
        a[i] = (i == k) ? rk : a[i] - c[i] * rk;
    }
  }
  if (!active) return;
  if (lane < R) {
    T *dst = inv + row * (int64_t)R * R;
#pragma unroll
    for (int i = 0; i < RMAX; ++i)
      if (i < R) dst[i * R + lane] = (T)a[i];
  }
  if (!__all_sync(0xffffffffu, ok) && lane == 0) atomicAdd(nbad, 1ull);
}

// y_i = M_i x_i for symmetric R x R blocks M_i (R <= 32): warp per row, lane
// j accumulates column j (coalesced loads of M_i[k][j]).
template <typename T>
__global__ void __launch_bounds__(128) batched_symv_kernel(int R, int64_t nrows,
                                                           const T *__restrict__ M,
                                                           const T *__restrict__ x,
                                                           T *__restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= nrows) return;
  const T *Mr = M + row * (int64_t)R * R;
  const double xl = lane < R ? (double)__ldg(x + row * R + lane) : 0.0;
  double acc = 0.0;
#pragma unroll 8
  for (int k = 0; k < R; ++k) {
    const double xk = __shfl_sync(0xffffffffu, xl, k);
    if (lane < R) acc += (double)__ldg(Mr + k * R + lane) * xk;
  }
  if (lane < R) y[row * R + lane] = (T)acc;
}

template <typename T>
__global__ void axpby_kernel(int64_t n, double a, const T *__restrict__ x, double b,
                             const T *__restrict__ y, T *__restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = (T)(a * (double)x[k] + b * (double)y[k]);
}

template <typename T, int LPE>
static int launch_subst(const SubstParams &p, cudaStream_t s) {
  constexpr int G = 32 / LPE;
  const int64_t warps = (p.nnz + G - 1) / G;
  int64_t blocks = (warps + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  tttp_subst_kernel<T, LPE><<<(unsigned)blocks, 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("tttp_subst");
  return CPFIT_OK;
}

template <typename T, int VEC, int LPE>
static int launch_subst_vec(const SubstParams &p, cudaStream_t s) {
  const int64_t warps = (p.nnz + 31) / 32;
  int64_t blocks = (warps + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (p.order == 3)
    tttp_subst_vec_kernel<T, VEC, LPE, 3><<<(unsigned)blocks, 256, 0, s>>>(p);
  else if (p.order == 4)
    tttp_subst_vec_kernel<T, VEC, LPE, 4><<<(unsigned)blocks, 256, 0, s>>>(p);
  else
    tttp_subst_vec_kernel<T, VEC, LPE, 0><<<(unsigned)blocks, 256, 0, s>>>(p);
  CPFIT_LAUNCH_CHECK("tttp_subst_vec");
  return CPFIT_OK;
}

template <typename T, int VEC>
static int run_subst_vec(const SubstParams &p, cudaStream_t s) {
  const int nv = (p.rank + VEC - 1) / VEC;
  if (nv <= 4) return launch_subst_vec<T, VEC, 4>(p, s);
  if (nv <= 8) return launch_subst_vec<T, VEC, 8>(p, s);
  if (nv <= 16) return launch_subst_vec<T, VEC, 16>(p, s);
  return launch_subst_vec<T, VEC, 32>(p, s);
}

template <typename T>
static int run_subst(const SubstParams &p, cudaStream_t s) {
  const void *ptrs[2 * CPFIT_MAXN];
  for (int n = 0; n < p.order; ++n) {
    ptrs[2 * n] = p.fac[n];
    ptrs[2 * n + 1] = p.x[n];
  }
  const int vec = pick_vec<T>(p.rank, ptrs, 2 * p.order);
  const int maxvec = 16 / (int)sizeof(T);
  if (vec == maxvec && p.rank <= 32 * vec) return run_subst_vec<T, 16 / sizeof(T)>(p, s);
  if (vec == 1 && p.rank <= 32) return run_subst_vec<T, 1>(p, s);
  if (p.rank <= 1) return launch_subst<T, 1>(p, s);
  if (p.rank <= 2) return launch_subst<T, 2>(p, s);
  if (p.rank <= 4) return launch_subst<T, 4>(p, s);
  if (p.rank <= 8) return launch_subst<T, 8>(p, s);
  if (p.rank <= 16) return launch_subst<T, 16>(p, s);
  return launch_subst<T, 32>(p, s);
}

}  // namespace cpfit

using namespace cpfit;

extern "C" {

int cpfit_tttp_subst(cpfit_pattern *pt, int dtype, int rank, const void *w,
                     const void *const *factors, const void *const *xblocks, void *out,
                     void *stream) {
  if (!pt) { set_error("null pattern"); return CPFIT_EINVAL; }
  if (rank < 1) { set_error("rank must be >= 1"); return CPFIT_EINVAL; }
  SubstParams p{};
  p.order = pt->order;
  p.rank = rank;
  p.nnz = pt->nnz;
  for (int n = 0; n < pt->order; ++n) {
    if (!factors[n] || !xblocks[n]) {
      set_error("factor[%d] and its update block are required", n);
      return CPFIT_EINVAL;
    }
    p.idx[n] = pt->coords[n];
    p.fac[n] = factors[n];
    p.x[n] = xblocks[n];
  }
  p.w = w;
  p.out = out;
  if (pt->nnz == 0) return CPFIT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64) return run_subst<double>(p, s);
  if (dtype == CPFIT_F32) return run_subst<float>(p, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_spd_inverse_rows(int dtype, int rank, int64_t nrows, const void *gram,
                           int64_t gram_stride, double shift, void *inv_out, int64_t *nbad,
                           void *stream) {
  *nbad = 0;
  if (rank < 1 || rank > 32) { set_error("spd_inverse_rows needs 1 <= rank <= 32"); return CPFIT_EINVAL; }
  if (nrows <= 0) return CPFIT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch<unsigned long long> cnt(s);
  CPFIT_TRY(cnt.alloc(1));
  CPFIT_CUDA(cudaMemsetAsync(cnt.ptr, 0, sizeof(unsigned long long), s));
  const unsigned grid = (unsigned)((nrows + 3) / 4);
#define CPFIT_INV(T, RM)                                                                  \
  spd_inverse_kernel<T, RM><<<grid, 128, 0, s>>>(rank, nrows, (const T *)gram, gram_stride, \
                                                  shift, (T *)inv_out, cnt.ptr)
  if (dtype == CPFIT_F64) {
    if (rank <= 8) CPFIT_INV(double, 8);
    else if (rank <= 16) CPFIT_INV(double, 16);
    else CPFIT_INV(double, 32);
  } else if (dtype == CPFIT_F32) {
    if (rank <= 8) CPFIT_INV(float, 8);
    else if (rank <= 16) CPFIT_INV(float, 16);
    else CPFIT_INV(float, 32);
  } else {
    set_error("unknown dtype %d", dtype);
    return CPFIT_EINVAL;
  }
#undef CPFIT_INV
  CPFIT_LAUNCH_CHECK("spd_inverse");
  unsigned long long h = 0;
  CPFIT_CUDA(cudaMemcpyAsync(&h, cnt.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
  CPFIT_CUDA(cudaStreamSynchronize(s));
  *nbad = (int64_t)h;
  return CPFIT_OK;
}

int cpfit_batched_symv(int dtype, int rank, int64_t nrows, const void *mats, const void *x,
                       void *y, void *stream) {
  if (rank < 1 || rank > 32) { set_error("batched_symv needs 1 <= rank <= 32"); return CPFIT_EINVAL; }
  if (nrows <= 0) return CPFIT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)((nrows + 3) / 4);
  if (dtype == CPFIT_F64)
    batched_symv_kernel<double><<<grid, 128, 0, s>>>(rank, nrows, (const double *)mats,
                                                     (const double *)x, (double *)y);
  else if (dtype == CPFIT_F32)
    batched_symv_kernel<float><<<grid, 128, 0, s>>>(rank, nrows, (const float *)mats,
                                                    (const float *)x, (float *)y);
  else { set_error("unknown dtype %d", dtype); return CPFIT_EINVAL; }
  CPFIT_LAUNCH_CHECK("batched_symv");
  return CPFIT_OK;
}

int cpfit_axpby(int dtype, int64_t n, double a, const void *x, double b, const void *y,
                void *out, void *stream) {
  if (n <= 0) return CPFIT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    axpby_kernel<double><<<grid_for(n, 256, 4), 256, 0, s>>>(n, a, (const double *)x, b,
                                                             (const double *)y, (double *)out);
  else if (dtype == CPFIT_F32)
    axpby_kernel<float><<<grid_for(n, 256, 4), 256, 0, s>>>(n, a, (const float *)x, b,
                                                            (const float *)y, (float *)out);
  else { set_error("unknown dtype %d", dtype); return CPFIT_EINVAL; }
  CPFIT_LAUNCH_CHECK("axpby");
  return CPFIT_OK;
}

}  // extern "C"
