/*
 * cpfit_b200.h -- C-ABI of the B200-native sparse CP-completion kernels.
 *
 * Drop-in boundary for the hot path of the reference package `cpfit`
 * (/root/reference/pkg/src/cpfit).  The reference has no native code; its
 * only compiled seam is the numba pair in _jit.py, called from kernels.py:
 *
 *   _jit.tttp3(vals, i0, i1, i2, f0, f1, f2, out)         (_jit.py:49-59,
 *                                                          kernels.py:123-128)
 *   _jit.mttkrp3(sorted_vals, idx_a, idx_b, starts, rows,  (_jit.py:35-47,
 *                fac_a, fac_b, out)                        kernels.py:66-74)
 *
 * plus the numpy/BLAS/LAPACK bodies of kernels.gram_blocks / solve_factor
 * (kernels.py:159-267), the layout caches of SparseTensor (coords(),
 * mode_group(), counting_sort_by_mode: core.py:141-157, 234-249) and
 * SparseTensor.sample (core.py:173-183).  Each entry point below names the
 * reference interface it replaces.
 *
 * Conventions: plain pointers and sizes only.  "device" pointers are CUDA
 * global-memory pointers on the current device; `stream` is a cudaStream_t
 * (NULL = legacy default stream).  Factor matrices are row-major I_n x R,
 * contiguous.  Arrays of per-mode pointers are host arrays of device pointers.
 * Every function returns CPFIT_OK (0) or an error code; cpfit_last_error()
 * gives the message of the last failure on the calling thread.  Results are
 * deterministic run to run: no floating-point atomics anywhere.
 */
#ifndef CPFIT_B200_H
#define CPFIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (the Python shim maps them onto the reference's exceptions) */
#define CPFIT_OK 0
#define CPFIT_EINVAL 1      /* ValueError: shapes, ranks, modes, ranges        */
#define CPFIT_ECUDA 2       /* CUDA runtime / launch failure                   */
#define CPFIT_ESINGULAR 3   /* NumericalError "mode m row i: singular ..."     */
#define CPFIT_EEMPTYROW 4   /* NumericalError "mode m row i: no incident ..."  */
#define CPFIT_ENEGWEIGHT 5  /* ValueError: negative normal-equation weights    */
#define CPFIT_ENONFINITE 6  /* non-finite values where finiteness is required  */
#define CPFIT_ENOMEM 7      /* device allocation failed                        */

/* value dtypes */
#define CPFIT_F64 0
#define CPFIT_F32 1

typedef struct cpfit_pattern cpfit_pattern; /* device-resident sparsity pattern */

const char *cpfit_version(void);
const char *cpfit_last_error(void);

/* ---- pattern (layout) ------------------------------------------------- */

/* Build a device pattern from sorted linearized keys (device uint64[nnz]).
 * Delinearizes on the device into int32 per-mode coordinates.
 * Replaces: SparseTensor.coords / delinearize_many (core.py:93-102,141-145). */
int cpfit_pattern_create(int order, const int64_t *dims, int64_t nnz,
                         const uint64_t *keys, void *stream,
                         cpfit_pattern **out);

/* Build a pattern from per-mode int32 coordinates already on the device and
 * already in canonical (key) order; the arrays are copied. */
int cpfit_pattern_create_coords(int order, const int64_t *dims, int64_t nnz,
                                const int32_t *const *coords, void *stream,
                                cpfit_pattern **out);

int cpfit_pattern_destroy(cpfit_pattern *p);

/* As cpfit_pattern_destroy, but stream-ordered: every buffer is released with
 * cudaFreeAsync on `stream` and the call never synchronises the device.  The
 * caller guarantees that all work using the pattern was submitted to `stream`
 * (the host mirror tracks this per pattern and falls back to
 * cpfit_pattern_destroy otherwise).  Sampled SGD patterns are created and
 * destroyed once per step (optim.py:300-330): this keeps that off the
 * device-wide synchronisation path. */
int cpfit_pattern_destroy_async(cpfit_pattern *p, void *stream);

int cpfit_pattern_info(const cpfit_pattern *p, int *order, int64_t *nnz);

/* Device pointer to the int32 coordinates of `mode` (canonical order). */
int cpfit_pattern_coords(const cpfit_pattern *p, int mode,
                         const int32_t **coords);

/* Entries per work task of the segmented kernels (default 1024).  Long
 * mode slices are split into tasks of at most this many entries and
 * combined deterministically.  Must be set before a mode layout is built. */
int cpfit_pattern_set_task_size(cpfit_pattern *p, int64_t entries);

/* Stable grouping by mode index (built once, cached in the pattern):
 * perm int32[nnz] lists entry positions grouped by mode index, stable within
 * groups; offsets int64[dims[mode]+1].  Bit-exact with
 * counting_sort_by_mode (core.py:234-249) / SparseTensor.mode_group
 * (core.py:147-157).  Device radix sort; no host round trip of entries. */
int cpfit_pattern_mode_group(cpfit_pattern *p, int mode, void *stream,
                             const int32_t **perm, const int64_t **offsets);

/* Work-table statistics of the mode layout (built on demand): number of
 * tasks, of split slices (needing the fix-up pass) and of partial slots. */
int cpfit_pattern_mode_stats(cpfit_pattern *p, int mode, void *stream,
                             int64_t *ntasks, int64_t *nsplit, int64_t *nslots);

/* out[k] = vals[perm[k]] (values into the mode-sorted order of `mode`).
 * Replaces: sorted_vals = t.values[perm] (kernels.py:60). */
int cpfit_permute_values(cpfit_pattern *p, int mode, int dtype,
                         const void *vals, void *out, void *stream);

/* ---- kernels ---------------------------------------------------------- */

/* TTTP: out[e] = vals[e] * sum_r prod_{n: factors[n] != NULL}
 *                  factors[n][coords_n[e], r].
 * Replaces: kernels.tttp (kernels.py:105-149), _jit.tttp3 (_jit.py:49-59). */
int cpfit_tttp(cpfit_pattern *p, int dtype, int rank, const void *vals,
               const void *const *factors, void *out, void *stream);

/* MTTKRP: out[i, r] = sum_{e: i_mode(e) = i} vals[e] * prod_{k != mode}
 *                       factors[k][i_k(e), r];  rows without entries are 0.
 * `vals_sorted` != 0 means `vals` is already in the mode-sorted order
 * (cpfit_permute_values), otherwise it is in canonical order.
 * Every element of `out` is stored exactly once (no zero fill followed by
 * accumulation), so `out` may be device memory or device-accessible pinned
 * host memory (the numpy binding passes its result buffer).
 * Replaces: kernels.mttkrp (kernels.py:46-91), _jit.mttkrp3 (_jit.py:35-47). */
int cpfit_mttkrp(cpfit_pattern *p, int mode, int dtype, int rank,
                 const void *vals, int vals_sorted,
                 const void *const *factors, void *out, void *stream);

/* Per-row Gram blocks G_i = sum_{e in row i} w_e h_e h_e^T with
 * h_e = prod_{k != mode} factors[k][i_k(e), :]  (weights NULL = unit mask).
 * Writes gram_out[dims[mode] * rank * rank].  Negative weights ->
 * CPFIT_ENEGWEIGHT.  Replaces: kernels.gram_blocks (kernels.py:159-212). */
int cpfit_gram(cpfit_pattern *p, int mode, int dtype, int rank,
               const void *weights, int weights_sorted,
               const void *const *factors, void *gram_out, void *stream);

/* Per-row regularised normal equations (G_i + reg I) x_i = rhs_i with the
 * reference's empty-row and singular-row semantics; *bad_row receives the
 * offending row on CPFIT_EEMPTYROW / CPFIT_ESINGULAR.  gram_out (nullable)
 * receives G.  Replaces: kernels.solve_factor (kernels.py:215-267). */
int cpfit_solve_factor(cpfit_pattern *p, int mode, int dtype, int rank,
                       const void *weights, int weights_sorted,
                       const void *const *factors, const void *rhs,
                       double reg, void *x_out, void *gram_out,
                       int64_t *bad_row, void *stream);

/* One least-squares ALS mode update with the right-hand side fused into the
 * Gram pass: rhs_i = sum_{e in row i} vals[e] h_e (the MTTKRP of `vals`,
 * same h_e as the Gram), then (G_i + reg I) x_i = rhs_i with
 * cpfit_solve_factor's semantics and error order.  The factor rows are
 * gathered once per entry instead of twice.  vals_sorted as in cpfit_mttkrp;
 * gram_out / rhs_out nullable.  Replaces the pair kernels.mttkrp +
 * kernels.solve_factor in the ALS sweep (optim.py:214-228). */
int cpfit_als_update(cpfit_pattern *p, int mode, int dtype, int rank,
                     const void *vals, int vals_sorted,
                     const void *const *factors, double reg, void *x_out,
                     void *gram_out, void *rhs_out, int64_t *bad_row,
                     void *stream);

/* Gram-free normal-equations product of one ALS mode (BASELINE cfg 3 "ALS
 * completion with implicit CG"; the reference solves each row with LAPACK,
 * kernels.py:259, and has no counterpart):
 *   out[i, :] = sum_{e in row i} w_e h_e (h_e . x[i, :]),
 *   h_e = prod_{k != mode} factors[k][i_k(e), :]   (kernels.py:196-204),
 * i.e. G_i x_i without materialising the I x R x R blocks of
 * kernels.gram_blocks.  weights nullable (unit weights: the observation
 * mask); weights_sorted as in cpfit_mttkrp.  row_active (nullable, int32 per
 * row of the mode): rows with 0 are skipped and their output row is 0. */
int cpfit_gram_matvec(cpfit_pattern *p, int mode, int dtype, int rank,
                      const void *weights, int weights_sorted,
                      const void *const *factors, const void *x,
                      const int32_t *row_active, void *out, void *stream);

/* Per-row CG recurrences for (G_i + reg I) x_i = b_i, every row with its own
 * alpha / beta (the systems are independent), in the form of pcg_solve
 * (optim.py:493-533) applied per row: stop a row when ||r_i|| <= tol ||b_i||
 * or on nonpositive curvature.  All arrays are device memory: b, x, r, p
 * nrows x rank of `dtype`; rho, thresh2 double[nrows]; active int32[nrows];
 * status int64[2] = {rows still active after the call, sticky non-finite flag}.
 * init: r = b - (ax + reg x) (ax = G x0 from cpfit_gram_matvec, or NULL for
 * x0 = 0 -- x is then not read), p = r; rows with b_i = 0 get x_i = 0.
 * step: q = G p from cpfit_gram_matvec(..., p, active, ...); updates x, r, p,
 * rho and active in place. */
int cpfit_cg_rows_init(int dtype, int64_t nrows, int rank, double reg, double tol,
                       const void *b, const void *ax, void *x, void *r, void *p,
                       double *rho, double *thresh2, int32_t *active,
                       int64_t *status, void *stream);
int cpfit_cg_rows_step(int dtype, int64_t nrows, int rank, double reg,
                       const void *q, void *x, void *r, void *p, double *rho,
                       const double *thresh2, int32_t *active, int64_t *status,
                       void *stream);

/* TTTP whose result is also delivered to HOST memory (the reference's
 * numpy-returning tttp, kernels.py:105-149): the nonzeros are processed in
 * chunks (chunk <= 0: nnz/8, at most 16 chunks) and each chunk is copied
 * into host_out (pinned memory for an asynchronous DMA) while the next one
 * computes.  dev_out receives the device copy.  Asynchronous on `stream`:
 * host_out is complete once `stream` is synchronised. */
int cpfit_tttp_host(cpfit_pattern *p, int dtype, int rank, const void *vals,
                    const void *const *factors, void *dev_out, void *host_out,
                    int64_t chunk, void *stream);

/* As cpfit_tttp_host, but `stream` is not joined to the copies: it runs on
 * while the device->host transfers drain, and *done receives an event that
 * completes when host_out is filled.  The caller must pass it to
 * cpfit_event_wait (destroy = 1) exactly once, and keep dev_out / host_out
 * alive until then. */
int cpfit_tttp_host_async(cpfit_pattern *p, int dtype, int rank, const void *vals,
                          const void *const *factors, void *dev_out,
                          void *host_out, int64_t chunk, void **done, void *stream);
int cpfit_event_wait(void *event, int destroy);

/* Device -> pinned (device-mapped) host copy done by a kernel: the PCIe
 * writes come from the SMs, so a small result is not queued behind a large
 * transfer left running on the copy engine.  Stream-ordered on `stream`. */
int cpfit_copy_to_host(int64_t nbytes, const void *src, void *host_dst, void *stream);

/* TTTP with an affine epilogue: out[e] = alpha * m_e + beta * vals[e], with
 * m_e = sum_r prod_n factors[n][i_n(e), r].  alpha = 2, beta = -2 gives the
 * least-squares derivative tensor 2(m - t) (losses.py:41-48, model via
 * model_at_observed = TTTP on the unit mask, losses.py:107-114); alpha = -1,
 * beta = 1 the residual t - m (optim.py:250, 642-652). */
int cpfit_tttp_axpby(cpfit_pattern *p, int dtype, int rank, const void *vals,
                     const void *const *factors, double alpha, double beta,
                     void *out, void *stream);

/* ---- second-order step (optim.py:348-598, gn_step / hessian_matvec) ---- */

/* out[e] = w[e] * sum_d sum_r x_d[i_d(e), r] * prod_{p != d} factors[p][i_p(e), r]:
 * the sum over d of the TTTPs with slot d substituted by its update block
 * (hessian_matvec's z, optim.py:372-376), one gather of the 2N rows per
 * entry.  w nullable (unit weights); every factor and block is required. */
int cpfit_tttp_subst(cpfit_pattern *p, int dtype, int rank, const void *w,
                     const void *const *factors, const void *const *xblocks,
                     void *out, void *stream);

/* Block-diagonal preconditioner of the second-order step (optim.py:467-487),
 * inverted once per step: inv_out[i] = (gram[i] + shift I)^{-1} for rank <= 32
 * (warp Gauss-Jordan on the SPD blocks).  *nbad = rows whose pivots were not
 * positive (then the caller solves that mode with cpfit_solve_rows, whose
 * LU fallback reports singular systems like np.linalg.solve).  Synchronous. */
int cpfit_spd_inverse_rows(int dtype, int rank, int64_t nrows, const void *gram,
                           int64_t gram_stride, double shift, void *inv_out,
                           int64_t *nbad, void *stream);

/* y[i] = mats[i] x[i] for symmetric rank x rank blocks (rank <= 32). */
int cpfit_batched_symv(int dtype, int rank, int64_t nrows, const void *mats,
                       const void *x, void *y, void *stream);

/* out[k] = a * x[k] + b * y[k] (PCG vector updates, optim.py:513-531). */
int cpfit_axpby(int dtype, int64_t n, double a, const void *x, double b,
                const void *y, void *out, void *stream);

/* ---- sampling (SparseTensor.sample, core.py:173-183) ------------------ */

/* Keep entry e iff u_e < rate where u_e is draw (counter_offset + e) of
 * numpy Generator(Philox(key)).random() -- bit-exact Philox4x64-10, so a
 * shard with counter_offset = its first global entry reproduces the
 * single-device sample.  *out is a new pattern holding the survivors in
 * order; cpfit_pattern_parent_index gives their positions in `src`. */
int cpfit_sample(cpfit_pattern *src, uint64_t key0, uint64_t key1,
                 int64_t counter_offset, double rate, void *stream,
                 cpfit_pattern **out);

int cpfit_pattern_parent_index(const cpfit_pattern *p, const int32_t **idx);

/* out[k] = in[idx[k]], k < n (values of sampled / permuted entries). */
int cpfit_gather_values(int dtype, int64_t n, const int32_t *idx,
                        const void *in, void *out, void *stream);

/* ---- reductions and updates ------------------------------------------- */

/* Deterministic (fixed-order) reductions in fp64, result copied to the host:
 * op 0: sum x^2;  op 1: sum (x - y)^2;  op 2: sum x*y;  op 3: sum x.
 * Serves objective / rmse (losses.py:126-150, optim.py:642-652). */
int cpfit_reduce(int op, int dtype, int64_t n, const void *x, const void *y,
                 double *result, void *stream);

/* Device-side factor validation (validation.py:47-59): *flag (a DEVICE int,
 * zeroed by the caller) is OR-ed with 1 if any of the n elements is NaN or
 * infinite.  Asynchronous: read the flag after synchronising the stream. */
int cpfit_check_finite(int dtype, int64_t n, const void *x, int *flag, void *stream);

/* SGD step out = (a - step*grad) - shrink*a in numpy's evaluation order
 * (optim.py:313-330); *nonfinite = 1 if any result is not finite. */
int cpfit_sgd_update(int dtype, int64_t n, const void *a, const void *grad,
                     double step, double shrink, void *out, int *nonfinite,
                     void *stream);

/* CCD++ (least squares, optim.py:235-268 column-then-mode order).  The
 * device keeps rhat = the residual with the current rank-one column r added
 * back: in exact arithmetic it is the `rho` of every mode update of column r
 * (optim.py:254), so no per-mode residual pass is needed.  Each mode n keeps
 * its own copy rhat_n in its mode-sorted order (mode 0: canonical order);
 * start with rhat_n = (t - model) permuted (cpfit_permute_values).  A sweep
 * is, per column r, for n = 0..N-1:
 *   cpfit_ccd_step(n, rhat_n, rhat_sorted = 1, fold_sub = new column r-1
 *                  (NULL for r = 0), fold_add = column r as it was before
 *                  this sweep touched it)
 * and after the last column cpfit_ccd_fold(mode 0, sub = column R-1, add =
 * NULL) on rhat_0 leaves the residual t - model in canonical order.
 *
 * cpfit_ccd_step: cols[q] = column r of factor q (contiguous fp64, length
 * dims[q]); modes q > `mode` must not have been updated yet in this column
 * (fold_add[q] == cols[q] there, which the pass relies on).  With fold_sub / fold_add, rhat is first replaced by
 * (rhat - prod fold_sub) + prod fold_add at every entry (needs rhat_sorted
 * or an identity-order mode) and written back.  rhat_sorted = 0: a
 * canonical rhat read through the mode permutation, not folded.
 * numden == NULL: cols[mode] is updated in place, new_i = num_i / (den_i +
 * reg), the old value kept where den_i + reg <= 0 (optim.py:260-263), with
 * num_i = sum rhat_e partial_e, den_i = sum partial_e^2 over row i.
 * numden != NULL (distributed: nonzeros sharded, one all-reduce
 * per (r, mode)): writes numden[i] = num_i, numden[dims[mode] + i] = den_i
 * (zero for rows without local entries) and leaves cols untouched; after
 * the caller sums numden over ranks, cpfit_ccd_finalize applies the update
 * rule to the column.  One rank reproduces the fused path bit for bit.
 * cpfit_ccd_fold: the fold alone on a copy in mode `mode`'s sorted order
 * (mode = -1: canonical order). */
int cpfit_ccd_step(cpfit_pattern *p, int mode, double *const *cols, double *rhat,
                   int rhat_sorted, const double *const *fold_sub,
                   const double *const *fold_add, double reg, double *numden,
                   void *stream);
int cpfit_ccd_fold(cpfit_pattern *p, int mode, const double *const *sub,
                   const double *const *add, double *rhat, void *stream);
int cpfit_ccd_finalize(int64_t dim, const double *numden, double reg,
                       double *col, void *stream);

/* ---- ingest -------------------------------------- */
/* from_coords on the device (core.py:78-90, 208-231): coords[q] = n device
 * coordinates of mode q (int32 if coord_bytes == 4, int64 if 8), vals = n
 * fp64 values, any order, duplicates allowed.  Writes the strictly
 * increasing unique linearized keys (row-major, last mode fastest) to
 * keys_out and their values to vals_out (duplicates summed exactly as
 * np.add.reduceat does in stable key order: bit-identical), *nnz_out = the
 * unique count (both outputs need room for n).  A coordinate outside
 * [0, dims[q]) returns CPFIT_EINVAL with *bad_mode = the lowest such mode
 * (the reference's ValueError "coordinate out of range [0, d) in mode q"). */
int cpfit_from_coords(int order, const int64_t *dims, int64_t n, int coord_bytes,
                      const void *const *coords, const double *vals,
                      uint64_t *keys_out, double *vals_out, int64_t *nnz_out,
                      int *bad_mode, void *stream);

/* ---- pairwise (hypersparse) baseline, hypersparse.py */
/* CCSR x dense: payload[slot, :] = sum_j values[j] * dense[col_ids[j], :]
 * over slot's entries, per column in np.add.reduceat's order along the entry
 * axis (first product + numpy's pairwise sum of the rest). */
int cpfit_ccsr_spmm(int64_t nrows, const int64_t *row_offsets, const int64_t *col_ids,
                    const double *values, const double *dense, int rank,
                    double *payload, void *stream);
/* pairwise TTTP: out[e] = row sum over r (numpy's order) of
 * ((values[e] * F0[i0(e), r]) * F1[i1(e), r]) ...; idx[n] = int32 device
 * coordinates of the n-th provided factor's mode; R <= 256. */
int cpfit_pairwise_tttp(int64_t nnz, int nfac, int rank, const int32_t *const *idx,
                        const double *const *factors, const double *values,
                        double *out, void *stream);
/* pairwise MTTKRP tail: w[f, r] = payload[f, r] * prod_n factors[n][idx[n][f], r],
 * out[i, r] = 0.0 + sum of w over fibers with target[f] = i in fiber order
 * (np.bincount); out is dim x rank. */
int cpfit_pairwise_fold_sum(int64_t nfibers, int rank, int nfold, const int32_t *const *idx,
                            const double *const *factors, const double *payload,
                            const int32_t *target, int64_t dim, double *out, void *stream);

/* ---- generalized losses (losses.py:22-104) ---------------------------- */
/* Loss ids: 0 = least squares (phi = (t - m)^2, dphi = 2 (m - t), d2phi = 2),
 * 1 = Poisson log link (phi = exp(m~) - t m, dphi = exp(m~) - t, d2phi =
 * exp(m~), m~ = min(m, 50): POISSON_EXP_CLAMP, losses.py:19-91).  *clamped
 * (host, nullable) receives the number of entries with m > 50 (the
 * reference's diagnostics["exp_clamped"] counts one per entry per exp call).
 *
 * cpfit_tttp_loss: the derivative tensors at the model of `factors` on the
 * pattern (model_at_observed + derivative_tensors, losses.py:107-123) in one
 * pass: TTTP with the loss epilogue, dphi / d2phi written in canonical order.
 * cpfit_loss_eval: elementwise phi / dphi / d2phi (outputs nullable). */
int cpfit_tttp_loss(cpfit_pattern *p, int dtype, int rank, const void *t_vals,
                    const void *const *factors, int loss, void *dphi, void *d2phi,
                    int64_t *clamped, void *stream);
int cpfit_loss_eval(int loss, int dtype, int64_t n, const void *t, const void *m,
                    void *phi, void *dphi, void *d2phi, int64_t *clamped,
                    void *stream);

/* Inner-Newton CCD++ column step for generalized losses (optim.py:269-294),
 * fp64, canonical entry order.  cpfit_ccd_gen_weights: part_e = prod_{p !=
 * mode} cols[p][i_p(e)], w1 = part * dphi(t, model), w2 = part^2 * d2phi
 * (loss 2: a user-registered loss whose dphi / d2phi the caller evaluated
 * on the host -- passed in place of t / model);
 * the row sums num / den come from cpfit_mttkrp (R = 1, unit columns);
 * cpfit_ccd_gen_update: delta = -(num + 2 reg col) / (den + 2 reg) where the
 * denominator is > 0, else 0, col += delta; cpfit_ccd_gen_model:
 * model_e += part_e * delta[i_mode(e)]. */
int cpfit_ccd_gen_weights(cpfit_pattern *p, int mode, int loss,
                          const double *const *cols, const double *t,
                          const double *model, double *w1, double *w2,
                          double *part, int64_t *clamped, void *stream);
int cpfit_ccd_gen_update(int64_t dim, const double *num, const double *den,
                         double reg, double *col, double *delta, void *stream);
int cpfit_ccd_gen_model(cpfit_pattern *p, int mode, const double *part,
                        const double *delta, double *model, void *stream);

/* Batched regularised SPD solves without a tensor pattern:
 * (G_i + reg I) x_i = rhs_i for i < nrows, G_i = gram + i * gram_stride
 * (gram_stride 0: one shared G, e.g. the dense CP-ALS Gram (B^T B)*(C^T C)).
 * Same kernels and singular-row semantics as cpfit_solve_factor. */
int cpfit_solve_rows(int dtype, int rank, int64_t nrows, const void *gram,
                     int64_t gram_stride, const void *rhs, double reg,
                     void *x_out, int64_t *bad_row, void *stream);

/* ---- dense tensors (BASELINE cfg 4; no reference counterpart: its oracle
 * is kernels.mttkrp on a fully observed tensor, kernels.py:46-91) -------- */

/* axis 1: out[i, r] = sum_j T[i, j, r] W[j, r]   (out I x R)
 * axis 0: out[j, r] = sum_i T[i, j, r] W[i, r]   (out J x R)
 * Epilogue of the dense MTTKRP after the plain GEMM T = X_(IJ x K) C. */
int cpfit_dense_reduce(int dtype, int64_t I, int64_t J, int rank, const void *T,
                       const void *W, int axis, void *out, void *stream);

/* out[(i*J + j), r] = A[i, r] * B[j, r]  (Khatri-Rao product, IJ x R). */
int cpfit_khatri_rao(int dtype, int64_t I, int64_t J, int rank, const void *A,
                     const void *B, void *out, void *stream);

/* Dense MTTKRP of an order-3 row-major tensor X (I x J x K), one pass over X
 * with the Khatri-Rao operand formed in shared memory (csrc/dense_dmma.cu,
 * csrc/dense_tc.cu):
 *   mode 0: out[i, r] = sum_jk X[i,j,k] B[j,r] C[k,r]   (einsum('ijk,jr,kr->ir'))
 *   mode 1: out[j, r] = sum_ik X[i,j,k] A[i,r] C[k,r]
 *   mode 2: out[k, r] = sum_ij X[i,j,k] A[i,r] B[j,r]
 * Replaces kernels.mttkrp on a fully observed tensor (kernels.py:46-91; the
 * reference has no dense type).  F64: FP64 DMMA (parity path);
 * F32: TF32 tcgen05.mma with TMEM accumulators (TF32 accuracy class).
 * Factors are row-major (dim x rank); the factor of `mode` may be NULL. */
int cpfit_dense_mttkrp(int dtype, int64_t I, int64_t J, int64_t K, int rank,
                       const void *X, const void *A, const void *B, const void *C,
                       int mode, void *out, void *stream);

/* T[(i*J + j), r] = sum_k X[i,j,k] C[k,r]: the GEMM a dense CP-ALS sweep
 * shares between modes 0 and 1 (epilogues: cpfit_dense_reduce). */
int cpfit_dense_xc(int dtype, int64_t I, int64_t J, int64_t K, int rank, const void *X,
                   const void *C, void *T, void *stream);

/* G[a, b] = prod_f sum_i F_f[i, a] F_f[i, b]: the Hadamard product of the
 * factors' Gramians, i.e. the shared normal-equation matrix of a dense
 * CP-ALS mode update (optim.py:192-206 with every entry observed). */
int cpfit_dense_gram(int dtype, int nfactors, const int64_t *rows, int rank,
                     const void *const *factors, void *G, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* CPFIT_B200_H */
