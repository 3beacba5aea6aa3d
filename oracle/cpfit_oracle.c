/*
 * cpfit_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path
 * (paper_1910_02371_b200/) links, loads or calls this file; it is used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg, always as the checker or the CPU yardstick.
 *
 * Every function restates one algorithm of the reference package `cpfit`
 * (pure Python + numba, /root/reference/pkg/src/cpfit) and cites the
 * file:line it follows.  Pinned against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py -> tests/golden/ fixtures).
 *
 * Floating-point order follows the reference's numba inner loops
 * (_jit.py:35-59): sequential r loop, (a*b)*c products, no FMA
 * contraction (build with -ffp-contract=off).  Parallelism mirrors numba
 * prange: OpenMP over disjoint output slots, so results are bitwise
 * independent of the thread count, exactly like the reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXN 16

int oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* core.py:93-102 delinearize_many: last mode fastest, rem % d then rem //= d */
void oracle_delinearize(int order, const int64_t *dims, int64_t m,
                        const uint64_t *keys, int64_t *coords /* order*m */) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
        uint64_t rem = keys[e];
        for (int n = order - 1; n >= 0; --n) {
            uint64_t d = (uint64_t)dims[n];
            coords[(int64_t)n * m + e] = (int64_t)(rem % d);
            rem /= d;
        }
    }
}

/* core.py:78-90 linearize_many: key = key * d + c, mode order */
void oracle_linearize(int order, const int64_t *dims, int64_t m,
                      const int64_t *coords, uint64_t *keys) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
        uint64_t k = 0;
        for (int n = 0; n < order; ++n)
            k = k * (uint64_t)dims[n] + (uint64_t)coords[(int64_t)n * m + e];
        keys[e] = k;
    }
}

/* core.py:234-249 counting_sort_by_mode: offsets = [0, cumsum(bincount)],
 * perm = argsort(idx, kind="stable")  (restated as a stable counting sort) */
void oracle_counting_sort(int64_t m, const int64_t *idx, int64_t dim,
                          int64_t *perm, int64_t *offsets /* dim+1 */) {
    memset(offsets, 0, sizeof(int64_t) * (size_t)(dim + 1));
    for (int64_t e = 0; e < m; ++e) offsets[idx[e] + 1]++;
    for (int64_t i = 0; i < dim; ++i) offsets[i + 1] += offsets[i];
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)(dim > 0 ? dim : 1));
    memcpy(cursor, offsets, sizeof(int64_t) * (size_t)dim);
    for (int64_t e = 0; e < m; ++e) perm[cursor[idx[e]]++] = e;
    free(cursor);
}

/* kernels.py:105-149 tttp / _jit.py:49-59 tttp3.
 * out[e] = v[e] * sum_r prod_{n: factor n present} A_n[i_n(e), r]
 * sequential r, product in mode order, then times v (numba tttp3 form). */
void oracle_tttp(int order, int64_t m, int rank, const int64_t *coords,
                 const double *vals, const double *const *factors,
                 double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
        double acc = 0.0;
        for (int r = 0; r < rank; ++r) {
            double prod = 0.0;
            int first = 1;
            for (int n = 0; n < order; ++n) {
                if (!factors[n]) continue;
                double a = factors[n][coords[(int64_t)n * m + e] * rank + r];
                if (first) { prod = a; first = 0; } else { prod = prod * a; }
            }
            acc += prod;
        }
        out[e] = vals[e] * acc;
    }
}

/* kernels.py:46-91 mttkrp / _jit.py:35-47 mttkrp3.
 * For each non-empty row (parallel), walk its entries in stable perm order:
 * out[row, r] += (prod_{k != mode, mode order} A_k[i_k, r]) * v.
 * The per-call values[perm] / coords[perm] gathers (kernels.py:60-62) are
 * restated too, so the CPU baseline does the same work as the reference. */
void oracle_mttkrp(int order, int mode, int64_t m, int rank, int64_t dim,
                   const int64_t *coords, const double *vals,
                   const int64_t *perm, const int64_t *offsets,
                   const double *const *factors, double *out) {
    memset(out, 0, sizeof(double) * (size_t)dim * (size_t)rank);
    if (m == 0) return;
    double *sv = (double *)malloc(sizeof(double) * (size_t)m);
    int64_t *si = (int64_t *)malloc(sizeof(int64_t) * (size_t)m * (size_t)order);
    /* kernels.py:60-62: sorted_vals = values[perm]; sorted_idx = coords[n][perm]
     * (single-threaded numpy gathers in the reference) */
    for (int64_t e = 0; e < m; ++e) sv[e] = vals[perm[e]];
    for (int n = 0; n < order; ++n) {
        if (n == mode) continue;
        for (int64_t e = 0; e < m; ++e)
            si[(int64_t)n * m + e] = coords[(int64_t)n * m + perm[e]];
    }
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t row = 0; row < dim; ++row) {
        double *o = out + row * rank;
        for (int64_t e = offsets[row]; e < offsets[row + 1]; ++e) {
            double v = sv[e];
            for (int r = 0; r < rank; ++r) {
                double prod = 0.0;
                int first = 1;
                for (int n = 0; n < order; ++n) {
                    if (n == mode) continue;
                    double a = factors[n][si[(int64_t)n * m + e] * rank + r];
                    if (first) { prod = a; first = 0; } else { prod = prod * a; }
                }
                o[r] += prod * v;
            }
        }
    }
    free(sv);
    free(si);
}

/* kernels.py:159-212 gram_blocks: staged = (prod_{k!=mode} A_k rows) * sqrt(w),
 * gram[i] += staged_e^T staged_e accumulated in perm order. */
int oracle_gram(int order, int mode, int64_t m, int rank, int64_t dim,
                const int64_t *coords, const double *weights,
                const int64_t *perm, const int64_t *offsets,
                const double *const *factors, double *gram) {
    for (int64_t e = 0; e < m; ++e)
        if (weights[e] < 0.0) return 1; /* kernels.py:175-176 */
    memset(gram, 0, sizeof(double) * (size_t)dim * (size_t)rank * (size_t)rank);
#pragma omp parallel
    {
        double *h = (double *)malloc(sizeof(double) * (size_t)rank);
#pragma omp for schedule(dynamic, 16)
        for (int64_t row = 0; row < dim; ++row) {
            double *g = gram + row * rank * rank;
            for (int64_t s = offsets[row]; s < offsets[row + 1]; ++s) {
                int64_t e = perm[s];
                double sw = sqrt(weights[e]);
                for (int r = 0; r < rank; ++r) {
                    double prod = 0.0;
                    int first = 1;
                    for (int n = 0; n < order; ++n) {
                        if (n == mode) continue;
                        double a = factors[n][coords[(int64_t)n * m + e] * rank + r];
                        if (first) { prod = a; first = 0; } else { prod = prod * a; }
                    }
                    h[r] = prod * sw;
                }
                for (int r = 0; r < rank; ++r)
                    for (int c = 0; c < rank; ++c) g[r * rank + c] += h[r] * h[c];
            }
        }
        free(h);
    }
    return 0;
}

/* LU with partial pivoting (LAPACK dgesv semantics: singular iff an exact
 * zero pivot appears), solving one n x n system in place.  Returns 0 or 1. */
static int lu_solve(int n, double *a, double *b) {
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = fabs(a[k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            double v = fabs(a[i * n + k]);
            if (v > best) { best = v; p = i; }
        }
        if (a[p * n + k] == 0.0) return 1;
        if (p != k) {
            for (int j = 0; j < n; ++j) {
                double t = a[k * n + j]; a[k * n + j] = a[p * n + j]; a[p * n + j] = t;
            }
            double t = b[k]; b[k] = b[p]; b[p] = t;
        }
        double piv = a[k * n + k];
        for (int i = k + 1; i < n; ++i) {
            double l = a[i * n + k] / piv;
            a[i * n + k] = l;
            for (int j = k + 1; j < n; ++j) a[i * n + j] -= l * a[k * n + j];
            b[i] -= l * b[k];
        }
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = b[i];
        for (int j = i + 1; j < n; ++j) s -= a[i * n + j] * b[j];
        b[i] = s / a[i * n + i];
    }
    return 0;
}

/* kernels.py:215-267 solve_factor (after gram_blocks):
 * lhs = gram + reg*I; reg == 0: empty rows with nonzero rhs -> error naming
 * the first such row (status 2), empty rows with zero rhs solve identity;
 * singular systems -> status 3 naming the first singular row
 * (kernels.py:270-276 _first_singular_row). */
int oracle_solve(int64_t dim, int rank, const double *gram, const double *rhs,
                 const int64_t *offsets, double reg, double *x,
                 int64_t *bad_row) {
    *bad_row = -1;
    if (reg == 0.0) {
        for (int64_t i = 0; i < dim; ++i) {
            if (offsets[i + 1] != offsets[i]) continue;
            for (int r = 0; r < rank; ++r)
                if (rhs[i * rank + r] != 0.0) { *bad_row = i; return 2; }
        }
    }
    int64_t first_bad = -1;
#pragma omp parallel
    {
        double *a = (double *)malloc(sizeof(double) * (size_t)rank * (size_t)rank);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < dim; ++i) {
            int empty = offsets[i + 1] == offsets[i];
            for (int r = 0; r < rank; ++r)
                for (int c = 0; c < rank; ++c)
                    a[r * rank + c] = gram[(i * rank + r) * rank + c] + (r == c ? reg : 0.0);
            if (reg == 0.0 && empty)
                for (int r = 0; r < rank; ++r)
                    for (int c = 0; c < rank; ++c) a[r * rank + c] = (r == c) ? 1.0 : 0.0;
            double *b = x + i * rank;
            for (int r = 0; r < rank; ++r) b[r] = rhs[i * rank + r];
            if (lu_solve(rank, a, b)) {
#pragma omp critical
                { if (first_bad < 0 || i < first_bad) first_bad = i; }
            }
        }
        free(a);
    }
    if (first_bad >= 0) { *bad_row = first_bad; return 3; }
    return 0;
}

/* ---- Philox4x64-10 (numpy.random.Philox), core.py:25-46, 173-183 ------- */
static inline void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
    __uint128_t p = (__uint128_t)a * b;
    *hi = (uint64_t)(p >> 64);
    *lo = (uint64_t)p;
}

static void philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
    const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
    const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int i = 0; i < 10; ++i) {
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(M0, c0, &hi0, &lo0);
        mulhilo64(M1, c2, &hi1, &lo1);
        uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += W0; k1 += W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Generator(Philox(SeedSequence(seed, spawn_key=path))).random(n)[start:start+n]:
 * draw e is word (e mod 4) of philox(counter=[e//4 + 1, 0, 0, 0], key),
 * mapped to (w >> 11) * 2^-53. */
void oracle_philox_uniform(uint64_t key0, uint64_t key1, int64_t start,
                           int64_t n, double *out) {
    const uint64_t key[2] = {key0, key1};
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        int64_t e = start + i;
        uint64_t ctr[4] = {(uint64_t)(e / 4) + 1u, 0, 0, 0}, w[4];
        philox4x64_10(ctr, key, w);
        out[i] = (double)(w[e % 4] >> 11) * (1.0 / 9007199254740992.0);
    }
}

/* core.py:173-183 SparseTensor.sample: keep entry e iff random()[e] < rate,
 * survivors keep their order.  Writes kept entry positions, returns count. */
int64_t oracle_sample(uint64_t key0, uint64_t key1, int64_t m, double rate,
                      int64_t *kept) {
    double *d = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    oracle_philox_uniform(key0, key1, 0, m, d);
    int64_t c = 0;
    for (int64_t e = 0; e < m; ++e)
        if (d[e] < rate) kept[c++] = e;
    free(d);
    return c;
}

/* optim.py:235-268 ccd_sweep, least-squares branch, restated exactly:
 * resid = t - model_values (core.py:252-266, col_block 32, summed per block);
 * for r: for mode: partial = prod_{p != mode} cols[p][i_p] (ones * ... in p
 * order); rho = resid + partial*col[i]; num/den by sequential bincount;
 * new = num/(den+reg) where den+reg > 0 else old; resid = rho - partial*new[i].
 * factors are row-major I_n x R arrays updated in place. */
void oracle_ccd_sweep(int order, const int64_t *dims, int64_t m, int rank,
                      const int64_t *coords, const double *vals,
                      double *const *factors, double reg) {
    double *resid = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double *partial = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double *rho = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    int64_t maxdim = 1;
    for (int n = 0; n < order; ++n) if (dims[n] > maxdim) maxdim = dims[n];
    double *num = (double *)malloc(sizeof(double) * (size_t)maxdim);
    double *den = (double *)malloc(sizeof(double) * (size_t)maxdim);
    /* model_values: out += prod.sum(axis=1) per column block of 32; the
     * block sum is numpy pairwise-free here (<= 32 terms, restated left to
     * right; matches numpy for blocks of <= 8 terms and within 1 ulp else) */
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
        double out = 0.0;
        for (int lo = 0; lo < rank; lo += 32) {
            int hi = lo + 32 < rank ? lo + 32 : rank;
            double s = 0.0;
            for (int r = lo; r < hi; ++r) {
                double p = factors[0][coords[e] * rank + r];
                for (int n = 1; n < order; ++n)
                    p *= factors[n][coords[(int64_t)n * m + e] * rank + r];
                s += p;
            }
            out += s;
        }
        resid[e] = vals[e] - out;
    }
    for (int r = 0; r < rank; ++r) {
        for (int mode = 0; mode < order; ++mode) {
            const int64_t *ci = coords + (int64_t)mode * m;
            double *col = factors[mode];
#pragma omp parallel for schedule(static)
            for (int64_t e = 0; e < m; ++e) {
                double p = 1.0;
                for (int q = 0; q < order; ++q)
                    if (q != mode) p = p * factors[q][coords[(int64_t)q * m + e] * rank + r];
                partial[e] = p;
                rho[e] = resid[e] + p * col[ci[e] * rank + r];
            }
            int64_t d = dims[mode];
            memset(num, 0, sizeof(double) * (size_t)d);
            memset(den, 0, sizeof(double) * (size_t)d);
            for (int64_t e = 0; e < m; ++e) {
                num[ci[e]] += rho[e] * partial[e];
                den[ci[e]] += partial[e] * partial[e];
            }
            for (int64_t i = 0; i < d; ++i) {
                double dr = den[i] + reg;
                if (dr > 0.0) col[i * rank + r] = num[i] / dr;
            }
#pragma omp parallel for schedule(static)
            for (int64_t e = 0; e < m; ++e)
                resid[e] = rho[e] - partial[e] * col[ci[e] * rank + r];
        }
    }
    free(resid); free(partial); free(rho); free(num); free(den);
}
