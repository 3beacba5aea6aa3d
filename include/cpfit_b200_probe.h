/*
 * cpfit_b200_probe.h -- measurement probes (not part of the reference API).
 *
 * cpfit_probe_gather: the gather ceiling of the memory system for the
 * TTTP/MTTKRP access pattern.  For e < n it reads, for each of `nrows_per`
 * index streams, the row idx[k][e] (row_bytes bytes, 16-byte vector loads,
 * row_bytes/16 lanes per row) from `table` and folds everything into one
 * checksum per lane (written to out[thread]).  No shuffles, no arithmetic
 * beyond the fold: what is left is the L1/L2 gather throughput that bounds
 * the sparse kernels.  bench.py reports the sparse kernels against it.
 *
 * cpfit_probe_l2_read: L2 -> SM read bandwidth.  `reps` coalesced passes
 * (16-byte ld.global.cg) over an L2-resident buffer of `bytes`, one folded
 * word per thread into out (out_len threads, multiple of 512).  The measured
 * GB/s is the denominator of roofline.frac_l2 (the sparse kernels' factor-row
 * gathers are served from L2).
 */
#ifndef CPFIT_B200_PROBE_H
#define CPFIT_B200_PROBE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int cpfit_probe_gather(const void *table, int row_bytes, int nrows_per,
                       const int32_t *const *idx, int64_t n, double *out,
                       int64_t out_len, void *stream);

int cpfit_probe_l2_read(const void *buf, int64_t bytes, int reps, void *out, int64_t out_len,
                        void *stream);

#ifdef __cplusplus
}
#endif

#endif /* CPFIT_B200_PROBE_H */
