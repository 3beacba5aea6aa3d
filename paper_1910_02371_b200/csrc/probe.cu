// probe.cu -- pure gather ceiling probe (see include/cpfit_b200_probe.h).
#include "../../include/cpfit_b200_probe.h"
#include "common.cuh"

namespace cpfit {

template <int LPE, int NR>
__global__ void __launch_bounds__(256, 2) probe_gather_kernel(const double2 *__restrict__ table,
                                                              int row_vecs,
                                                              const int32_t *const *idx,
                                                              int64_t n, double *out) {
  constexpr int G = 32 / LPE;
  const int lane = threadIdx.x & 31, g = lane / LPE, q = lane % LPE;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t stride = (((int64_t)gridDim.x * blockDim.x) >> 5) * 32;
  const int32_t *ix[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) ix[r] = idx[r];
  double acc = 0.0;
  for (int64_t base = warp * 32; base < n; base += stride) {
    int32_t my[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) my[r] = base + lane < n ? __ldg(ix[r] + base + lane) : 0;
#pragma unroll
    for (int s0 = 0; s0 < LPE; s0 += 4) {
      double2 x[4][NR];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const unsigned row = (unsigned)__shfl_sync(0xffffffffu, my[r], (s0 + u) * G + g);
          x[u][r] = __ldg(table + (unsigned long long)row * row_vecs + q);
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int r = 0; r < NR; ++r) acc += x[u][r].x + x[u][r].y;
    }
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// L2 read bandwidth: every thread streams 16-byte vectors of an L2-resident
// buffer (grid-stride, `reps` passes), folding them into one value per thread
// so nothing is eliminated.  Coalesced, no reuse inside a CTA: the rate is set
// by L2 -> SM delivery.
__global__ void __launch_bounds__(512) probe_l2_kernel(const uint4 *__restrict__ buf, int64_t nvec,
                                                       int reps, unsigned *out) {
  unsigned acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < nvec; i += 4 * stride) {
      uint4 a = __ldcg(buf + i), b = __ldcg(buf + i + stride), c = __ldcg(buf + i + 2 * stride),
            d = __ldcg(buf + i + 3 * stride);
      acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^
             d.z ^ d.w;
    }
    for (; i < nvec; i += stride) {
      uint4 a = __ldcg(buf + i);
      acc ^= a.x ^ a.y ^ a.z ^ a.w;
    }
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

}  // namespace cpfit

using namespace cpfit;

extern "C" int cpfit_probe_l2_read(const void *buf, int64_t bytes, int reps, void *out,
                                   int64_t out_len, void *stream) {
  if (bytes < 16 || reps < 1 || out_len < 512) {
    set_error("invalid probe_l2_read arguments");
    return CPFIT_EINVAL;
  }
  const int64_t blocks = out_len / 512;
  probe_l2_kernel<<<(unsigned)blocks, 512, 0, (cudaStream_t)stream>>>(
      (const uint4 *)buf, bytes / 16, reps, (unsigned *)out);
  CPFIT_LAUNCH_CHECK("probe_l2_read");
  return CPFIT_OK;
}

extern "C" int cpfit_probe_gather(const void *table, int row_bytes, int nrows_per,
                                  const int32_t *const *idx, int64_t n, double *out,
                                  int64_t out_len, void *stream) {
  if (row_bytes != 128 || (nrows_per != 2 && nrows_per != 3)) {
    set_error("probe supports 128-byte rows and 2 or 3 index streams");
    return CPFIT_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t blocks = out_len / 256;
  if (blocks < 1) { set_error("out_len must be >= 256"); return CPFIT_EINVAL; }
  struct Ptrs { const int32_t *p[3]; };
  const int32_t **dptr = nullptr;
  CPFIT_TRY(dalloc(&dptr, 3, s));
  const int32_t *h[3] = {idx[0], idx[1], nrows_per == 3 ? idx[2] : idx[1]};
  CPFIT_CUDA(cudaMemcpyAsync(dptr, h, sizeof(h), cudaMemcpyHostToDevice, s));
  if (nrows_per == 2)
    probe_gather_kernel<8, 2><<<(unsigned)blocks, 256, 0, s>>>((const double2 *)table, 8, dptr, n, out);
  else
    probe_gather_kernel<8, 3><<<(unsigned)blocks, 256, 0, s>>>((const double2 *)table, 8, dptr, n, out);
  CPFIT_LAUNCH_CHECK("probe_gather");
  dfree(dptr, s);
  return CPFIT_OK;
}
