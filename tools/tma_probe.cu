// Row-gather probe (B200): how fast can factor rows be fetched into an SM by
//   (a) LDG.128 lane groups (what the sparse kernels do),
//   (b) one cp.async.bulk (UBLKCP) per row into shared memory,
//   (c) cp.async.bulk.tensor ... tile::gather4 (4 rows per TMA instruction)?
// Random row indices over an L2-resident table; reports rows/us and GB/s.
// VERDICT r1 weak #4 ("TMA tile::gather4 was never tried").
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1910_02371_b200/csrc
//      -o variants/tma_probe tools/tma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tma.cuh"

using namespace cpfit;

constexpr int WARPS = 4;
constexpr int SLOTS = 4;

__device__ __forceinline__ bool mbar_wait_bounded(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  for (int spin = 0; spin < (1 << 22); ++spin) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(a), "r"(parity) : "memory");
    if (done) return true;
  }
  return false;
}

__device__ __forceinline__ void bulk_row(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void gather4(void *dst, const CUtensorMap *m, uint64_t *bar, int c0,
                                        int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(smem_u32(dst)), "l"((uint64_t)m), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar)) : "memory");
}

// MODE 0: bulk row copies; MODE 1: gather4
template <int ROWB, int MODE>
__global__ void __launch_bounds__(WARPS * 32)
tma_rows(const char *table, const __grid_constant__ CUtensorMap tmap, const int32_t *idx,
         int64_t nbatch, unsigned long long *out, int *err) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint64_t bars[WARPS][SLOTS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char *ring = smem + (size_t)warp * SLOTS * 32 * ROWB;
  if (lane == 0)
    for (int s = 0; s < SLOTS; ++s) mbar_init(&bars[warp][s], 1);
  fence_mbar_init();
  __syncthreads();
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp, nw = (int64_t)gridDim.x * WARPS;
  unsigned long long acc = 0;
  int64_t issued = 0, done = 0;
  int32_t my = gw < nbatch ? idx[gw * 32 + lane] : 0;
  for (int64_t b = gw; b < nbatch; b += nw) {
    const int slot = (int)(issued % SLOTS);
    if (issued >= SLOTS) {  // the slot's previous batch must have landed (and is consumed here)
      if (!mbar_wait_bounded(&bars[warp][slot], (uint32_t)((done / SLOTS) & 1))) {
        if (lane == 0) atomicExch(err, 1);
        return;
      }
      acc += *reinterpret_cast<const unsigned long long *>(ring + ((size_t)slot * 32 + lane) * ROWB);
      ++done;
      __syncwarp();
    }
    const int32_t nx = b + nw < nbatch ? idx[(b + nw) * 32 + lane] : 0;
    if (lane == 0) mbar_expect_tx(&bars[warp][slot], 32 * ROWB);
    __syncwarp();
    if (MODE == 0) {
      bulk_row(ring + ((size_t)slot * 32 + lane) * ROWB, table + (size_t)my * ROWB, ROWB,
               &bars[warp][slot]);
    } else {
      const int r0 = __shfl_sync(0xffffffffu, my, (lane & 7) * 4 + 0);
      const int r1 = __shfl_sync(0xffffffffu, my, (lane & 7) * 4 + 1);
      const int r2 = __shfl_sync(0xffffffffu, my, (lane & 7) * 4 + 2);
      const int r3 = __shfl_sync(0xffffffffu, my, (lane & 7) * 4 + 3);
      if (lane < 8)
        gather4(ring + ((size_t)slot * 32 + lane * 4) * ROWB, &tmap, &bars[warp][slot], 0, r0, r1,
                r2, r3);
    }
    ++issued;
    my = nx;
  }
  while (done < issued) {
    const int slot = (int)(done % SLOTS);
    if (!mbar_wait_bounded(&bars[warp][slot], (uint32_t)((done / SLOTS) & 1))) {
      if (lane == 0) atomicExch(err, 1);
      return;
    }
    acc += *reinterpret_cast<const unsigned long long *>(ring + ((size_t)slot * 32 + lane) * ROWB);
    ++done;
  }
  if (acc == 0x1234567ull) out[0] = acc;
  // checksum of the first word of every fetched row (validates the data path)
  atomicAdd(out + 1, acc);
}

// LDG reference: 8 lanes x 16 B per 128 B row segment, 4 rows per warp instruction
template <int ROWB>
__global__ void __launch_bounds__(256) ldg_rows(const char *table, const int32_t *idx,
                                                int64_t nbatch, unsigned long long *out) {
  const int lane = threadIdx.x & 31, g = lane >> 3, q = lane & 7;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long acc = 0;
  for (int64_t b = gw; b < nbatch; b += nw) {
    const int32_t my = idx[b * 32 + lane];
#pragma unroll
    for (int s = 0; s < 8; s += 4) {
      uint4 v[4][ROWB / 128];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int row = __shfl_sync(0xffffffffu, my, (s + u) * 4 + g);
#pragma unroll
        for (int h = 0; h < ROWB / 128; ++h)
          v[u][h] = __ldg(reinterpret_cast<const uint4 *>(table + (size_t)row * ROWB + h * 128) + q);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int h = 0; h < ROWB / 128; ++h) acc += v[u][h].x ^ v[u][h].z;
    }
  }
  if (acc == 0x1234567ull) out[0] = acc;
}

template <int ROWB>
void run(int64_t rows, int64_t nrows_fetch) {
  const int64_t nbatch = nrows_fetch / 32;
  std::vector<int32_t> h(nbatch * 32);
  uint64_t st = 88172645463325252ull;
  for (auto &x : h) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    x = (int32_t)(st % (uint64_t)rows);
  }
  std::vector<unsigned long long> tab((size_t)rows * ROWB / 8);
  for (size_t i = 0; i < tab.size(); ++i) tab[i] = i * 2654435761ull;
  unsigned long long want = 0;
  for (auto x : h) want += tab[(size_t)x * ROWB / 8];
  char *table;
  int32_t *idx;
  unsigned long long *out;
  int *err;
  cudaMalloc(&table, (size_t)rows * ROWB);
  cudaMalloc(&idx, h.size() * 4);
  cudaMalloc(&out, 16);
  cudaMalloc(&err, 4);
  cudaMemcpy(table, tab.data(), (size_t)rows * ROWB, cudaMemcpyHostToDevice);
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tmap;
  const uint64_t dims[2] = {(uint64_t)ROWB / 8, (uint64_t)rows};
  const uint32_t box[2] = {(uint32_t)ROWB / 8, 1};
  const bool have_map = make_tmap(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 2, table, dims, box,
                                  CU_TENSOR_MAP_SWIZZLE_NONE);
  const size_t smem = (size_t)WARPS * SLOTS * 32 * ROWB;
  cudaFuncSetAttribute(tma_rows<ROWB, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(tma_rows<ROWB, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tma_rows<ROWB, 0>, WARPS * 32, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    if (mode == 1 && !have_map) { printf("{\"rowb\": %d, \"mode\": \"gather4\", \"error\": \"tensor map\"}\n", ROWB); continue; }
    float best = 1e30f;
    bool ok = true, bad = false;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(out, 0, 16);
      cudaMemset(err, 0, 4);
      cudaEventRecord(e0);
      if (mode == 0) tma_rows<ROWB, 0><<<148 * per_sm, WARPS * 32, smem>>>(table, tmap, idx, nbatch, out, err);
      if (mode == 1) tma_rows<ROWB, 1><<<148 * per_sm, WARPS * 32, smem>>>(table, tmap, idx, nbatch, out, err);
      if (mode == 2) ldg_rows<ROWB><<<148 * 8, 256>>>(table, idx, nbatch, out);
      cudaEventRecord(e1);
      if (cudaEventSynchronize(e1) != cudaSuccess) { ok = false; break; }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
      int herr = 0;
      unsigned long long hout[2];
      cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(hout, out, 16, cudaMemcpyDeviceToHost);
      if (herr) { ok = false; break; }
      if (mode < 2 && hout[1] != want) bad = true;
    }
    const char *names[3] = {"bulk_row", "gather4", "ldg128"};
    if (!ok)
      printf("{\"rowb\": %d, \"rows\": %lld, \"mode\": \"%s\", \"error\": \"timeout or launch failure: %s\"}\n",
             ROWB, (long long)rows, names[mode], cudaGetErrorString(cudaGetLastError()));
    else
      printf("{\"rowb\": %d, \"rows\": %lld, \"mode\": \"%s\", \"ms\": %.4f, \"rows_per_us\": %.1f, \"gbs\": %.1f, \"ctas_per_sm\": %d, \"checksum_ok\": %s}\n",
             ROWB, (long long)rows, names[mode], best, nbatch * 32 / best / 1e3,
             (double)nbatch * 32 * ROWB / best / 1e6, mode == 2 ? 8 : per_sm,
             mode == 2 ? "null" : (bad ? "false" : "true"));
    fflush(stdout);
  }
  cudaFree(table); cudaFree(idx); cudaFree(out); cudaFree(err);
}

int main() {
  run<128>(10000, 20000000);   // cfg 2: fp64 R=16 rows, 1.28 MB table, 2 rows x 1e7 nnz
  run<256>(17770, 20000000);   // cfg 3 mode-1 factor: fp64 R=32 rows, 4.5 MB table
  run<256>(480189, 20000000);  // cfg 3 mode-0 factor: 123 MB table (L2 + HBM)
  return 0;
}
