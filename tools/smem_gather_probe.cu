// Gather-path probe (B200): does moving ONE of MTTKRP's two factor-row gathers
// from the L1tex path (LDG.128 lane groups, ~2 cycles per 128-B line per SM)
// to shared memory (LDS.128 from a staged row block) lift the gather ceiling?
//   mode 0: both rows by LDG from L2-resident tables (what mttkrp_kernel does)
//   mode 1: row A by LDG, row B by LDS from a block of BROWS rows staged in smem
//   mode 2: both rows by LDS (upper bound of the shared-memory path)
// 1e7 entries, fp64 R=16 (128-B rows), indices uniform.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o variants/smem_gather_probe tools/smem_gather_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cstring>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

constexpr int R = 16;          // doubles per row
constexpr int LPE = 8;         // lanes per entry (8 x 16 B = 128 B)

template <int MODE, int THREADS>
__global__ void __launch_bounds__(THREADS)
probe(const double *__restrict__ A, const double *__restrict__ B, const int32_t *__restrict__ ia,
      const int32_t *__restrict__ ib, int64_t nnz, int brows, double *out) {
  extern __shared__ __align__(16) double sB[];
  if (MODE >= 1) {
    const double2 *src = reinterpret_cast<const double2 *>(B);
    double2 *dst = reinterpret_cast<double2 *>(sB);
    for (int i = threadIdx.x; i < brows * R / 2; i += THREADS) dst[i] = src[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, l8 = lane & 7, q = lane >> 3;
  const int64_t nbatch = nnz / 32;
  const int64_t per = (nbatch + gridDim.x - 1) / gridDim.x;   // contiguous range per CTA
  const int64_t b0 = (int64_t)blockIdx.x * per, b1 = b0 + per < nbatch ? b0 + per : nbatch;
  double2 acc = make_double2(0.0, 0.0);
  const int warp = threadIdx.x >> 5, nwarp = THREADS / 32;
  int64_t b = b0 + warp;
  int32_t ja = 0, jb = 0;
  if (b < b1) { ja = ia[b * 32 + lane]; jb = ib[b * 32 + lane]; }
  for (; b < b1; b += nwarp) {
    int32_t na = 0, nb = 0;
    if (b + nwarp < b1) { na = ia[(b + nwarp) * 32 + lane]; nb = ib[(b + nwarp) * 32 + lane]; }
#pragma unroll
    for (int g = 0; g < 8; g += 4) {
      double2 va[4], vb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int src = 4 * (g + u) + q;
        const int32_t ra = __shfl_sync(0xffffffffu, ja, src);
        const int32_t rb = __shfl_sync(0xffffffffu, jb, src);
        if (MODE == 2)
          va[u] = *reinterpret_cast<const double2 *>(sB + (size_t)(ra & (brows - 1)) * R + 2 * l8);
        else
          va[u] = *reinterpret_cast<const double2 *>(A + (size_t)ra * R + 2 * l8);
        if (MODE >= 1)
          vb[u] = *reinterpret_cast<const double2 *>(sB + (size_t)rb * R + 2 * l8);
        else
          vb[u] = *reinterpret_cast<const double2 *>(B + (size_t)rb * R + 2 * l8);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x = fma(va[u].x, vb[u].x, acc.x);
        acc.y = fma(va[u].y, vb[u].y, acc.y);
      }
    }
    ja = na; jb = nb;
  }
  out[(size_t)blockIdx.x * THREADS + threadIdx.x] = acc.x + acc.y;
}

template <int MODE, int THREADS>
static void run(const char *name, int grid, size_t smem, const double *A, const double *B,
                const int32_t *ia, const int32_t *ib, int64_t nnz, int brows, double *out) {
  CK(cudaFuncSetAttribute(probe<MODE, THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float best = 1e9f;
  for (int it = 0; it < 8; ++it) {
    CK(cudaEventRecord(e0));
    probe<MODE, THREADS><<<grid, THREADS, smem>>>(A, B, ia, ib, nnz, brows, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (it >= 2 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  printf("%-44s grid %4d x %4d smem %6zu B: %.4f ms  (%.2f G entries/s, %.2f clk/entry/SM at 1.965 GHz)\n",
         name, grid, THREADS, smem, best, nnz / best * 1e-6, best * 1e-3 * 1.965e9 * 148 / nnz);
}


// MTTKRP-shaped probe: what do the value stream, the per-entry value shuffle
// and the task structure (persistent warps over TL-entry tasks, cross-group
// reduction + one 128-B row store per task) add to the pure gather time?
//   FEAT 0: gathers only, grid-stride batches     FEAT 1: + values
//   FEAT 2: + tasks (warp-strided)                FEAT 3: tasks, U = 8 (all 32 entries' rows in flight)
template <int FEAT, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
probe_task(const double *__restrict__ A, const double *__restrict__ B, const int32_t *__restrict__ ia,
           const int32_t *__restrict__ ib, const double *__restrict__ vals, int64_t nnz, int TL,
           double *out) {
  constexpr int U = FEAT == 3 ? 8 : 4;
  const int lane = threadIdx.x & 31, l8 = lane & 7, q = lane >> 3;
  const int64_t warp = ((int64_t)blockIdx.x * THREADS + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * THREADS) >> 5;
  const int64_t ntasks = FEAT >= 2 ? (nnz + TL - 1) / TL : nwarps;
  double2 keep = make_double2(0.0, 0.0);
  for (int64_t t = warp; t < ntasks; t += nwarps) {
    int64_t b0, b1, step;
    if (FEAT >= 2) { b0 = t * TL; b1 = b0 + TL < nnz ? b0 + TL : nnz; step = 32; }
    else { b0 = t * 32; b1 = nnz; step = nwarps * 32; }
    double2 acc = make_double2(0.0, 0.0);
    int32_t ja = 0, jb = 0; double v = 0.0;
    if (b0 + lane < b1) { ja = ia[b0 + lane]; jb = ib[b0 + lane]; if (FEAT >= 1) v = vals[b0 + lane]; }
    for (int64_t base = b0; base < b1; base += step) {
      int32_t na = 0, nb = 0; double nv = 0.0;
      if (base + step + lane < b1) {
        na = ia[base + step + lane]; nb = ib[base + step + lane];
        if (FEAT >= 1) nv = vals[base + step + lane];
      }
      const int cnt = (int)(b1 - base < 32 ? b1 - base : 32);
#pragma unroll
      for (int g = 0; g < 8; g += U) {
        if (FEAT >= 2 && g * 4 >= cnt) break;
        double2 va[U], vb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int src = 4 * (g + u) + q;
          const int32_t ra = __shfl_sync(0xffffffffu, ja, src);
          const int32_t rb = __shfl_sync(0xffffffffu, jb, src);
          va[u] = *reinterpret_cast<const double2 *>(A + (size_t)ra * R + 2 * l8);
          vb[u] = *reinterpret_cast<const double2 *>(B + (size_t)rb * R + 2 * l8);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (FEAT >= 1) {
            const double w = __shfl_sync(0xffffffffu, v, 4 * (g + u) + q);
            acc.x += (va[u].x * vb[u].x) * w;
            acc.y += (va[u].y * vb[u].y) * w;
          } else {
            acc.x = fma(va[u].x, vb[u].x, acc.x);
            acc.y = fma(va[u].y, vb[u].y, acc.y);
          }
        }
      }
      ja = na; jb = nb; v = nv;
    }
    if (FEAT >= 2) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 8);  acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 8);
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16); acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
      if (q == 0) *reinterpret_cast<double2 *>(out + t * R + 2 * l8) = acc;
    } else {
      keep.x += acc.x; keep.y += acc.y;
    }
  }
  if (FEAT < 2) out[(size_t)blockIdx.x * THREADS + threadIdx.x] = keep.x + keep.y;
}

template <int FEAT, int THREADS, int MINB>
static void run_task(const char *name, const double *A, const double *B, const int32_t *ia,
                     const int32_t *ib, const double *vals, int64_t nnz, int TL, double *out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float best = 1e9f;
  const int grid = 148 * MINB;
  for (int it = 0; it < 8; ++it) {
    CK(cudaEventRecord(e0));
    probe_task<FEAT, THREADS, MINB><<<grid, THREADS>>>(A, B, ia, ib, vals, nnz, TL, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (it >= 2 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  printf("%-52s %d x %d thr/SM TL %4d: %.4f ms (%.2f clk/entry/SM)\n", name, MINB, THREADS, TL, best,
         best * 1e-3 * 1.965e9 * 148 / nnz);
}


// No-shuffle variants: the 8 lanes of a group load their entry's scalars
// themselves (same address within the group: one wavefront per instruction)
//   REC 0: int2 index pairs (LDG.64) + values (LDG.64)
//   REC 1: 16-byte records {ia, ib, value} (one LDG.128)
template <int REC, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
probe_rec(const double *__restrict__ A, const double *__restrict__ B, const int2 *__restrict__ iab,
          const double *__restrict__ vals, const int4 *__restrict__ rec, int64_t nnz, int TL,
          double *out) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31, l8 = lane & 7, q = lane >> 3;
  const int64_t warp = ((int64_t)blockIdx.x * THREADS + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * THREADS) >> 5;
  const int64_t ntasks = (nnz + TL - 1) / TL;
  for (int64_t t = warp; t < ntasks; t += nwarps) {
    const int64_t b0 = t * TL, b1 = b0 + TL < nnz ? b0 + TL : nnz;
    double2 acc = make_double2(0.0, 0.0);
    // scalars of round 0
    int2 ix[U]; double w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = b0 + 4 * u + q;
      if (REC == 0) {
        ix[u] = e < b1 ? iab[e] : make_int2(0, 0);
        w[u] = e < b1 ? vals[e] : 0.0;
      } else {
        int4 r4 = e < b1 ? rec[e] : make_int4(0, 0, 0, 0);
        ix[u] = make_int2(r4.x, r4.y);
        w[u] = __hiloint2double(r4.w, r4.z);
      }
    }
    for (int64_t base = b0; base < b1; base += 4 * U) {
      double2 va[U], vb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        va[u] = *reinterpret_cast<const double2 *>(A + (size_t)ix[u].x * R + 2 * l8);
        vb[u] = *reinterpret_cast<const double2 *>(B + (size_t)ix[u].y * R + 2 * l8);
      }
      double wc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) wc[u] = w[u];
#pragma unroll
      for (int u = 0; u < U; ++u) {   // next round's scalars
        const int64_t e = base + 4 * U + 4 * u + q;
        if (REC == 0) {
          ix[u] = e < b1 ? iab[e] : make_int2(0, 0);
          w[u] = e < b1 ? vals[e] : 0.0;
        } else {
          int4 r4 = e < b1 ? rec[e] : make_int4(0, 0, 0, 0);
          ix[u] = make_int2(r4.x, r4.y);
          w[u] = __hiloint2double(r4.w, r4.z);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc.x += (va[u].x * vb[u].x) * wc[u];
        acc.y += (va[u].y * vb[u].y) * wc[u];
      }
    }
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 8);  acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 8);
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16); acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
    if (q == 0) *reinterpret_cast<double2 *>(out + t * R + 2 * l8) = acc;
  }
}

template <int REC, int THREADS, int MINB>
static void run_rec(const char *name, const double *A, const double *B, const int2 *iab,
                    const double *vals, const int4 *rec, int64_t nnz, int TL, double *out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float best = 1e9f;
  const int grid = 148 * MINB;
  for (int it = 0; it < 8; ++it) {
    CK(cudaEventRecord(e0));
    probe_rec<REC, THREADS, MINB><<<grid, THREADS>>>(A, B, iab, vals, rec, nnz, TL, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (it >= 2 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  printf("%-52s %d x %d thr/SM TL %4d: %.4f ms (%.2f clk/entry/SM)\n", name, MINB, THREADS, TL, best,
         best * 1e-3 * 1.965e9 * 148 / nnz);
}

static void task_suite() {
  const int64_t nnz = 10000000;
  const int rows = 10000;
  std::vector<int32_t> ha(nnz), hb(nnz);
  std::vector<double> hv(nnz), hA((size_t)rows * R), hB((size_t)rows * R);
  uint64_t s = 88172645463325252ull;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
  for (int64_t e = 0; e < nnz; ++e) { ha[e] = (int32_t)(rnd() % rows); hb[e] = (int32_t)(rnd() % rows); hv[e] = (double)(rnd() % 7); }
  for (auto &x : hA) x = (double)(rnd() % 1000) * 1e-3;
  for (auto &x : hB) x = (double)(rnd() % 1000) * 1e-3;
  double *A, *B, *out, *vals; int32_t *ia, *ib;
  CK(cudaMalloc(&A, hA.size() * 8)); CK(cudaMalloc(&B, hB.size() * 8));
  CK(cudaMalloc(&ia, nnz * 4)); CK(cudaMalloc(&ib, nnz * 4)); CK(cudaMalloc(&vals, nnz * 8));
  CK(cudaMalloc(&out, (nnz / 64 + 148 * 2048) * R * 8));
  CK(cudaMemcpy(A, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B, hB.data(), hB.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ia, ha.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ib, hb.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(vals, hv.data(), nnz * 8, cudaMemcpyHostToDevice));
  printf("== MTTKRP-shaped probe (two 10k-row tables in L2, 1e7 entries) ==\n");
  run_task<0, 256, 4>("gathers only", A, B, ia, ib, vals, nnz, 288, out);
  run_task<1, 256, 4>("+ values (stream + shuffle + (a*b)*v)", A, B, ia, ib, vals, nnz, 288, out);
  run_task<2, 256, 4>("+ tasks", A, B, ia, ib, vals, nnz, 288, out);
  run_task<2, 256, 4>("+ tasks", A, B, ia, ib, vals, nnz, 1024, out);
  run_task<2, 256, 4>("+ tasks", A, B, ia, ib, vals, nnz, 4096, out);
  run_task<3, 256, 4>("+ tasks, U=8 (64-reg cap)", A, B, ia, ib, vals, nnz, 288, out);
  run_task<3, 256, 3>("+ tasks, U=8", A, B, ia, ib, vals, nnz, 288, out);
  run_task<3, 256, 2>("+ tasks, U=8", A, B, ia, ib, vals, nnz, 288, out);
  run_task<2, 256, 3>("+ tasks", A, B, ia, ib, vals, nnz, 288, out);
  run_task<2, 512, 2>("+ tasks", A, B, ia, ib, vals, nnz, 288, out);
  run_task<2, 1024, 1>("+ tasks", A, B, ia, ib, vals, nnz, 288, out);
  run_task<2, 128, 8>("+ tasks", A, B, ia, ib, vals, nnz, 288, out);
  {
    std::vector<int2> hab(nnz); std::vector<int4> hrec(nnz);
    for (int64_t e = 0; e < nnz; ++e) {
      hab[e] = make_int2(ha[e], hb[e]);
      long long bits; memcpy(&bits, &hv[e], 8);
      hrec[e] = make_int4(ha[e], hb[e], (int)(bits & 0xffffffff), (int)(bits >> 32));
    }
    int2 *iab; int4 *rec;
    CK(cudaMalloc(&iab, nnz * 8)); CK(cudaMalloc(&rec, nnz * 16));
    CK(cudaMemcpy(iab, hab.data(), nnz * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(rec, hrec.data(), nnz * 16, cudaMemcpyHostToDevice));
    run_rec<0, 256, 4>("no shuffles: int2 pairs + values by group loads", A, B, iab, vals, rec, nnz, 288, out);
    run_rec<0, 256, 3>("no shuffles: int2 pairs + values by group loads", A, B, iab, vals, rec, nnz, 288, out);
    run_rec<0, 128, 8>("no shuffles: int2 pairs + values by group loads", A, B, iab, vals, rec, nnz, 288, out);
    run_rec<1, 256, 4>("no shuffles: 16-B records", A, B, iab, vals, rec, nnz, 288, out);
    run_rec<1, 256, 3>("no shuffles: 16-B records", A, B, iab, vals, rec, nnz, 288, out);
    run_rec<1, 128, 8>("no shuffles: 16-B records", A, B, iab, vals, rec, nnz, 288, out);
    run_rec<1, 256, 4>("no shuffles: 16-B records", A, B, iab, vals, rec, nnz, 144, out);
    cudaFree(iab); cudaFree(rec);
  }
}

int main() {
  task_suite();
  const int64_t nnz = 10000000 / 32 * 32;
  const int rowsA = 10000;
  for (int brows : {512, 1024}) {
    std::vector<int32_t> ha(nnz), hb(nnz), hb_full(nnz);
    uint64_t s = 88172645463325252ull;
    auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
    for (int64_t e = 0; e < nnz; ++e) {
      ha[e] = (int32_t)(rnd() % rowsA);
      hb[e] = (int32_t)(rnd() % brows);
      hb_full[e] = (int32_t)(rnd() % rowsA);
    }
    std::vector<double> hA((size_t)rowsA * R), hB((size_t)rowsA * R);
    for (auto &x : hA) x = (double)(rnd() % 1000) * 1e-3;
    for (auto &x : hB) x = (double)(rnd() % 1000) * 1e-3;
    double *A, *B, *out; int32_t *ia, *ib, *ibf;
    CK(cudaMalloc(&A, hA.size() * 8)); CK(cudaMalloc(&B, hB.size() * 8));
    CK(cudaMalloc(&ia, nnz * 4)); CK(cudaMalloc(&ib, nnz * 4)); CK(cudaMalloc(&ibf, nnz * 4));
    CK(cudaMalloc(&out, 148 * 8 * 1024 * 8));
    CK(cudaMemcpy(A, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(B, hB.data(), hB.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ia, ha.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ib, hb.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ibf, hb_full.data(), nnz * 4, cudaMemcpyHostToDevice));
    const size_t smem = (size_t)brows * R * 8;
    printf("== block rows %d (%zu KB of shared memory) ==\n", brows, smem / 1024);
    run<0, 256>("LDG + LDG (10k-row tables), 256 thr x 8/SM", 148 * 8, 0, A, B, ia, ibf, nnz, brows, out);
    run<0, 1024>("LDG + LDG (10k-row tables), 1024 thr x 2/SM", 148 * 2, 0, A, B, ia, ibf, nnz, brows, out);
    run<0, 1024>("LDG + LDG (2nd table = block rows, L1 hits)", 148 * 2, 0, A, B, ia, ib, nnz, brows, out);
    if (brows == 512) {
      run<1, 512>("LDG + LDS, 512 thr x 3/SM", 148 * 3, smem, A, B, ia, ib, nnz, brows, out);
      run<1, 1024>("LDG + LDS, 1024 thr x 2/SM", 148 * 2, smem, A, B, ia, ib, nnz, brows, out);
      run<2, 1024>("LDS + LDS, 1024 thr x 2/SM", 148 * 2, smem, A, B, ia, ib, nnz, brows, out);
    } else {
      run<1, 512>("LDG + LDS, 512 thr x 1/SM", 148, smem, A, B, ia, ib, nnz, brows, out);
      run<1, 1024>("LDG + LDS, 1024 thr x 1/SM", 148, smem, A, B, ia, ib, nnz, brows, out);
      run<2, 1024>("LDS + LDS, 1024 thr x 1/SM", 148, smem, A, B, ia, ib, nnz, brows, out);
    }
    cudaFree(A); cudaFree(B); cudaFree(ia); cudaFree(ib); cudaFree(ibf); cudaFree(out);
  }
  return 0;
}
