// dense_tc.cu -- TF32 dense MTTKRP on the 5th-generation tensor cores (sm_100a).
//
// The fp32 variant of the dense MTTKRP (BASELINE cfg 4 / north_star "dense
// MTTKRP on FP64/TF32 tensor cores"): the same single-pass formulation as the
// FP64 kernel (dense_dmma.cu),
//
//   M_n = X_(n) . KR,  KR[(p, q), r] = F1[p, r] * F2[q, r]  (formed in smem),
//
// but issued as tcgen05.mma.cta_group::1.kind::tf32 with the accumulator in
// tensor memory.  One CTA = one 128-row output tile x 64 columns over a
// range of 32-value reduction chunks; warp roles:
//
//   warp 0      TMA producer: X tile of each chunk (128 x 32 fp32, 128-byte
//               swizzle) -> stage s, completing on full_a[s]
//   warp 1      TMEM allocator + MMA issuer (one thread): 4 x (M128 N64 K8)
//               per chunk, tcgen05.commit -> empty[s]; after the last chunk
//               tcgen05.commit -> tmem_full
//   warps 2..9  KR builders in 4 groups of 2 warps (group g builds the
//               chunks it = g mod 4, so four chunks' factor-row loads are in
//               flight): thread r forms F1[p, r] * F2[q0 + q, r] for the 32 q
//               of its chunk, rounds to TF32 (cvt.rna) and stores its 128-byte
//               row in the K-major SW128 layout the MMA's smem descriptor
//               describes, fence.proxy.async, arrive on full_b[s]
//   warps 2..5  then the epilogue: tcgen05.ld 32x32b (warp w reads TMEM
//               lanes 32 (w mod 4) ..), partial tile -> global
//
// Modes 0 / 1 / 3 read X tiles K-major (rows = output index, 128 B of the
// contiguous k per row); mode 2's output index k IS the contiguous one, so
// its tiles are MN-major: four 32-row x 128-B boxes, loaded with the TMA
// swizzle in 32-byte atoms (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) -- the only
// MN-major smem layout UMMA accepts for 32-bit operands (SWIZZLE_128B_BASE32B,
// LBO 4 KB between 32-value M blocks, SBO 512 B between 4-row K groups).  Split-K partials are
// summed in split order by dense_split_sum (deterministic).
//
// Precision: TF32 operands (10-bit mantissa), FP32 accumulation -- the
// accuracy class of a TF32 GEMM (relative error ~1e-3 on N(0,1) data), not
// the fp64 parity path.  HBM-bound: X (2.05 GB at 800^3) is read once.
#include "common.cuh"
#include "tma.cuh"

namespace cpfit {
namespace tc {

constexpr int MT = 128;    // UMMA M
constexpr int NT = 64;     // UMMA N (output columns per CTA)
constexpr int KC = 32;     // fp32 values per chunk (one 128-byte swizzle row)
#ifndef CPFIT_TC_STAGES
#define CPFIT_TC_STAGES 6
#endif
constexpr int STAGES = CPFIT_TC_STAGES;
constexpr int A_BYTES = MT * KC * 4;   // 16 KB
constexpr int B_BYTES = NT * KC * 4;   // 8 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int THREADS = 320;
constexpr int GROUPS = 4;     // KR builder groups (2 warps each)
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t TMEM_COLS = 64;

struct Args {
  int mode;
  int R;
  int64_t I, J, K;
  const float *X;
  const float *F1, *F2;
  int64_t rows, nq, nqc, nchunks, per_split;
  float *out;
  int use_tma;
};

// layout: 2 = SWIZZLE_128B (16-byte chunks), 1 = SWIZZLE_128B_BASE32B (32-byte chunks)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) |  // descriptor version (sm_100)
         ((uint64_t)layout << 61);
}

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return u;
}

__device__ __forceinline__ float x_at(const Args &a, int64_t m, int64_t p, int64_t q) {
  switch (a.mode) {
    case 0:
      return (m < a.I && q < a.K) ? a.X[(m * a.J + p) * a.K + q] : 0.f;
    case 1:
      return (m < a.J && q < a.K) ? a.X[(p * a.J + m) * a.K + q] : 0.f;
    case 2:
      return (m < a.K && q < a.J) ? a.X[(p * a.J + q) * a.K + m] : 0.f;
    default:
      return (m < a.rows && q < a.K) ? a.X[m * a.K + q] : 0.f;
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    dense_tc_kernel(const __grid_constant__ CUtensorMap tmap, const Args a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned base by pointer arithmetic on the shared array (keeps the
  // shared address space visible to the compiler: LDS/STS, not generic LD/ST)
  unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *full_a = (uint64_t *)(smem + STAGES * STAGE_BYTES);
  uint64_t *full_b = full_a + STAGES;
  uint64_t *empty = full_b + STAGES;
  uint64_t *tmem_full = empty + STAGES;
  uint32_t *tmem_slot = (uint32_t *)(tmem_full + 1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = (int64_t)blockIdx.x * MT;
  const int split = blockIdx.y;
  const int n0 = blockIdx.z * NT;
  const int64_t c_begin = (int64_t)split * a.per_split;
  const int64_t c_end = min(a.nchunks, c_begin + a.per_split);
  const int n = (int)(c_end - c_begin);

  if (tid == 0) {
    if (a.use_tma) tma_prefetch_desc(&tmap);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_a[s], 1);
      mbar_init(&full_b[s], 64);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  auto stage_a = [&](int s) { return smem + s * STAGE_BYTES; };
  auto stage_b = [&](int s) { return smem + s * STAGE_BYTES + A_BYTES; };

  if (warp == 0) {
    // ---------------- producer: X tiles ----------------
    for (int it = 0; it < n; ++it) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty[s], (uint32_t)(((it / STAGES) - 1) & 1));
      const int64_t c = c_begin + it;
      const int p = (int)(c / a.nqc), q0 = (int)(c % a.nqc) * KC;
      unsigned char *dst = stage_a(s);
      if (a.use_tma) {
        if (lane == 0) {
          mbar_expect_tx(&full_a[s], A_BYTES);
          switch (a.mode) {
            case 0: tma_load_3d(dst, &tmap, &full_a[s], q0, p, (int)m0); break;
            case 1: tma_load_3d(dst, &tmap, &full_a[s], q0, (int)m0, p); break;
            case 2:
#pragma unroll
              for (int b = 0; b < MT / 32; ++b)
                tma_load_3d(dst + b * 4096, &tmap, &full_a[s], (int)m0 + 32 * b, q0, p);
              break;
            default: tma_load_2d(dst, &tmap, &full_a[s], q0, (int)m0); break;
          }
        }
      } else {
        // generic path: the warp writes the same swizzled layout TMA would
        for (int e = lane; e < MT * KC; e += 32) {
          const int m = e / KC, k = e % KC;
          const float v = x_at(a, m0 + m, p, (int64_t)q0 + k);
          int off;
          if (a.mode == 2) {  // MN-major: block m/32, row k, 32-byte atoms XOR row mod 4
            const int row = (m >> 5) * 32 + k, col = m & 31;
            off = row * 128 + ((((col >> 3) ^ (row & 3))) << 5) + (col & 7) * 4;
          } else {            // K-major: row m, 16-byte chunks XOR row mod 8
            off = m * 128 + ((((k >> 2) ^ (m & 7))) << 4) + (k & 3) * 4;
          }
          *(float *)(dst + off) = v;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_a[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = (1u << 4)                       // D: f32
                             | (2u << 7) | (2u << 10)        // A, B: tf32
                             | ((a.mode == 2 ? 1u : 0u) << 15)  // A major (MN for mode 2)
                             | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(MT >> 4) << 24);
      for (int it = 0; it < n; ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (uint32_t)((it / STAGES) & 1);
        mbar_wait(&full_a[s], ph);
        mbar_wait(&full_b[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t abase = smem_u32(stage_a(s)), bbase = smem_u32(stage_b(s));
#pragma unroll
        for (int kk = 0; kk < KC / 8; ++kk) {
          const uint64_t ad = a.mode == 2 ? smem_desc(abase + kk * 1024, 4096, 512, 1)
                                          : smem_desc(abase + kk * 32, 16, 1024, 2);
          const uint64_t bd = smem_desc(bbase + kk * 32, 16, 1024, 2);
          const uint32_t accum = (it > 0 || kk > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"(accum)
              : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&empty[s]))
            : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(tmem_full))
          : "memory");
    }
    __syncwarp();
  } else {
    // ---------------- KR builders, then the epilogue ----------------
    const int g = (warp - 2) >> 1;     // builder group: chunks it = g (mod GROUPS)
    const int r = tid - 64 - 64 * g;   // KR row (output column) 0..63
    const int col = n0 + r;
    const bool colok = col < a.R;
    for (int it = g; it < n; it += GROUPS) {
      const int s = it % STAGES;
      const int64_t c = c_begin + it;
      const int64_t p = c / a.nqc, q0 = (c % a.nqc) * KC;
      const float f1 = (a.F1 && colok) ? __ldg(a.F1 + p * a.R + col) : 1.f;
      float v[KC];
#ifdef CPFIT_TC_NOBUILD
#pragma unroll
      for (int j = 0; j < KC; ++j) v[j] = 0.f;
#else
      if (colok && q0 + KC <= a.nq) {  // whole chunk inside: unpredicated strided loads
        const float *src = a.F2 + q0 * a.R + col;
#pragma unroll
        for (int j = 0; j < KC; ++j) v[j] = __ldg(src + j * a.R);
      } else {
#pragma unroll
        for (int j = 0; j < KC; ++j) {
          const int64_t q = q0 + j;
          v[j] = (colok && q < a.nq) ? __ldg(a.F2 + q * a.R + col) : 0.f;
        }
      }
#endif
      if (it >= STAGES) mbar_wait(&empty[s], (uint32_t)(((it / STAGES) - 1) & 1));
      unsigned char *dst = stage_b(s) + r * 128;
#pragma unroll
      for (int h = 0; h < KC / 4; ++h) {
        const uint4 w = make_uint4(tf32_rna(f1 * v[4 * h]), tf32_rna(f1 * v[4 * h + 1]),
                                   tf32_rna(f1 * v[4 * h + 2]), tf32_rna(f1 * v[4 * h + 3]));
        *(uint4 *)(dst + ((h ^ (r & 7)) << 4)) = w;
      }
      fence_proxy_async_smem();
      mbar_arrive(&full_b[s]);
    }
    if (warp < 6) {  // epilogue: warps 2..5 cover the four TMEM lane quarters
      mbar_wait(tmem_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int quarter = warp & 3;
      const int64_t m = m0 + quarter * 32 + lane;
      float *out = a.out + (int64_t)split * a.rows * a.R;
  #pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t v[32];
        const uint32_t addr = tmem + ((uint32_t)(quarter * 32) << 16) + h * 32;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
              "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
              "=r"(v[31])
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (m < a.rows) {
  #pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int cc = n0 + h * 32 + j;
            if (cc < a.R) out[m * a.R + cc] = __uint_as_float(v[j]);
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

}  // namespace tc

int split_sum_f32(const float *part, int nsplit, int64_t n, float *out, cudaStream_t s);

int dense_tc_run(int mode, int64_t I, int64_t J, int64_t K, int R, const float *X,
                 const float *F1, const float *F2, float *out, cudaStream_t s) {
  using namespace tc;
  Args a{};
  a.mode = mode;
  a.R = R;
  a.I = I;
  a.J = J;
  a.K = K;
  a.X = X;
  a.F1 = F1;
  a.F2 = F2;
  int64_t np;
  switch (mode) {
    case 0: a.rows = I; np = J; a.nq = K; break;
    case 1: a.rows = J; np = I; a.nq = K; break;
    case 2: a.rows = K; np = I; a.nq = J; break;
    default: a.rows = I * J; np = 1; a.nq = K; break;
  }
  a.nqc = (a.nq + KC - 1) / KC;
  a.nchunks = np * a.nqc;
  const int sms = num_sms();
  const int64_t n_mt = (a.rows + MT - 1) / MT, n_nt = (R + NT - 1) / NT;
  const int64_t tiles = n_mt * n_nt;
  int64_t ns = tiles >= sms ? 1 : sms / tiles;
  if (ns > a.nchunks) ns = a.nchunks;
  if (ns < 1) ns = 1;
  a.per_split = (a.nchunks + ns - 1) / ns;
  const int64_t nsplit = (a.nchunks + a.per_split - 1) / a.per_split;

  CUtensorMap map;
  memset(&map, 0, sizeof(map));
  bool tma = false;
  if (a.rows < (1ll << 31) && np < (1ll << 31) && a.nq < (1ll << 31)) {
    if (mode == 3) {
      const uint64_t dims[2] = {(uint64_t)K, (uint64_t)(I * J)};
      const uint32_t box[2] = {32, (uint32_t)MT};
      tma = make_tmap(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 2, X, dims, box);
    } else {
      const uint64_t dims[3] = {(uint64_t)K, (uint64_t)J, (uint64_t)I};
      uint32_t box[3];
      if (mode == 0) { box[0] = 32; box[1] = 1; box[2] = MT; }
      else if (mode == 1) { box[0] = 32; box[1] = MT; box[2] = 1; }
      else { box[0] = 32; box[1] = 32; box[2] = 1; }
      tma = make_tmap(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 3, X, dims, box,
                      mode == 2 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
    }
  }
  a.use_tma = tma ? 1 : 0;

  Scratch<float> part(s);
  if (nsplit > 1) {
    CPFIT_TRY(part.alloc((size_t)nsplit * a.rows * R));
    a.out = part.ptr;
  } else {
    a.out = out;
  }
  static bool configured = false;
  if (!configured) {
    CPFIT_CUDA(cudaFuncSetAttribute(dense_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    SMEM));
    configured = true;
  }
  dim3 grid((unsigned)n_mt, (unsigned)nsplit, (unsigned)n_nt);
  dense_tc_kernel<<<grid, THREADS, SMEM, s>>>(map, a);
  CPFIT_LAUNCH_CHECK("dense_tc_kernel");
  if (nsplit > 1) {
    CPFIT_TRY(split_sum_f32(part.ptr, (int)nsplit, a.rows * R, out, s));
  }
  return CPFIT_OK;
}

}  // namespace cpfit
