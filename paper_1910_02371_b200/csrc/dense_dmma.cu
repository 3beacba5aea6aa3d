// dense_dmma.cu -- hand-written FP64 dense MTTKRP (BASELINE cfg 4) for sm_100a.
//
// einsum('ijk,jr,kr->ir') and its mode-1 / mode-2 analogues as ONE pass over
// the dense tensor X (I x J x K, row-major, fp64):
//
//   M_n = X_(n) . KR,   KR[(p, q), r] = F1[p, r] * F2[q, r]
//
// with the Khatri-Rao operand formed tile by tile in shared memory (never in
// HBM).  The reduction index (p, q) is walked in chunks of KC = 32 values of
// the contiguous q for one p:
//
//   mode 0: out rows i, p = j, q = k   (F1 = B, F2 = C)   X tile [i][k]  (K-major)
//   mode 1: out rows j, p = i, q = k   (F1 = A, F2 = C)   X tile [j][k]  (K-major)
//   mode 2: out rows k, p = i, q = j   (F1 = A, F2 = B)   X tile [j][k]  (MN-major)
//   mode 3: T = X_(IJ x K) . C  (out rows (i, j), q = k, F1 = 1): the GEMM a
//           CP-ALS sweep shares between modes 0 and 1 (cpfit_dense_xc)
//
// X tiles are loaded by TMA (cp.async.bulk.tensor, 128-byte swizzle, one
// mbarrier per stage, 3 stages) -- UTMALDG in SASS; the KR tile is built by
// the threads from L2-resident factor rows whose loads are issued one stage
// ahead, before the math of the current stage.  Math: FP64 tensor-core MMA
// (mma.sync m8n8k4 -> DMMA.8x8x4, the only FP64 MMA shape on sm_100a: the
// m16n8k{8,16} f64 forms lower to the same instruction; tcgen05 has no f64
// kind).  CTA = 8 warps (2 per SM sub-partition: the DMMA pipe is per
// sub-partition, so an uneven warp count leaves sub-partitions idle at the
// per-stage barrier), 4 along M x 2 along N; warp tile (8 TM) x 32 = TM x 4
// DMMA tiles, CTA tile MT x 64 with MT = 32 TM, TM = 4 or 5 chosen so the
// 800-row outputs of cfg 4 tile exactly (MT = 160).
//
// Split-K: the chunk range is divided over `nsplit` CTAs per output tile so
// one wave fills the 148 SMs; each split writes its partial tile and
// dense_split_sum adds the partials in split order -- deterministic, no
// atomics (SURVEY.md section 4's determinism contract).
//
// Reference: there is no dense tensor in the reference; its
// oracle is kernels.mttkrp on a fully observed SparseTensor
// (kernels.py:46-91), which tests/test_gpu_dense.py checks against.
#include "common.cuh"
#include "tma.cuh"

namespace cpfit {
namespace dmma {

constexpr int KC = 32;      // reduction values per stage

struct Args {
  int mode;
  int R;
  int64_t I, J, K;
  const double *X;
  const double *F1, *F2;
  int64_t rows;       // output rows
  int64_t nq;         // extent of the chunked index q
  int64_t nqc;        // chunks per p
  int64_t nchunks;    // total chunks
  int64_t per_split;  // chunks per split
  double *out;        // [nsplit][rows][R] partials (or the result when nsplit == 1)
  int use_tma;
};

// WN = warps along N: 2 -> 64-column CTA tile, 8 warps, 3 stages, 1 CTA/SM;
//                     1 -> 32-column CTA tile, 4 warps, 2 stages, 2 CTAs/SM
//                          (one CTA's per-stage barrier is covered by the other's math)
template <int TM, int WN>
struct Cfg {
  static constexpr int MT = 32 * TM;   // 4 warps along M, 8 TM rows each
  static constexpr int NT = 32 * WN;
  static constexpr int THREADS = 128 * WN;
  static constexpr int STAGES = WN == 2 ? 3 : 2;
  static constexpr int MINB = WN == 2 ? 1 : 2;
  static constexpr int BP = NT + 8;    // KR tile pitch: rows 0..3 of a B fragment hit 2 bank groups
  static constexpr int A_DBL = MT * KC;
  static constexpr int B_DBL = KC * BP;
  static constexpr int STAGE_BYTES = ((A_DBL + B_DBL) * 8 + 1023) / 1024 * 1024;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 64;
};

// element offset of (m, k) in a stage's X tile, matching the TMA 128-byte
// swizzle (16-byte chunk index XOR row index mod 8 inside 1024-byte blocks)
template <int MT>
__device__ __forceinline__ int a_off_k(int m, int k) {  // modes 0, 1, 3: rows m, 128-B rows of k
  return (k >> 4) * (MT * 16) + m * 16 + (((((k & 15) >> 1) ^ (m & 7))) << 1) + (k & 1);
}
__device__ __forceinline__ int a_off_mn(int m, int k) {  // mode 2: rows k (= j), 128-B rows of m
  return (m >> 4) * 512 + k * 16 + (((((m & 15) >> 1) ^ (k & 7))) << 1) + (m & 1);
}

// X element of output row `m`, reduction (p, q); 0 outside the tensor
__device__ __forceinline__ double x_at(const Args &a, int64_t m, int64_t p, int64_t q) {
  switch (a.mode) {
    case 0:
      return (m < a.I && q < a.K) ? a.X[(m * a.J + p) * a.K + q] : 0.0;
    case 1:
      return (m < a.J && q < a.K) ? a.X[(p * a.J + m) * a.K + q] : 0.0;
    case 2:
      return (m < a.K && q < a.J) ? a.X[(p * a.J + q) * a.K + m] : 0.0;
    default:
      return (m < a.rows && q < a.K) ? a.X[m * a.K + q] : 0.0;
  }
}

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int TM, int WN, bool MN>
__global__ void __launch_bounds__(128 * WN, (WN == 2 ? 1 : 2))
    dense_dmma_kernel(const __grid_constant__ CUtensorMap tmap, const Args a) {
  typedef Cfg<TM, WN> C;
  constexpr int STAGES = C::STAGES, NT = C::NT, BP = C::BP;
  constexpr int MT = C::MT;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned base by pointer arithmetic on the shared array (keeps the
  // shared address space visible to the compiler: LDS/STS, not generic LD/ST)
  unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t *bar = (uint64_t *)(smem + STAGES * C::STAGE_BYTES);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  const int64_t m0 = (int64_t)blockIdx.x * MT;
  const int split = blockIdx.y;
  const int n0 = blockIdx.z * NT;
  const int64_t c_begin = (int64_t)split * a.per_split;
  const int64_t c_end = min(a.nchunks, c_begin + a.per_split);
  const int n = (int)(c_end - c_begin);

  if (tid == 0) {
    if (a.use_tma) tma_prefetch_desc(&tmap);
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto stage_a = [&](int s) { return (double *)(smem + s * C::STAGE_BYTES); };
  auto stage_b = [&](int s) { return (double *)(smem + s * C::STAGE_BYTES + C::A_DBL * 8); };

  // X tile of chunk c -> stage s (TMA: thread 0 issues, the mbarrier completes)
  auto issue_a = [&](int s, int64_t c) {
    const int p = (int)(c / a.nqc), q0 = (int)(c % a.nqc) * KC;
    double *dst = stage_a(s);
    mbar_expect_tx(&bar[s], MT * KC * 8);
    switch (a.mode) {
      case 0:
        tma_load_3d(dst, &tmap, &bar[s], q0, p, (int)m0);
        tma_load_3d(dst + MT * 16, &tmap, &bar[s], q0 + 16, p, (int)m0);
        break;
      case 1:
        tma_load_3d(dst, &tmap, &bar[s], q0, (int)m0, p);
        tma_load_3d(dst + MT * 16, &tmap, &bar[s], q0 + 16, (int)m0, p);
        break;
      case 2:
#pragma unroll
        for (int b = 0; b < MT / 16; ++b)
          tma_load_3d(dst + b * 512, &tmap, &bar[s], (int)m0 + 16 * b, q0, p);
        break;
      default:
        tma_load_2d(dst, &tmap, &bar[s], q0, (int)m0);
        tma_load_2d(dst + MT * 16, &tmap, &bar[s], q0 + 16, (int)m0);
        break;
    }
  };
  // generic path (tensor not describable by TMA): synchronous loads
  auto load_a_sync = [&](int s, int64_t c) {
    const int64_t p = c / a.nqc, q0 = (c % a.nqc) * KC;
    double *dst = stage_a(s);
    for (int e = tid; e < MT * KC; e += C::THREADS) {
      const int m = e / KC, k = e % KC;
      const double v = x_at(a, m0 + m, p, q0 + k);
      if (MN)
        dst[a_off_mn(m, k)] = v;
      else
        dst[a_off_k<MT>(m, k)] = v;
    }
  };

  // KR tile: thread t -> row q = t / 8, columns 8 (t % 8) .. +7.  F2 rows are
  // read as 16-byte vectors when the rank allows; the F1 row (fixed p) is
  // re-read only when p changes.
  constexpr bool builder = true;
  const int bq = tid / (NT / 8), bn = (tid % (NT / 8)) * 8;
  const bool vec = (a.R % 2 == 0) && (((uintptr_t)a.F2 | (uintptr_t)a.F1) % 16 == 0);
  double f1r[8], f2r[8];
  int64_t f1_p = -1;
  auto fetch_b = [&](int64_t c) {
    const int64_t p = c / a.nqc, q = (c % a.nqc) * KC + bq;
    if (p != f1_p) {
      f1_p = p;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = n0 + bn + j;
        f1r[j] = (a.F1 && col < a.R) ? __ldg(a.F1 + p * a.R + col) : 1.0;
      }
    }
    if (vec && q < a.nq && n0 + bn + 8 <= a.R) {
      const double2 *src = reinterpret_cast<const double2 *>(a.F2 + q * a.R + n0 + bn);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 v = __ldg(src + j);
        f2r[2 * j] = v.x;
        f2r[2 * j + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = n0 + bn + j;
        f2r[j] = (col < a.R && q < a.nq) ? __ldg(a.F2 + q * a.R + col) : 0.0;
      }
    }
  };
  auto store_b = [&](int s) {
    double *dst = stage_b(s) + bq * BP + bn;
#pragma unroll
    for (int j = 0; j < 8; j += 2)
      *reinterpret_cast<double2 *>(dst + j) = make_double2(f1r[j] * f2r[j], f1r[j + 1] * f2r[j + 1]);
  };

  // prologue: stages 0 .. STAGES-2
  const int pre = n < STAGES - 1 ? n : STAGES - 1;
  for (int s = 0; s < pre; ++s) {
    if (a.use_tma) {
      if (tid == 0) issue_a(s, c_begin + s);
    } else {
      load_a_sync(s, c_begin + s);
    }
    if (builder) {
      fetch_b(c_begin + s);
      store_b(s);
    }
  }
  __syncthreads();

  double acc[TM][4][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int fr = lane >> 2, fk = lane & 3;
  for (int it = 0; it < n; ++it) {
    const int s = it % STAGES;
    const int nxt = it + STAGES - 1;
    const bool have_next = nxt < n;
    if (have_next) {
      if (a.use_tma && tid == 0) issue_a(nxt % STAGES, c_begin + nxt);
      if (builder) fetch_b(c_begin + nxt);
    }
    if (a.use_tma) mbar_wait(&bar[s], (uint32_t)((it / STAGES) & 1));
    const double *As = stage_a(s);
    const double *Bs = stage_b(s);
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      const int k = ks * 4 + fk;
      double av[TM], bv[4];
#pragma unroll
      for (int mi = 0; mi < TM; ++mi) {
        const int m = wm * (8 * TM) + mi * 8 + fr;
        av[mi] = MN ? As[a_off_mn(m, k)] : As[a_off_k<MT>(m, k)];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bv[ni] = Bs[k * BP + wn * 32 + ni * 8 + fr];
#pragma unroll
      for (int mi = 0; mi < TM; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], av[mi], bv[ni]);
    }
    if (have_next) {
      if (builder) store_b(nxt % STAGES);
      if (!a.use_tma) load_a_sync(nxt % STAGES, c_begin + nxt);
    }
    __syncthreads();
  }

  // epilogue: partial (or final) tile
  double *out = a.out + (int64_t)split * a.rows * a.R;
#pragma unroll
  for (int mi = 0; mi < TM; ++mi) {
    const int64_t m = m0 + wm * (8 * TM) + mi * 8 + fr;
    if (m >= a.rows) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int col = n0 + wn * 32 + ni * 8 + 2 * fk;
      if (col < a.R) out[m * a.R + col] = acc[mi][ni][0];
      if (col + 1 < a.R) out[m * a.R + col + 1] = acc[mi][ni][1];
    }
  }
}

}  // namespace dmma

// out[e] = sum_{s < nsplit} part[s * n + e]  (split order: deterministic)
template <typename T, typename P>
__global__ void dense_split_sum(const P *__restrict__ part, int nsplit, int64_t n,
                                T *__restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < nsplit; ++s) acc += (double)part[(int64_t)s * n + e];
    out[e] = (T)acc;
  }
}

int split_sum_f32(const float *part, int nsplit, int64_t n, float *out, cudaStream_t s) {
  dense_split_sum<float, float><<<grid_for(n, 256), 256, 0, s>>>(part, nsplit, n, out);
  CPFIT_LAUNCH_CHECK("dense_split_sum");
  return CPFIT_OK;
}

// G[a, b] = prod_f sum_i F_f[i, a] F_f[i, b]: one CTA per row a, thread (slice, b)
// sums its row slice, slices combined in order (deterministic)
template <typename T>
__global__ void dense_gram_kernel(int nf, CpfitDims rows, int R, CpfitCoordPtrs<T> F,
                                  T *__restrict__ G) {
  extern __shared__ double red[];
  const int a = blockIdx.x, t = threadIdx.x;
  const int S = blockDim.x / R, b = t % R, sl = t / R;
  double prod = 1.0;
  for (int f = 0; f < nf; ++f) {
    const T *p = F.p[f];
    const int64_t n = rows.d[f], per = (n + S - 1) / S;
    double acc = 0.0;
    if (sl < S) {
      const int64_t i1 = min(n, (sl + 1) * per);
      for (int64_t i = sl * per; i < i1; ++i)
        acc += (double)__ldg(p + i * R + a) * (double)__ldg(p + i * R + b);
    }
    red[t] = acc;
    __syncthreads();
    if (sl == 0) {
      double tot = red[b];
      for (int k = 1; k < S; ++k) tot += red[k * R + b];
      prod *= tot;
    }
    __syncthreads();
  }
  if (sl == 0) G[a * R + b] = (T)prod;
}

namespace dmma {

struct Plan {
  int tm, wn;
  int64_t n_mt, nsplit, per_split, n_nt;
};

inline Plan plan(int64_t rows, int64_t nchunks, int R, int wn) {
  const int sms = num_sms();
  const int per_sm = wn == 2 ? 1 : 2;   // resident CTAs per SM
  const int NT = 32 * wn;
  Plan best{};
  double best_cost = -1;
  for (int tm = 4; tm <= 5; ++tm) {
    const int MT = 32 * tm;
    Plan p;
    p.tm = tm;
    p.wn = wn;
    p.n_mt = (rows + MT - 1) / MT;
    p.n_nt = (R + NT - 1) / NT;
    const int64_t tiles = p.n_mt * p.n_nt;
    const int64_t slots = (int64_t)sms * per_sm;
    int64_t ns = tiles >= slots ? 1 : slots / tiles;
    if (ns > nchunks) ns = nchunks;
    if (ns < 1) ns = 1;
    p.per_split = (nchunks + ns - 1) / ns;
    p.nsplit = (nchunks + p.per_split - 1) / p.per_split;
    const int64_t ctas = tiles * p.nsplit;
    const double cost = (double)((ctas + slots - 1) / slots) * (double)p.per_split * MT;
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = p;
    }
  }
  return best;
}

template <int TM, int WN, bool MN>
int launch(const CUtensorMap &map, const Args &a, const Plan &p, cudaStream_t s) {
  typedef Cfg<TM, WN> C;
  static bool configured = false;
  if (!configured) {
    CPFIT_CUDA(cudaFuncSetAttribute(dense_dmma_kernel<TM, WN, MN>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    configured = true;
  }
  dim3 grid((unsigned)p.n_mt, (unsigned)p.nsplit, (unsigned)p.n_nt);
  dense_dmma_kernel<TM, WN, MN><<<grid, C::THREADS, C::SMEM, s>>>(map, a);
  CPFIT_LAUNCH_CHECK("dense_dmma_kernel");
  return CPFIT_OK;
}

template <int WN>
int launch_wn(const CUtensorMap &map, const Args &a, const Plan &p, cudaStream_t s) {
  const bool mn = a.mode == 2;
  if (p.tm == 4) return mn ? launch<4, WN, true>(map, a, p, s) : launch<4, WN, false>(map, a, p, s);
  return mn ? launch<5, WN, true>(map, a, p, s) : launch<5, WN, false>(map, a, p, s);
}

// CTA shape (measurement knob; default: the faster one on B200)
inline int cta_wn() {
  static int wn = 0;
  if (!wn) {
    const char *e = getenv("CPFIT_DMMA_WN");
    wn = (e && atoi(e) == 2) ? 2 : 1;  // 1: 2 CTAs/SM (0.81-0.83 of cuBLAS DGEMM vs 0.79-0.80)
  }
  return wn;
}

// Runs one dense KR-GEMM (modes 0..2) or the X.C GEMM (mode 3) in fp64.
inline int run(int mode, int64_t I, int64_t J, int64_t K, int R, const double *X,
               const double *F1, const double *F2, double *out, cudaStream_t s) {
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
  Plan p = plan(a.rows, a.nchunks, R, cta_wn());
  a.per_split = p.per_split;
  const int MT = 32 * p.tm;

  CUtensorMap map;
  memset(&map, 0, sizeof(map));
  bool tma = false;
  if (a.rows < (1ll << 31) && np < (1ll << 31) && a.nq < (1ll << 31)) {
    if (mode == 3) {
      const uint64_t dims[2] = {(uint64_t)K, (uint64_t)(I * J)};
      const uint32_t box[2] = {16, (uint32_t)MT};
      tma = make_tmap(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 2, X, dims, box);
    } else {
      const uint64_t dims[3] = {(uint64_t)K, (uint64_t)J, (uint64_t)I};
      uint32_t box[3];
      if (mode == 0) { box[0] = 16; box[1] = 1; box[2] = (uint32_t)MT; }
      else if (mode == 1) { box[0] = 16; box[1] = (uint32_t)MT; box[2] = 1; }
      else { box[0] = 16; box[1] = 32; box[2] = 1; }
      tma = make_tmap(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 3, X, dims, box);
    }
  }
  a.use_tma = tma ? 1 : 0;

  Scratch<double> part(s);
  if (p.nsplit > 1) {
    CPFIT_TRY(part.alloc((size_t)p.nsplit * a.rows * R));
    a.out = part.ptr;
  } else {
    a.out = out;
  }
  if (p.wn == 2)
    CPFIT_TRY(launch_wn<2>(map, a, p, s));
  else
    CPFIT_TRY(launch_wn<1>(map, a, p, s));
  if (p.nsplit > 1) {
    const int64_t n = a.rows * R;
    dense_split_sum<double, double><<<grid_for(n, 256), 256, 0, s>>>(part.ptr, (int)p.nsplit, n,
                                                                     out);
    CPFIT_LAUNCH_CHECK("dense_split_sum");
  }
  return CPFIT_OK;
}

}  // namespace dmma

// implemented in dense_tc.cu (TF32 tcgen05 path)
int dense_tc_run(int mode, int64_t I, int64_t J, int64_t K, int R, const float *X,
                 const float *F1, const float *F2, float *out, cudaStream_t s);

}  // namespace cpfit

using namespace cpfit;

extern "C" {

int cpfit_dense_mttkrp(int dtype, int64_t I, int64_t J, int64_t K, int rank, const void *X,
                       const void *A, const void *B, const void *C, int mode, void *out,
                       void *stream) {
  if (I < 1 || J < 1 || K < 1 || rank < 1 || mode < 0 || mode > 2 || !X || !out) {
    set_error("invalid dense_mttkrp arguments");
    return CPFIT_EINVAL;
  }
  const void *F1 = mode == 0 ? B : A;
  const void *F2 = mode == 2 ? B : C;
  if (!F1 || !F2) {
    set_error("dense_mttkrp: missing factor for mode %d", mode);
    return CPFIT_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    return dmma::run(mode, I, J, K, rank, (const double *)X, (const double *)F1,
                     (const double *)F2, (double *)out, s);
  if (dtype == CPFIT_F32)
    return dense_tc_run(mode, I, J, K, rank, (const float *)X, (const float *)F1,
                        (const float *)F2, (float *)out, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_dense_xc(int dtype, int64_t I, int64_t J, int64_t K, int rank, const void *X,
                   const void *C, void *T, void *stream) {
  if (I < 1 || J < 1 || K < 1 || rank < 1 || !X || !C || !T) {
    set_error("invalid dense_xc arguments");
    return CPFIT_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == CPFIT_F64)
    return dmma::run(3, I, J, K, rank, (const double *)X, nullptr, (const double *)C,
                     (double *)T, s);
  if (dtype == CPFIT_F32)
    return dense_tc_run(3, I, J, K, rank, (const float *)X, nullptr, (const float *)C,
                        (float *)T, s);
  set_error("unknown dtype %d", dtype);
  return CPFIT_EINVAL;
}

int cpfit_dense_gram(int dtype, int nfactors, const int64_t *rows, int rank,
                     const void *const *factors, void *G, void *stream) {
  if (nfactors < 1 || nfactors > CPFIT_MAXN || rank < 1 || !rows || !factors || !G) {
    set_error("invalid dense_gram arguments");
    return CPFIT_EINVAL;
  }
  CpfitDims d{};
  for (int f = 0; f < nfactors; ++f) d.d[f] = rows[f];
  cudaStream_t s = (cudaStream_t)stream;
  if (rank > 1024) {
    set_error("dense_gram: rank %d > 1024", rank);
    return CPFIT_EINVAL;
  }
  const int S = 256 / rank > 0 ? 256 / rank : 1;
  const int threads = rank * S;
  const size_t shm = (size_t)threads * sizeof(double);
  if (dtype == CPFIT_F64) {
    CpfitCoordPtrs<double> F{};
    for (int f = 0; f < nfactors; ++f) F.p[f] = (const double *)factors[f];
    dense_gram_kernel<double><<<rank, threads, shm, s>>>(nfactors, d, rank, F, (double *)G);
  } else if (dtype == CPFIT_F32) {
    CpfitCoordPtrs<float> F{};
    for (int f = 0; f < nfactors; ++f) F.p[f] = (const float *)factors[f];
    dense_gram_kernel<float><<<rank, threads, shm, s>>>(nfactors, d, rank, F, (float *)G);
  } else {
    set_error("unknown dtype %d", dtype);
    return CPFIT_EINVAL;
  }
  CPFIT_LAUNCH_CHECK("dense_gram");
  return CPFIT_OK;
}

}  // extern "C"
