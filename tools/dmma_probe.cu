// DMMA.8x8x4 issue-rate probe (B200): FP64 tensor throughput vs warps per SM
// sub-partition and independent accumulator chains per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o variants/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void probe(double *out, int iters, double a0, double b0) {
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0.0;
  double a = a0 + threadIdx.x, b = b0 - threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
void run(int warps_per_sm, double *out) {
  int sms = 148;
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<NACC><<<sms, warps_per_sm * 32>>>(out, 100, 1.0, 2.0);
  cudaEventRecord(e0);
  probe<NACC><<<sms, warps_per_sm * 32>>>(out, iters, 1.0, 2.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 8 * 8 * 4 * (double)NACC * iters * warps_per_sm * sms;
  printf("{\"nacc\": %d, \"warps_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f, \"cycles_per_dmma_per_smsp\": %.2f}\n",
         NACC, warps_per_sm, ms, flops / ms / 1e9,
         ms * 1e-3 * 1.965e9 / ((double)NACC * iters * warps_per_sm / 4.0));
}

int main() {
  double *out;
  cudaMalloc(&out, 148 * 1024 * sizeof(double));
  for (int w : {4, 8, 12, 16, 32}) {
    run<1>(w, out);
    run<2>(w, out);
    run<4>(w, out);
    run<10>(w, out);
  }
  return 0;
}
