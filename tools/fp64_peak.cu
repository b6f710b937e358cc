// fp64 peak probes for the roofline denominators (SURVEY.md §8(d) "fp64 peak"):
//   dfma: every thread runs 8 independent FMA chains (no memory), grid = 148 x 8 CTAs x 256 threads
//   dmma: mma.sync.aligned.m8n8k4.row.col.f64 (the sm_80+ fp64 tensor-core MMA, still executed on sm_100a)
//         with 4 independent accumulators per warp, same grid
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu
// prints one JSON object: {"dfma_tflops": ..., "dmma_tflops": ...} (best of 5, CUDA events)
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double* out, double a0, double b0) {
  double a = a0 + threadIdx.x * 1e-6, b = b0 - threadIdx.x * 1e-6;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll 1
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best_f = 1e30f, best_m = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(d, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r) best_f = ms < best_f ? ms : best_f;
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(d, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (r) best_m = ms < best_m ? ms : best_m;
  }
  const double thr = (double)blocks * threads;
  const double f_flops = thr * ITERS * 8 * 2.0;                  // 8 chains x 1 FMA
  const double m_flops = thr / 32.0 * (ITERS / 4) * 4 * 8 * 8 * 4 * 2.0;   // per warp: 4 MMAs of 8x8x4
  printf("{\"sms\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"dfma_ms\": %.4f, \"dmma_ms\": %.4f, "
         "\"err\": \"%s\"}\n",
         sms, f_flops / best_f / 1e9, m_flops / best_m / 1e9, best_f, best_m, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
