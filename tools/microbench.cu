// Micro-benchmarks of the per-supernode device routines (one warp, shared memory), clock64 cycles.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
#include <cstdio>
#include "../paper_2207_09442_b200/csrc/phases.cuh"
using namespace dnls;

__global__ void kbench(long long* out, double* gbuf) {
  __shared__ double P[64 * 19];
  __shared__ double xinv[36];
  __shared__ double xs[64];
  __shared__ int fail;
  const int lane = threadIdx.x;
  const int m = 18, ld = 19, w = 6;
  for (int i = lane; i < ld * w; i += 32) P[i] = (i % ld == i / ld) ? 10.0 : 0.01 * (i % 7);
  for (int i = lane; i < 64; i += 32) xs[i] = 1.0 + i;
  if (lane == 0) fail = 0;
  __syncwarp();
  long long t0 = clock64();
  panel_factor<6>(P, m, ld, w, 1e-30, Team{lane, 32, 0}, &fail, xinv);
  __syncwarp();
  long long t1 = clock64();
  warp_trsv_lower<1>(P, ld, w, xs);
  __syncwarp();
  long long t2 = clock64();
  double r = 0;
  for (int k = 0; k < 6; ++k) r += rsqrt(P[k * ld + k] + lane);
  long long t3 = clock64();
  double q = 1.0;
  #pragma unroll 1
  for (int k = 0; k < 16; ++k) q = rsqrt(q + 1.0);
  long long t4 = clock64();
  double z = 1.0;
  #pragma unroll 1
  for (int k = 0; k < 16; ++k) z = 1.0 / (z + 1.0);
  long long t5 = clock64();
  double y = 1.0;
  #pragma unroll 1
  for (int k = 0; k < 16; ++k) y = fma(y, 1.0000001, 1e-9);
  long long t6 = clock64();
  double gl = 0;
  #pragma unroll 1
  for (int k = 0; k < 16; ++k) gl = gbuf[(int)(gl * 0) + k * 1024 + lane];
  long long t7 = clock64();
  volatile double* vs = P;
  double sl = 0;
  #pragma unroll 1
  for (int k = 0; k < 16; ++k) sl = vs[(int)sl * 0 + k];
  long long t8 = clock64();
  if (lane == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = (t4 - t3) / 16; out[4] = (t5 - t4) / 16;
    out[5] = (t6 - t5) / 16; out[6] = (t7 - t6) / 16; out[7] = (t8 - t7) / 16;
    out[8] = (long long)(r + q + z + y + gl + sl);
  }
}

int main() {
  long long* d;
  double* gb;
  cudaMalloc(&d, 16 * sizeof(long long));
  cudaMalloc(&gb, 1 << 24);
  cudaMemset(gb, 0, 1 << 24);
  for (int rep = 0; rep < 3; ++rep) kbench<<<1, 32>>>(d, gb);
  long long h[16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("panel_factor(6x18): %lld cycles\ntrsv_lower(w=6): %lld\n6 rsqrt (independent): %lld\n"
         "rsqrt latency: %lld\ndiv latency: %lld\nfma latency: %lld\nglobal load latency (L2 miss->hit): %lld\n"
         "smem load latency: %lld\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  return 0;
}
