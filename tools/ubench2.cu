// generic-pointer vs shared-state-space load latency / throughput (cycles), one SM
#include <cstdio>
__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
  return c;
}
__global__ void k(long long* out, double* gbuf, int sel) {
  extern __shared__ double sh[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sh[i] = (double)((i * 37 + 11) % 8192);
  __syncthreads();
  double* gp = sel ? gbuf : sh;   // generic pointer that the compiler cannot resolve
  int idx = threadIdx.x;
  long long t0 = clk();
  for (int r = 0; r < 64; ++r) idx = (int)gp[idx];
  long long t1 = clk();
  int idx2 = threadIdx.x;
  for (int r = 0; r < 64; ++r) idx2 = (int)sh[idx2];
  long long t2 = clk();
  // throughput: 8 independent chains per thread
  int a[8];
  for (int j = 0; j < 8; ++j) a[j] = (threadIdx.x * 8 + j) & 8191;
  __syncthreads();
  long long t3 = clk();
  for (int r = 0; r < 32; ++r)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = (int)gp[a[j]];
  __syncthreads();
  long long t4 = clk();
  for (int r = 0; r < 32; ++r)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = (int)sh[a[j]];
  __syncthreads();
  long long t5 = clk();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / 64; out[1] = (t2 - t1) / 64; out[2] = (t4 - t3) / 32; out[3] = (t5 - t4) / 32;
    out[4] = idx + idx2 + a[0] + a[7];
  }
}
int main() {
  long long* o; double* g;
  cudaMalloc(&o, 64); cudaMalloc(&g, 8192 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  long long r[8];
  for (int nt : {32, 384}) {
    for (int rep = 0; rep < 2; ++rep) k<<<1, nt, 65536>>>(o, g, 0);
    cudaMemcpy(r, o, 40, cudaMemcpyDeviceToHost);
    printf("threads %d: generic->smem chase %lld | lds chase %lld | generic 8-chain round %lld | lds 8-chain round %lld cycles\n", nt, r[0], r[1], r[2], r[3]);
  }
}
