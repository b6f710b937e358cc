// Latency microbenchmarks on one SM (cycles): dependent fp64 ops, a 6x6 Cholesky on one thread,
// __syncthreads with 256 threads, shared / L2 load round trips.  nvcc -arch=sm_100a tools/ubench.cu
#include <cstdio>
__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
  return c;
}
__global__ void k(long long* out, double* gbuf, double seed) {
  __shared__ double sh[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = (double)((i * 7) % 1024);
  __syncthreads();
  double a = seed;
  long long t0 = clk();
#pragma unroll
  for (int i = 0; i < 64; ++i) a = fma(a, 1.0000001, 1e-12);
  asm volatile("" ::"d"(a));
  long long t1 = clk();
  double c = a;
#pragma unroll
  for (int i = 0; i < 16; ++i) c = rsqrt(c + 2.0);
  asm volatile("" ::"d"(c));
  long long t2 = clk();
  double d = c;
#pragma unroll
  for (int i = 0; i < 16; ++i) d = 1.0 / (d + 2.0);
  asm volatile("" ::"d"(d));
  long long t3 = clk();
  // 6x6 Cholesky (SPD) one thread, registers
  double m[6][6];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) m[i][j] = (i == j ? 10.0 + d : 0.5 + 0.01 * (i + j) * d);
  long long t4 = clk();
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    double piv = m[j][j];
#pragma unroll
    for (int k2 = 0; k2 < j; ++k2) piv = fma(-m[j][k2], m[j][k2], piv);
    const double inv = rsqrt(piv);
    m[j][j] = piv * inv;
#pragma unroll
    for (int i = j + 1; i < 6; ++i) {
      double s = m[i][j];
#pragma unroll
      for (int k2 = 0; k2 < j; ++k2) s = fma(-m[i][k2], m[j][k2], s);
      m[i][j] = s * inv;
    }
  }
  asm volatile("" ::"d"(m[5][5]), "d"(m[5][4]));
  long long t5 = clk();
  __syncthreads();
  long long t6 = clk();
  for (int r = 0; r < 16; ++r) __syncthreads();
  long long t7 = clk();
  // shared-memory pointer chase
  int idx = threadIdx.x & 7;
  for (int r = 0; r < 32; ++r) idx = (int)sh[idx];
  long long t8 = clk();
  // L2 pointer chase (gbuf holds indices, stride 4096 doubles)
  double p = gbuf[threadIdx.x];
  int gi = (int)p;
  long long t9 = clk();
  for (int r = 0; r < 16; ++r) gi = (int)__ldcg(gbuf + gi);
  long long t10 = clk();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / 64; out[1] = (t2 - t1) / 16; out[2] = (t3 - t2) / 16; out[3] = t5 - t4;
    out[4] = t7 - t6; out[5] = (t8 - t7) / 32; out[6] = (t10 - t9) / 16;
    out[7] = (long long)(m[5][5] + idx + gi);
  }
}
int main() {
  long long* o;
  double* g;
  cudaMalloc(&o, 16 * 8);
  const int n = 1 << 22;
  cudaMalloc(&g, n * 8);
  double* h = new double[n];
  for (int i = 0; i < n; ++i) h[i] = (double)((i + 4096 * 33) % n);
  cudaMemcpy(g, h, n * 8, cudaMemcpyHostToDevice);
  long long r[16];
  for (int rep = 0; rep < 3; ++rep) k<<<1, 256>>>(o, g, 1.3);
  cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
  printf("dfma %lld | rsqrt %lld | div %lld | chol6 (1 thread) %lld | 16x syncthreads(256) %lld | lds chase %lld | L2 chase %lld cycles\n",
         r[0], r[1], r[2], r[3], r[4], r[5], r[6]);
}
