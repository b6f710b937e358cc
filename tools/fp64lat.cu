// fp64 latency microbenchmark (one warp), cycles per dependent operation
#include <cstdio>
__global__ void k(long long* out, double seed) {
  double a = seed, b = seed * 0.5;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) a = fma(a, 1.0000001, 1e-12);
  long long t1 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) b = b * 1.0000001;
  long long t2 = clock64();
  double c = seed;
#pragma unroll
  for (int i = 0; i < 16; ++i) c = rsqrt(c + 2.0);
  long long t3 = clock64();
  double d = seed;
#pragma unroll
  for (int i = 0; i < 16; ++i) d = 1.0 / (d + 2.0);
  long long t4 = clock64();
  double e = seed;
#pragma unroll
  for (int i = 0; i < 16; ++i) e = sqrt(e + 2.0);
  long long t5 = clock64();
  double f = seed;
#pragma unroll
  for (int i = 0; i < 16; ++i) f = sin(f) + 0.5;
  long long t6 = clock64();
  double h = seed;
#pragma unroll
  for (int i = 0; i < 16; ++i) h = atan2(h, 1.5) + 0.5;
  long long t7 = clock64();
  float fa = (float)seed;
#pragma unroll
  for (int i = 0; i < 64; ++i) fa = fmaf(fa, 1.0000001f, 1e-7f);
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / 64; out[1] = (t2 - t1) / 64; out[2] = (t3 - t2) / 16; out[3] = (t4 - t3) / 16;
    out[4] = (t5 - t4) / 16; out[5] = (t6 - t5) / 16; out[6] = (t7 - t6) / 16; out[7] = (t8 - t7) / 64;
    out[8] = (long long)(a + b + c + d + e + f + h + fa);
  }
}
int main() {
  long long* d; cudaMalloc(&d, 16 * 8);
  for (int r = 0; r < 3; ++r) k<<<1, 32>>>(d, 1.3);
  long long h[16]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("fp64 fma %lld, mul %lld, rsqrt %lld, div %lld, sqrt %lld, sin %lld, atan2 %lld | fp32 fma %lld cycles\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
}
