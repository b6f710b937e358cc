// Latency of one single-pose dense step (chol_regs + TRSM rows + store + y = L^-1 t) on a
// shared-memory panel, as in level_factor_teams, with a barrier per step (cycles per step).
#include <cstdio>
#include "../paper_2207_09442_b200/csrc/phases.cuh"
using namespace dnls;
__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)::"memory");
  return c;
}
template <int MODE>
__global__ void k(long long* out, int m) {
  constexpr int D = 6;
  __shared__ double P[64 * 6 + 64];
  __shared__ double xs[8];
  const int ld = m | 1;
  for (int i = threadIdx.x; i < ld * 6; i += blockDim.x) {
    const int c = i / ld, r = i - c * ld;
    P[i] = (r == c) ? 10.0 : 0.01 * ((r * 7 + c * 3) % 11);
  }
  if (threadIdx.x < 8) xs[threadIdx.x] = 1.0;
  __syncthreads();
  long long t0 = clk();
  for (int rep = 0; rep < 64; ++rep) {
    const int rank = threadIdx.x;
    if (MODE == 0) {   // warp: redundant chol, rows, lane 0 store + trsv
      if (rank < 32) {
        double a[D][D], iv[D];
        const bool bad = chol_regs<D>(P, ld, 0, 1e-13, a, iv);
        for (int r = D + rank; r < m; r += 32) trsm_row_regs<D>(P, ld, 0, r, a, iv);
        if (rank == 0) {
          store_diag<D>(P, ld, 0, a, iv);
          double y[D];
          for (int q = 0; q < D; ++q) {
            double s = xs[q];
            for (int kk = 0; kk < q; ++kk) s = fma(-a[q][kk], y[kk], s);
            y[q] = s * iv[q];
          }
          for (int q = 0; q < D; ++q) xs[q] = y[q] * 1e-3 + 1.0;
          if (bad) xs[7] = 1.0;
        }
      }
    } else if (MODE == 1) {   // chol only (lane 0), store
      if (rank == 0) {
        double a[D][D], iv[D];
        chol_regs<D>(P, ld, 0, 1e-13, a, iv);
        store_diag<D>(P, ld, 0, a, iv);
      }
    } else {   // barrier only
    }
    __syncthreads();
    // restore the diagonal block so every repetition factors the same SPD matrix
    if (threadIdx.x < 36) {
      const int c = threadIdx.x / 6, r = threadIdx.x % 6;
      if (r >= c) P[c * ld + r] = (r == c) ? 10.0 : 0.01 * ((r * 7 + c * 3) % 11);
    }
    __syncthreads();
  }
  long long t1 = clk();
  if (threadIdx.x == 0) out[MODE] = (t1 - t0) / 64;
}
int main() {
  long long* o;
  cudaMalloc(&o, 64);
  long long r[4];
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 384>>>(o, 30);
    k<1><<<1, 384>>>(o, 30);
    k<2><<<1, 384>>>(o, 30);
  }
  cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost);
  printf("per step (cycles): warp chol+trsm+store+trsv %lld | lane-0 chol+store %lld | 2 barriers + restore %lld\n",
         r[0], r[1], r[2]);
}
