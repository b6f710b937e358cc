// Per-element device phases of one GN/LM iteration.  One CUDA block ("CTA"), or a cluster of CL
// CTAs for few large problems, owns one batch element; every phase below is executed
// cooperatively by its threads.  Phases:
//   linearize_phase a1+a2: per-cost residual + compact Jacobian, single-writer assembly of H, b, S
//   factor_phase    a3: supernodal left-looking Cholesky, level-synchronous (+ fused y = L^-1 b)
//   solve_phase     a4: backward (and standalone forward) substitution
//   retract_phase   a5: T <- T Exp(-alpha delta)
//   objective_phase    S(theta) only (LM trial, final objective)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lie.cuh"
#include "symbolic.h"

namespace dnls {

// ----------------------------------------------------------------------------- tracing (debug builds)
// Compiled with -DDNLS_TRACE: thread 0 of block 0 records (tag, clock64) pairs so the fused
// kernel's time can be attributed to phases / levels (tools/trace.py).  No-op otherwise.
#ifdef DNLS_TRACE
__device__ long long g_trace[2 * 8192];
__device__ int g_trace_n;
#define DNLS_TRACE_POINT(tag)                                         \
  do {                                                                \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                        \
      int i_ = g_trace_n;                                             \
      if (i_ < 8192) {                                                \
        g_trace[2 * i_] = (tag);                                      \
        g_trace[2 * i_ + 1] = clock64();                              \
        g_trace_n = i_ + 1;                                           \
      }                                                               \
    }                                                                 \
  } while (0)
#else
#define DNLS_TRACE_POINT(tag) \
  do {                        \
  } while (0)
#endif

// -DDNLS_LIN_PROBE: thread 0 of block 0 accumulates the cycles of linearisation segments into
// g_probe (clock deltas kept in registers -- no dependent global reads on the measured path)
#ifdef DNLS_LIN_PROBE
__device__ unsigned long long g_probe[8];
#define DNLS_PROBE_NOW(v) const long long v = clock64()
#define DNLS_PROBE_ADD(i, a, b) \
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_probe[i], (unsigned long long)((b) - (a)))
#else
#define DNLS_PROBE_NOW(v)
#define DNLS_PROBE_ADD(i, a, b)
#endif

// device view of the symbolic analysis (int32 arrays uploaded once per graph; only what the numeric
// kernels read -- the update / solve lists travel inside the per-level descriptor packets `pk`)
struct DevGraph {
  int D, N, E, P, S, storage, n;
  int x_smem;     // 1: the solution vector x lives in shared memory (offset 0, n_pad doubles)
  int n_pad;      // n rounded up to an even count (16-byte alignment of the next area)
  int res_lo;     // storage offsets >= res_lo are resident in shared memory (top levels)
  int res_n;      // resident doubles (even)
  int stage_n;    // doubles of the level-staging area (largest staged level prefix)
  const int *perm, *iperm, *edges, *prior_vars;
  const int *sn_first, *sn_m, *sn_ld, *sn_w, *sn_off;   // per supernode: panel geometry and offset
  const int *level_off, *level_stage_hi;                 // per level: storage range, staged prefix end
  const int *snr_ptr, *snr;                              // per supernode: below-diagonal pose rows
  const int *blk_off, *blk_ld, *blk_cptr, *blk_con;      // per storage block: offset, ld, contributing slots
  const int *bc_ptr, *bc;                                // per pose: its cost slots (fixed gather order)
  const int4* slot_desc;            // 3 int4 per cost slot (block offsets / lds of its H blocks)
  const int* pose_sn;               // supernode of each permuted pose column
  const int* dup_blk;               // blk_* indices of off-diagonal blocks shared by several edges
  int ndup;
  const int* pk;       // per-level descriptor packets (ints), pk_off[npk+1] offsets
  const int* pk_off;
  int pk_max;          // ints of the largest packet
  int npk;             // number of packets (levels split into size-bounded chunks)
};

// ---- CTA groups: CL CTAs of one thread-block cluster share one batch element (CL == 1: the CTA
// alone).  Item loops run over the group's CL * NT threads; gsync<CL>() is the group barrier
// (a cluster barrier with release/acquire semantics orders the global-memory writes of all its
// CTAs, few large problems).
template <int CL>
__device__ __forceinline__ int crank() {
  if constexpr (CL == 1) {
    return 0;
  } else {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return (int)r;
  }
}
// The non-.aligned barrier form tolerates warps that have not reconverged after divergent item
// loops (the compiler does not reconverge around inline asm); the cluster-scope fence after the
// wait invalidates this SM's L1 (CCTL.IVALL) so global data written by the other CTAs is re-read.
template <int CL>
__device__ __forceinline__ void gsync() {
  if constexpr (CL == 1) {
    __syncthreads();
  } else {
#ifdef DNLS_STRONG_GSYNC
    __threadfence();
#endif
#ifndef DNLS_NO_CLUSTER_FENCE
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;\n\tfence.acq_rel.cluster;" :::
                 "memory");
#else
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
#endif
#ifdef DNLS_STRONG_GSYNC
    __threadfence();
#endif
  }
}

// problem inputs (see dnls_problem)
struct DevProb {
  double* poses;
  const double* meas;
  const double* prior_meas;
  long long pm_bstride;
  const double* w_edge;
  long long we_bstride;
  const double* w_prior;
  long long wp_bstride;
  const double* radius;   // Welsch radius (nullptr: quadratic costs), readings W1-W3
  long long r_bstride;
};

// per-call workspace views (device)
struct DevWs {
  double* L;      // [B][storage]
  double* x;      // [B][n]   rhs / solution (permuted order)
  double* bsave;  // [B][n]   Dogleg: the gradient b = J^T r of the current linearisation
  double* jac;    // [B][E+P][JS]  weighted J_i, J_j, r per cost slot
  double* cost;   // [B][E+P]      1/2 |r|^2 per slot (or weight gradient in backward)
  double* rgrad;  // [B][E+P]      per-slot radius gradient (backward with a Welsch kernel)
  double* clred;  // [B][2 * CL]   cross-CTA exchange of a cluster (max diagonal, failure flags)
  double* trial;  // [B][N][PS]    LM trial poses
  double* S;      // [B] current objective
  double* Sprev;  // [B]
  double* lam;    // [B]
  double* maxd;   // [B] max diagonal of the matrix last assembled/imported
  int* st;        // [B] status
  int* it;        // [B] iterations
  // unroll / truncated history (backward_mode UNROLL / TRUNCATED), `keep` iterations per element in a
  // ring (iteration k in slot k % keep), element-major:
  int keep;
  double* hT;     // [B][keep][N][PS]   theta_k
  double* hd;     // [B][keep][n]       delta_k (permuted order)
  double* hL;     // [B][keep][storage] the factor of H(theta_k)
};

__host__ __device__ constexpr int pad4(int x) { return (x + 3) & ~3; }
template <int D>
struct Scr;
template <int D>
struct GT {
  static constexpr int PS = (D == 6) ? 12 : 6;   // doubles per pose
  static constexpr int JS = Scr<D>::SIZE;   // scratch doubles per cost slot
};

// Factor storage view.  Offsets >= rlo (the top elimination-tree levels) are RESIDENT in
// shared memory `r`; offsets in [lo, hi) (the level being processed) are STAGED in shared
// memory `s`; everything else is in global memory `g`.  Generic pointers serve all three.
struct LView {
  double* g;
  double* r;
  int rlo;
  double* s;
  int lo, hi;
  __device__ __forceinline__ double* at(int off) const {
    return off >= rlo ? r + (off - rlo) : ((off >= lo && off < hi) ? s + (off - lo) : g + off);
  }
  __device__ __forceinline__ LView level(double* stage, int l0, int h0) const {
    LView v = *this;
    v.s = stage;
    v.lo = l0;
    v.hi = h0;
    return v;
  }
};

// CTA-cooperative copies of a contiguous range (16-byte vectors when both ends are aligned)
template <int NT>
__device__ __forceinline__ void copy_range(double* __restrict__ dst, const double* __restrict__ src, int n) {
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const int n2 = n >> 1;
    double2* d2 = reinterpret_cast<double2*>(dst);
    const double2* s2 = reinterpret_cast<const double2*>(src);
    for (int i = threadIdx.x; i < n2; i += NT) d2[i] = s2[i];
    if ((n & 1) && threadIdx.x == 0) dst[n - 1] = src[n - 1];
  } else {
    for (int i = threadIdx.x; i < n; i += NT) dst[i] = src[i];
  }
}

// ----------------------------------------------------------------------------- TMA bulk copies
// 1-D bulk async copy global -> shared (cp.async.bulk, completion through an mbarrier with a
// transaction count).  Sizes / addresses are 16-byte multiples (panels are padded to even
// double counts).  One elected thread issues; every thread waits on the mbarrier phase.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* mbar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  const uint32_t a = smem_u32(mbar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}
// CTA-wide: every thread orders its prior generic-proxy accesses (global writes of the panels,
// shared reads of the staging area) before the async proxy, barrier, thread 0 issues the bulk
// copy, every thread waits on the mbarrier phase (phase toggles per use).
template <int NT>
__device__ __forceinline__ void bulk_load(double* dst, const double* src, int ndoubles, uint64_t* mbar,
                                          uint32_t& phase) {
  __syncthreads();
  if (ndoubles <= 0) return;
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async;" ::: "memory");
    const uint32_t bytes = (uint32_t)ndoubles * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
    for (uint32_t o = 0; o < bytes; o += 65536u) {
      const uint32_t sz = min(65536u, bytes - o);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(reinterpret_cast<const char*>(dst) + o)),
          "l"(reinterpret_cast<const char*>(src) + o), "r"(sz), "r"(smem_u32(mbar))
          : "memory");
    }
  }
  mbar_wait(mbar, phase);
  phase ^= 1u;
}

// ============================================================================= cost evaluation
// Unweighted cost c and Jacobians of a Between edge / prior from poses held in registers
// (SURVEY.md §8(a) a1): c = Log(Z^-1 T_i^-1 T_j), C_j = Jr^-1(c), C_i = -Jr^-1(c) Ad(T_j^-1 T_i);
// prior c = Log(Z^-1 T), C = Jr^-1(c).  Ci/Cj row-major D x D.
__device__ __forceinline__ void edge_eval(const dev::SE3& Ti, const dev::SE3& Tj, const dev::SE3& Z, double* c,
                                          double* Ci, double* Cj, bool need_jac) {
  using namespace dev;
  SE3 X = se3_between(Ti, Tj);
  se3_log(se3_between(Z, X), c);
  if (!need_jac) return;
  M3 Ji, U;
  se3_jr_inv(c, Ji, U);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      Cj[r * 6 + q] = Ji.m[r][q];
      Cj[r * 6 + q + 3] = U.m[r][q];
      Cj[(r + 3) * 6 + q] = 0.0;
      Cj[(r + 3) * 6 + q + 3] = Ji.m[r][q];
    }
  // Ci = -Jr^-1(c) Ad(Tj^-1 Ti),  Ad(M) = [[R, t^ R], [0, R]]
  SE3 M = se3_between(Tj, Ti);
  M3 R, tR;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) R.m[r][q] = M.R[r][q];
  tR = mul(hat(M.t), R);
  M3 JR = mul(Ji, R);
  M3 JtR = mul(Ji, tR);
  M3 UR = mul(U, R);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      Ci[r * 6 + q] = -JR.m[r][q];
      Ci[r * 6 + q + 3] = -(JtR.m[r][q] + UR.m[r][q]);
      Ci[(r + 3) * 6 + q] = 0.0;
      Ci[(r + 3) * 6 + q + 3] = -JR.m[r][q];
    }
}
__device__ __forceinline__ void prior_eval(const dev::SE3& T, const dev::SE3& Z, double* c, double* C, bool need_jac) {
  using namespace dev;
  se3_log(se3_between(Z, T), c);
  if (!need_jac) return;
  M3 Ji, U;
  se3_jr_inv(c, Ji, U);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      C[r * 6 + q] = Ji.m[r][q];
      C[r * 6 + q + 3] = U.m[r][q];
      C[(r + 3) * 6 + q] = 0.0;
      C[(r + 3) * 6 + q + 3] = Ji.m[r][q];
    }
}
__device__ __forceinline__ void edge_eval(const dev::SE2& Ti, const dev::SE2& Tj, const dev::SE2& Z, double* c,
                                          double* Ci, double* Cj, bool need_jac) {
  using namespace dev;
  se2_log(se2_between(Z, se2_between(Ti, Tj)), c);
  if (!need_jac) return;
  double J[3][3];
  se2_jr_inv(c, J);
  SE2 M = se2_between(Tj, Ti);
  // Ad(M) = [[R, (t_y, -t_x)^T], [0, 1]]
  double Ad[3][3] = {{M.R[0][0], M.R[0][1], M.t[1]}, {M.R[1][0], M.R[1][1], -M.t[0]}, {0.0, 0.0, 1.0}};
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      Cj[r * 3 + q] = J[r][q];
      Ci[r * 3 + q] = -(J[r][0] * Ad[0][q] + J[r][1] * Ad[1][q] + J[r][2] * Ad[2][q]);
    }
}
__device__ __forceinline__ void prior_eval(const dev::SE2& T, const dev::SE2& Z, double* c, double* C, bool need_jac) {
  using namespace dev;
  se2_log(se2_between(Z, T), c);
  if (!need_jac) return;
  double J[3][3];
  se2_jr_inv(c, J);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) C[r * 3 + q] = J[r][q];
}
template <int D>
struct PoseT {
  using T = dev::SE3;
  static __device__ __forceinline__ T load(const double* p) { return dev::se3_load(p); }
};
template <>
struct PoseT<3> {
  using T = dev::SE2;
  static __device__ __forceinline__ T load(const double* p) { return dev::se2_load(p); }
};

// Unweighted cost c and Jacobians of slot `slot` (edge e < E, else prior slot - E) at poses Tb.
// Ci/Cj are row-major D x D.  For priors only Ci is written.
template <int D>
__device__ __forceinline__ void eval_slot(const DevGraph& g, const DevProb& pr, const double* Tb, int b,
                                          int slot, double* c, double* Ci, double* Cj, bool need_jac) {
  constexpr int PS = GT<D>::PS;
  using P = PoseT<D>;
  if (slot < g.E) {
    const int i = g.edges[2 * slot], j = g.edges[2 * slot + 1];
    edge_eval(P::load(Tb + (size_t)i * PS), P::load(Tb + (size_t)j * PS),
              P::load(pr.meas + ((size_t)b * g.E + slot) * PS), c, Ci, Cj, need_jac);
  } else {
    const int k = slot - g.E;
    prior_eval(P::load(Tb + (size_t)g.prior_vars[k] * PS),
               P::load(pr.prior_meas + (size_t)b * pr.pm_bstride + (size_t)k * PS), c, Ci, need_jac);
  }
}

template <int D>
__device__ __forceinline__ double slot_weight(const DevGraph& g, const DevProb& pr, int b, int slot) {
  return slot < g.E ? pr.w_edge[(size_t)b * pr.we_bstride + slot]
                    : pr.w_prior[(size_t)b * pr.wp_bstride + (slot - g.E)];
}

// Cost of a slot from its weighted squared error s = ||w c||^2 (readings A6, W1-W2): returns the
// slot's objective term and sets psi, the IRLS weight of its Jacobian/residual (1 if quadratic).
//   quadratic: s / 2, psi = 1;   Welsch (edges, radius k): -k^2/2 expm1(-s/k^2), psi = e^{-s/k^2}
__device__ __forceinline__ double slot_cost(const DevGraph& g, const DevProb& pr, int b, int slot, double s,
                                            double& psi) {
  if (pr.radius == nullptr || slot >= g.E) {
    psi = 1.0;
    return 0.5 * s;
  }
  const double k = pr.radius[(size_t)b * pr.r_bstride];
  const double x = -s / (k * k);
  psi = exp(x);
  return -0.5 * k * k * expm1(x);
}

// deterministic CTA-wide sum of v[0..n) : warp 0 only, fixed summation order.  Returns the
// value on every thread of warp 0 (callers use lane 0).
__device__ __forceinline__ double warp0_sum(const double* v, int n) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s += v[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// objective only (LM trial / final objective without implicit)
template <int D, int NT, int CL = 1>
__device__ void objective_phase(const DevGraph& g, const DevProb& pr, const double* Tb, int b, double* cost_b) {
  const int nslot = g.E + g.P;
  for (int slot = crank<CL>() * NT + threadIdx.x; slot < nslot; slot += CL * NT) {
    double c[D];
    eval_slot<D>(g, pr, Tb, b, slot, c, nullptr, nullptr, false);
    const double w = slot_weight<D>(g, pr, b, slot);
    double n2 = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) n2 += (w * c[q]) * (w * c[q]);
    double psi;
    cost_b[slot] = slot_cost(g, pr, b, slot, n2, psi);
  }
}

// ---------------------------------------------------------------------------- fused linearisation
// Compact weighted-Jacobian form of one cost slot, kept in registers:
//  SE3: C_j = Jr^-1(c) = [[A, U], [0, A]],  C_i = -[[P, Q], [0, P]] with P = A R, Q = A t^R + U R
//       (R, t of T_j^-1 T_i); a prior has C = [[A, U], [0, A]].
//  SE2: full 3x3 C_j = Jr^-1(c), C_i = -C_j Ad(T_j^-1 T_i).
template <int D>
struct SlotJ;
template <>
struct SlotJ<6> {
  double c[6], A[3][3], U[3][3], P[3][3], Q[3][3], ww;
};
template <>
struct SlotJ<3> {
  double c[3], Cj[3][3], Ci[3][3], ww;
};

template <int D>
__device__ __forceinline__ void slot_jac(const DevGraph& g, const DevProb& pr, const double* Tb, int b, int slot,
                                         SlotJ<D>& J);
template <>
__device__ __forceinline__ void slot_jac<6>(const DevGraph& g, const DevProb& pr, const double* Tb, int b, int slot,
                                            SlotJ<6>& J) {
  using namespace dev;
  constexpr int PS = 12;
  dev::M3 Ji, U;
  if (slot < g.E) {
    const int i = g.edges[2 * slot], j = g.edges[2 * slot + 1];
    SE3 Ti = se3_load(Tb + (size_t)i * PS), Tj = se3_load(Tb + (size_t)j * PS);
    SE3 Z = se3_load(pr.meas + ((size_t)b * g.E + slot) * PS);
    se3_log(se3_between(Z, se3_between(Ti, Tj)), J.c);
    se3_jr_inv(J.c, Ji, U);
    SE3 M = se3_between(Tj, Ti);
    M3 R;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q) R.m[r][q] = M.R[r][q];
    const M3 AR = mul(Ji, R);
    const M3 AtR = mul(Ji, mul(hat(M.t), R));
    const M3 UR = mul(U, R);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        J.P[r][q] = AR.m[r][q];
        J.Q[r][q] = AtR.m[r][q] + UR.m[r][q];
      }
  } else {
    const int k = slot - g.E;
    SE3 T = se3_load(Tb + (size_t)g.prior_vars[k] * PS);
    SE3 Z = se3_load(pr.prior_meas + (size_t)b * pr.pm_bstride + (size_t)k * PS);
    se3_log(se3_between(Z, T), J.c);
    se3_jr_inv(J.c, Ji, U);
  }
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      J.A[r][q] = Ji.m[r][q];
      J.U[r][q] = U.m[r][q];
    }
  const double w = slot_weight<6>(g, pr, b, slot);
  J.ww = w * w;
}
template <>
__device__ __forceinline__ void slot_jac<3>(const DevGraph& g, const DevProb& pr, const double* Tb, int b, int slot,
                                            SlotJ<3>& J) {
  double Ci[9], Cj[9];
  eval_slot<3>(g, pr, Tb, b, slot, J.c, Ci, Cj, true);
  // a prior's Jacobian plays the role of C_j (block 0 / rhs side 0), as for SE3
  const bool edge = slot < g.E;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      J.Ci[r][q] = edge ? Ci[r * 3 + q] : 0.0;
      J.Cj[r][q] = edge ? Cj[r * 3 + q] : Ci[r * 3 + q];
    }
  const double w = slot_weight<3>(g, pr, b, slot);
  J.ww = w * w;
}

// (X^T Y)[a][q] for 3x3 blocks
__device__ __forceinline__ double tdot3(const double (&X)[3][3], const double (&Y)[3][3], int a, int q) {
  return fma(X[0][a], Y[0][q], fma(X[1][a], Y[1][q], X[2][a] * Y[2][q]));
}

// SE3 6x6 blocks of the compact Jacobian: which = 0: C_j^T C_j (or prior), 1: C_i^T C_i,
// 2: C_i^T C_j (row i, col j), 3: C_j^T C_i.  Entry (a, q), a, q in 0..5 (rho first).
__device__ __forceinline__ double se3_block(const SlotJ<6>& J, int which, int a, int q) {
  const int ba = a / 3, ra = a - 3 * ba, bq = q / 3, rq = q - 3 * bq;
  // column blocks: C_j: [A;0], [U;A]   C_i: -[P;0], -[Q;P]
  double v;
  if (which == 0) {   // [[A'A, A'U], [U'A, U'U + A'A]]
    if (ba == 0 && bq == 0) v = tdot3(J.A, J.A, ra, rq);
    else if (ba == 0) v = tdot3(J.A, J.U, ra, rq);
    else if (bq == 0) v = tdot3(J.U, J.A, ra, rq);
    else v = tdot3(J.U, J.U, ra, rq) + tdot3(J.A, J.A, ra, rq);
  } else if (which == 1) {   // [[P'P, P'Q], [Q'P, Q'Q + P'P]]
    if (ba == 0 && bq == 0) v = tdot3(J.P, J.P, ra, rq);
    else if (ba == 0) v = tdot3(J.P, J.Q, ra, rq);
    else if (bq == 0) v = tdot3(J.Q, J.P, ra, rq);
    else v = tdot3(J.Q, J.Q, ra, rq) + tdot3(J.P, J.P, ra, rq);
  } else if (which == 2) {   // -[[P'A, P'U], [Q'A, Q'U + P'A]]
    if (ba == 0 && bq == 0) v = -tdot3(J.P, J.A, ra, rq);
    else if (ba == 0) v = -tdot3(J.P, J.U, ra, rq);
    else if (bq == 0) v = -tdot3(J.Q, J.A, ra, rq);
    else v = -(tdot3(J.Q, J.U, ra, rq) + tdot3(J.P, J.A, ra, rq));
  } else {   // transpose of which == 2: (C_j^T C_i)[a][q] = (C_i^T C_j)[q][a]
    if (bq == 0 && ba == 0) v = -tdot3(J.P, J.A, rq, ra);
    else if (bq == 0) v = -tdot3(J.P, J.U, rq, ra);
    else if (ba == 0) v = -tdot3(J.Q, J.A, rq, ra);
    else v = -(tdot3(J.Q, J.U, rq, ra) + tdot3(J.P, J.A, rq, ra));
  }
  return J.ww * v;
}
__device__ __forceinline__ double se3_rhs(const SlotJ<6>& J, int side, int a) {
  // side 0: C_j^T c (or prior), side 1: C_i^T c
  const int ba = a / 3, ra = a - 3 * ba;
  const double* cr = J.c;
  const double* cw = J.c + 3;
  double v;
  if (side == 0)
    v = ba == 0 ? fma(J.A[0][ra], cr[0], fma(J.A[1][ra], cr[1], J.A[2][ra] * cr[2]))
                : fma(J.U[0][ra], cr[0], fma(J.U[1][ra], cr[1], J.U[2][ra] * cr[2])) +
                      fma(J.A[0][ra], cw[0], fma(J.A[1][ra], cw[1], J.A[2][ra] * cw[2]));
  else
    v = -(ba == 0 ? fma(J.P[0][ra], cr[0], fma(J.P[1][ra], cr[1], J.P[2][ra] * cr[2]))
                  : fma(J.Q[0][ra], cr[0], fma(J.Q[1][ra], cr[1], J.Q[2][ra] * cr[2])) +
                        fma(J.P[0][ra], cw[0], fma(J.P[1][ra], cw[1], J.P[2][ra] * cw[2])));
  return J.ww * v;
}
__device__ __forceinline__ double se2_block(const SlotJ<3>& J, int which, int a, int q) {
  double v = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double xa = (which == 0 || which == 3) ? J.Cj[k][a] : J.Ci[k][a];
    const double yq = (which == 0 || which == 2) ? J.Cj[k][q] : J.Ci[k][q];
    v = fma(xa, yq, v);
  }
  return J.ww * v;
}
__device__ __forceinline__ double se2_rhs(const SlotJ<3>& J, int side, int a) {
  double v = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) v = fma(side == 0 ? J.Cj[k][a] : J.Ci[k][a], J.c[k], v);
  return J.ww * v;
}
template <int D, class JT>
__device__ __forceinline__ double blk(const JT& J, int which, int a, int q) {
  if constexpr (D == 6) return se3_block(J, which, a, q);
  else return se2_block(J, which, a, q);
}
template <int D, class JT>
__device__ __forceinline__ double rhs(const JT& J, int side, int a) {
  if constexpr (D == 6) return se3_rhs(J, side, a);
  else return se2_rhs(J, side, a);
}

// Fused linearisation, single-writer:
//  1. zero the factor storage (fill blocks and the unused upper triangles of diagonal blocks);
//  2. thread per cost slot: compact Jacobian in registers, 1/2 |w c|^2 to cost_b; the slot's
//     off-diagonal H block J_row^T J_col is STORED directly (plain stores, no read-modify-write)
//     when the slot is the only edge between its two poses; its two diagonal contributions
//     J_i^T J_i, J_j^T J_j (lower triangles), its two J^T r parts (and a shared off-diagonal
//     block) go to the per-slot scratch `scr` (fire-and-forget stores, no barriers between slots);
//  3. one barrier, then thread per pose: its diagonal block and b segment are the sums of its
//     slots' scratch contributions in the fixed order of the symbolic list bc (deterministic, no
//     atomics), damped (lam > 0; damping 0: Marquardt diag *= 1 + lam, 1: diag += lam) and written
//     once; shared off-diagonal blocks are summed the same way.  Max diagonal -> s_red per warp.
template <int D>
struct Scr {   // per-slot scratch layout (doubles); every field starts on a 32-byte boundary so a
               // slot writes it with 256-bit stores (one L1 wavefront per 4 doubles instead of one
               // per double: the slots of a warp are 800 B apart, so every store is uncoalesced)
  static constexpr int NL = D * (D + 1) / 2;
  static constexpr int H0 = 0, H1 = pad4(NL), B0 = 2 * pad4(NL), B1 = B0 + pad4(D), HIJ = B1 + pad4(D);
  static constexpr int SIZE = pad4(HIJ + D * D);
};
__device__ __forceinline__ void st_v4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ void ld_v4(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p) : "memory");
}
// (q, a) of entry e of a packed lower triangle (column-major, a >= q); folds for constant e
__device__ __forceinline__ void lower_qa(int e, int D, int& q, int& a) {
  int qq = 0, rem = e;
  while (rem >= D - qq) {
    rem -= D - qq;
    ++qq;
  }
  q = qq;
  a = qq + rem;
}
template <int D, int WHICH, class JT>
__device__ __forceinline__ void store_lower_v4(const JT& J, double* o) {
  // nested constant-bound loops (fully unrolled: the J entries are indexed by constants, so J stays
  // in registers), flushed every four entries
  double buf[4] = {0.0, 0.0, 0.0, 0.0};
  int nb = 0, e0 = 0;
#pragma unroll
  for (int q = 0; q < D; ++q)
#pragma unroll
    for (int a = q; a < D; ++a) {
      buf[nb++] = blk<D>(J, WHICH, a, q);
      if (nb == 4) {
        st_v4(o + e0, buf[0], buf[1], buf[2], buf[3]);
        e0 += 4;
        nb = 0;
      }
    }
  if (nb > 0) st_v4(o + e0, buf[0], nb > 1 ? buf[1] : 0.0, nb > 2 ? buf[2] : 0.0, 0.0);
}
template <int D, int SIDE, class JT>
__device__ __forceinline__ void store_rhs_v4(const JT& J, double* o) {
#pragma unroll
  for (int a0 = 0; a0 < D; a0 += 4) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = (a0 + u < D) ? rhs<D>(J, SIDE, a0 + u) : 0.0;
    st_v4(o + a0, v[0], v[1], v[2], v[3]);
  }
}

// the slot's scratch contributions (lower triangles packed column-wise, then J^T r parts)
template <int D, class JT>
__device__ __forceinline__ void slot_blocks_edge(const JT& J, double* o) {
  using SC = Scr<D>;
  store_lower_v4<D, 1>(J, o + SC::H0);
  store_lower_v4<D, 0>(J, o + SC::H1);
  store_rhs_v4<D, 1>(J, o + SC::B0);
  store_rhs_v4<D, 0>(J, o + SC::B1);
}
template <int D, class JT>
__device__ __forceinline__ void slot_blocks_prior(const JT& J, double* o) {
  using SC = Scr<D>;
  store_lower_v4<D, 0>(J, o + SC::H0);
  store_rhs_v4<D, 0>(J, o + SC::B0);
}
template <int D, int WHICH, class JT>
__device__ __forceinline__ void slot_offdiag(const JT& J, double* O, int ld) {
  // each block column is D contiguous doubles: 128-bit stores where 16-byte aligned (the odd
  // leading dimensions alternate the alignment of consecutive columns)
#pragma unroll
  for (int q = 0; q < D; ++q) {
    double v[D];
#pragma unroll
    for (int a = 0; a < D; ++a) v[a] = blk<D>(J, WHICH, a, q);
    double* c = O + (size_t)q * ld;
    if ((reinterpret_cast<uintptr_t>(c) & 15) == 0) {
#pragma unroll
      for (int a = 0; a + 1 < D; a += 2) *reinterpret_cast<double2*>(c + a) = make_double2(v[a], v[a + 1]);
      if (D & 1) c[D - 1] = v[D - 1];
    } else {
      c[0] = v[0];
#pragma unroll
      for (int a = 1; a + 1 < D; a += 2) *reinterpret_cast<double2*>(c + a) = make_double2(v[a], v[a + 1]);
      if (!(D & 1)) c[D - 1] = v[D - 1];
    }
  }
}
template <int D, int NT, int CL = 1>
__device__ void linearize_phase(const DevGraph& g, const DevProb& pr, const double* Tb, int b, const LView& L,
                                double* x_b, double* cost_b, double* scr, double lam, int damping, double* s_red) {
  using SC = Scr<D>;
  constexpr int NL = SC::NL, GN = CL * NT;
  const int gt = crank<CL>() * NT + threadIdx.x;
  DNLS_PROBE_NOW(p0);
  {   // zero the global part with 256-bit stores (32-byte aligned body, scalar head / tail)
    const int head = min((int)(((32 - (reinterpret_cast<uintptr_t>(L.g) & 31)) & 31) >> 3), L.rlo);
    const int nbody = (L.rlo - head) >> 2;
    if (gt < head) L.g[gt] = 0.0;
    for (int i = gt; i < nbody; i += GN) st_v4(L.g + head + 4 * i, 0.0, 0.0, 0.0, 0.0);
    for (int i = head + 4 * nbody + gt; i < L.rlo; i += GN) L.g[i] = 0.0;
  }
  for (int i = L.rlo + gt; i < g.storage; i += GN) L.r[i - L.rlo] = 0.0;
  gsync<CL>();
  DNLS_PROBE_NOW(p1);
  DNLS_PROBE_ADD(0, p0, p1);
  DNLS_TRACE_POINT(210);
  const int nslot = g.E + g.P;
  for (int slot = gt; slot < nslot; slot += GN) {
    SlotJ<D> J;
#ifndef DNLS_SKIP_JAC
    slot_jac<D>(g, pr, Tb, b, slot, J);
#else
    J = SlotJ<D>{};
    J.ww = 1.0;
#endif
    double n2 = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) n2 = fma(J.c[q], J.c[q], n2);
    double psi;
    cost_b[slot] = slot_cost(g, pr, b, slot, J.ww * n2, psi);
    J.ww *= psi;   // IRLS rescaling of the slot's H blocks and J^T r (W2)
    const int4 d0 = g.slot_desc[3 * slot], d1 = g.slot_desc[3 * slot + 1], d2 = g.slot_desc[3 * slot + 2];
    const bool edge = d0.y >= 0;
    double* o = scr + (size_t)slot * SC::SIZE;
    // side 0 = endpoint i (a prior's pose: its Jacobian has the C_j form, block 0 / rhs 0).  The
    // block kinds are compile-time in every branch (a runtime `which` made the compiler evaluate
    // the four block formulas with predication)
    if (edge) {
      slot_blocks_edge<D>(J, o);
      double* O = d2.z ? L.at(d0.z) : o + SC::HIJ;
      const int ld = d2.z ? d1.z : D;
      if (d0.w) slot_offdiag<D, 3>(J, O, ld);   // row pose is j: C_j^T C_i
      else slot_offdiag<D, 2>(J, O, ld);        // row pose is i: C_i^T C_j
    } else {
      slot_blocks_prior<D>(J, o);
    }
  }
  DNLS_PROBE_NOW(p2);
  DNLS_PROBE_ADD(1, p1, p2);
  gsync<CL>();
  DNLS_PROBE_NOW(p3);
  DNLS_PROBE_ADD(2, p2, p3);
  DNLS_TRACE_POINT(220);
  // thread per pose: its diagonal block and b segment are the sums of its slots' scratch fields
  // (256-bit loads: every field is 32-byte aligned), fixed order of the symbolic list bc
  double mymax = 0.0;
  for (int p = gt; p < g.N; p += GN) {
    constexpr int NH = pad4(NL), NR = pad4(D);
    double h[NH], r[NR];
#pragma unroll
    for (int i = 0; i < NH; ++i) h[i] = 0.0;
#pragma unroll
    for (int a = 0; a < NR; ++a) r[a] = 0.0;
    const int c0 = g.bc_ptr[p], c1 = g.bc_ptr[p + 1];
    for (int c = c0; c < c1; ++c) {
      const int code = g.bc[c];
      const double* o = scr + (size_t)(code >> 1) * SC::SIZE;
      const int side = code & 1;
      const double* oh = o + (side ? SC::H1 : SC::H0);
      const double* orh = o + (side ? SC::B1 : SC::B0);
#pragma unroll
      for (int i = 0; i < NH; i += 4) {
        double v0, v1, v2, v3;
        ld_v4(oh + i, v0, v1, v2, v3);
        h[i] += v0;
        h[i + 1] += v1;
        h[i + 2] += v2;
        h[i + 3] += v3;
      }
#pragma unroll
      for (int a = 0; a < NR; a += 4) {
        double v0, v1, v2, v3;
        ld_v4(orh + a, v0, v1, v2, v3);
        r[a] += v0;
        r[a + 1] += v1;
        r[a + 2] += v2;
        r[a + 3] += v3;
      }
    }
    const int s = g.pose_sn[p], ld = g.sn_ld[s];
    const int cc = D * (p - g.sn_first[s]);
    double* T = L.at(g.sn_off[s] + cc * ld + cc);
    // damping / max on the diagonal, then each lower column (D - q contiguous doubles) with 128-bit
    // stores where 16-byte aligned
#pragma unroll
    for (int q = 0, e = 0; q < D; e += D - q, ++q) {
      double v = h[e];
      if (lam > 0.0) v = (damping == 0) ? v * (1.0 + lam) : v + lam;
      mymax = fmax(mymax, v);
      h[e] = v;
    }
#pragma unroll
    for (int q = 0, e = 0; q < D; e += D - q, ++q) {
      double* c = T + (size_t)q * ld + q;
      const int n = D - q;
      if ((reinterpret_cast<uintptr_t>(c) & 15) == 0) {
#pragma unroll
        for (int k = 0; k < n; k += 2) {
          if (k + 1 < n) *reinterpret_cast<double2*>(c + k) = make_double2(h[e + k], h[e + k + 1]);
          else c[k] = h[e + k];
        }
      } else {
        c[0] = h[e];
#pragma unroll
        for (int k = 1; k < n; k += 2) {
          if (k + 1 < n) *reinterpret_cast<double2*>(c + k) = make_double2(h[e + k], h[e + k + 1]);
          else c[k] = h[e + k];
        }
      }
    }
#pragma unroll
    for (int a = 0; a < D; ++a) x_b[(size_t)D * p + a] = r[a];
  }
  for (int k = gt; k < g.ndup; k += GN) {   // off-diagonal blocks shared by several edges
    const int bk = g.dup_blk[k];
    double h[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) h[i] = 0.0;
    for (int c = g.blk_cptr[bk]; c < g.blk_cptr[bk + 1]; ++c) {
      const double* o = scr + (size_t)(g.blk_con[c] >> 2) * SC::SIZE + SC::HIJ;
#pragma unroll
      for (int i = 0; i < D * D; ++i) h[i] += o[i];
    }
    double* T = L.at(g.blk_off[bk]);
    const int ld = g.blk_ld[bk];
#pragma unroll
    for (int q = 0; q < D; ++q)
#pragma unroll
      for (int a = 0; a < D; ++a) T[(size_t)q * ld + a] = h[q * D + a];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mymax = fmax(mymax, __shfl_xor_sync(0xffffffffu, mymax, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = mymax;
  DNLS_PROBE_NOW(p4);
  DNLS_PROBE_ADD(3, p3, p4);
}

// Warp-level dense triangular solves on a panel's w x w diagonal block (P column-major, leading
// dim m), rows owned by lanes (row r = lane + 32 j), values held in registers, each step one
// shuffle broadcast.  MAXR = max ceil(w / 32).
template <int MAXR>
__device__ __forceinline__ void warp_trsv_lower(const double* P, int ld, int w, double* xs) {
  const int lane = threadIdx.x & 31;
  double t[MAXR], inv[MAXR];
#pragma unroll
  for (int j = 0; j < MAXR; ++j) {
    const int r = lane + 32 * j;
    t[j] = (r < w) ? xs[r] : 0.0;
    inv[j] = (r < w) ? 1.0 / P[(size_t)r * ld + r] : 0.0;
  }
#pragma unroll
  for (int sj = 0; sj < MAXR; ++sj) {
    if (32 * sj >= w) break;
    const int cend = min(32, w - 32 * sj);
    for (int cl = 0; cl < cend; ++cl) {
      const int c = 32 * sj + cl;
      const double xc = __shfl_sync(0xffffffffu, t[sj] * inv[sj], cl);
      if (lane == cl) t[sj] = xc;
      const double* col = P + (size_t)c * ld;
#pragma unroll
      for (int j = sj; j < MAXR; ++j) {
        const int r = lane + 32 * j;
        if (r > c && r < w) t[j] = fma(-col[r], xc, t[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < MAXR; ++j) {
    const int r = lane + 32 * j;
    if (r < w) xs[r] = t[j];
  }
}

template <int MAXR>
__device__ __forceinline__ void warp_trsv_upper(const double* P, int ld, int w, double* xs) {
  // solve L^T x = t : step c from w-1 down to 0, rows r < c updated with L[c][r] = P[r*m + c]
  const int lane = threadIdx.x & 31;
  double t[MAXR], inv[MAXR];
#pragma unroll
  for (int j = 0; j < MAXR; ++j) {
    const int r = lane + 32 * j;
    t[j] = (r < w) ? xs[r] : 0.0;
    inv[j] = (r < w) ? 1.0 / P[(size_t)r * ld + r] : 0.0;
  }
#pragma unroll
  for (int sj = MAXR - 1; sj >= 0; --sj) {
    if (32 * sj >= w) continue;
    const int cend = min(32, w - 32 * sj);
    for (int cl = cend - 1; cl >= 0; --cl) {
      const int c = 32 * sj + cl;
      const double xc = __shfl_sync(0xffffffffu, t[sj] * inv[sj], cl);
      if (lane == cl) t[sj] = xc;
#pragma unroll
      for (int j = 0; j <= sj; ++j) {
        const int r = lane + 32 * j;
        if (r < c) t[j] = fma(-P[(size_t)r * ld + c], xc, t[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < MAXR; ++j) {
    const int r = lane + 32 * j;
    if (r < w) xs[r] = t[j];
  }
}

// ---- gathers with G cooperating lanes (G | 32, groups lane-aligned): the lanes of a group split
// the k-range (concatenated source columns, round robin) and combine with an xor-shuffle tree.
// Every lane of the warp must call the reduction (uniform trip counts); order is fixed, so the
// result is bitwise deterministic.
template <int N>
__device__ __forceinline__ void group_reduce(double (&acc)[N], int G) {
  for (int off = G >> 1; off > 0; off >>= 1) {
#pragma unroll
    for (int q = 0; q < N; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
  }
}

// variable-size aligned lane groups in one warp: 5 uniform xor steps, accumulate when off < G
template <int N>
__device__ __forceinline__ void group_reduce_var(double (&acc)[N], int G) {
  const int gmax = __reduce_max_sync(0xffffffffu, (unsigned)G);
  for (int off = gmax >> 1; off > 0; off >>= 1) {
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const double v = __shfl_xor_sync(0xffffffffu, acc[q], off);
      if (off < G) acc[q] += v;
    }
  }
}

// width-dispatched warp triangular solves (slots = ceil(w / 32) register rows per lane)
template <int D>
__device__ __forceinline__ void warp_trsv_lower_w(const double* P, int ld, int w, double* xs) {
  if (w <= 32) warp_trsv_lower<1>(P, ld, w, xs);
  else if (w <= 64) warp_trsv_lower<2>(P, ld, w, xs);
  else if (w <= 128) warp_trsv_lower<4>(P, ld, w, xs);
  else warp_trsv_lower<(64 * D + 31) / 32>(P, ld, w, xs);
}
template <int D>
__device__ __forceinline__ void warp_trsv_upper_w(const double* P, int ld, int w, double* xs) {
  if (w <= 32) warp_trsv_upper<1>(P, ld, w, xs);
  else if (w <= 64) warp_trsv_upper<2>(P, ld, w, xs);
  else if (w <= 128) warp_trsv_upper<4>(P, ld, w, xs);
  else warp_trsv_upper<(64 * D + 31) / 32>(P, ld, w, xs);
}

// ----------------------------------------------------------------------------- packet-driven levels
// Every elimination-tree level has a descriptor packet (symbolic.cpp 5b'); packets are
// prefetched into a double buffer in shared memory by TMA bulk copies one level ahead, so all
// index reads of the numeric phases hit shared memory.
struct Pk {
  int ntasks, ncons, nrows, nfcons, nsn, nsnr, nul, nfl, maxb, level, first, last, nul3;
  const int4 *task4, *con4, *row4, *fcon4, *sna, *snb;
  const int *snr, *ulane, *flane, *ulane3, *snm, *snw;   // ulane: 1-row update items, ulane3: UPD_ROWS-row items
};
__device__ __forceinline__ Pk pk_view(const int* b) {
  Pk p;
  const int4 h0 = reinterpret_cast<const int4*>(b)[0], h1 = reinterpret_cast<const int4*>(b)[1];
  const int4 h2 = reinterpret_cast<const int4*>(b)[2], h3 = reinterpret_cast<const int4*>(b)[3];
  p.ntasks = h0.x; p.ncons = h0.y; p.nrows = h0.z; p.nfcons = h0.w;
  p.nsn = h1.x; p.nsnr = h1.y; p.nul = h1.z; p.nfl = h1.w;
  p.maxb = h2.x;
  p.nul3 = h3.x;
  p.level = h2.y;
  p.first = h2.z;
  p.last = h2.w;
  p.task4 = reinterpret_cast<const int4*>(b) + 4;
  p.con4 = p.task4 + p.ntasks;
  p.row4 = p.con4 + p.ncons;
  p.fcon4 = p.row4 + p.nrows;
  p.sna = p.fcon4 + p.nfcons;
  p.snb = p.sna + p.nsn;
  p.snr = reinterpret_cast<const int*>(p.snb + p.nsn);
  p.ulane = p.snr + p.nsnr;
  p.flane = p.ulane + p.nul;
  p.ulane3 = p.flane + p.nfl;
  p.snm = p.ulane3 + p.nul3;
  p.snw = p.snm + p.nsn + 1;
  return p;
}

// double-buffered packet prefetcher (state identical in every thread)
struct PkPipe {
  int* buf[2];
  uint64_t* mb[2];
  uint32_t ph[2];
};
// thread 0 issues the copy of packet `lv` into buffer lv & 1 (caller: after a CTA barrier that
// follows the last read of that buffer, with every thread having executed fence.proxy.async)
__device__ __forceinline__ void pk_issue(const DevGraph& g, PkPipe& pp, int lv) {
  if (threadIdx.x == 0 && lv >= 0 && lv < g.npk) {
    const int o0 = g.pk_off[lv], o1 = g.pk_off[lv + 1];
    const uint32_t bytes = (uint32_t)(o1 - o0) * 4u;
    uint64_t* mb = pp.mb[lv & 1];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(pp.buf[lv & 1])),
        "l"(g.pk + o0), "r"(bytes), "r"(smem_u32(mb))
        : "memory");
  }
}
__device__ __forceinline__ Pk pk_wait(PkPipe& pp, int lv) {
  mbar_wait(pp.mb[lv & 1], pp.ph[lv & 1]);
  pp.ph[lv & 1] ^= 1u;
  return pk_view(pp.buf[lv & 1]);
}
// all threads: order prior generic accesses before the async proxy, then barrier
// packets are read-only (never written by the generic proxy), so a plain barrier orders the
// last reads of a buffer before the next bulk copy into it
__device__ __forceinline__ void proxy_barrier() { __syncthreads(); }

// level staging with plain vector loads (the staged panels were written back by generic stores
// earlier in the same kernel; the generic proxy keeps that ordering without proxy fences)
template <int NT>
__device__ __forceinline__ void stage_in(double* __restrict__ dst, const double* __restrict__ src, int n) {
  const int n2 = n >> 1;
  double2* d2 = reinterpret_cast<double2*>(dst);
  const double2* s2 = reinterpret_cast<const double2*>(src);
  int i = threadIdx.x;
  for (; i + 3 * NT < n2; i += 4 * NT) {
    const double2 a = s2[i], b = s2[i + NT], c = s2[i + 2 * NT], d = s2[i + 3 * NT];
    d2[i] = a;
    d2[i + NT] = b;
    d2[i + 2 * NT] = c;
    d2[i + 3 * NT] = d;
  }
  for (; i < n2; i += NT) d2[i] = s2[i];
  if ((n & 1) && threadIdx.x == 0) dst[n - 1] = src[n - 1];
  __syncthreads();
}

// staging of a level's contiguous panel range: TMA bulk copy (one thread issues, the copy engine
// moves the range; the panels were written by generic stores, hence the proxy fence in bulk_load)
// or plain vector loads
template <int NT>
__device__ __forceinline__ void stage_level(double* dst, const double* src, int n, uint64_t* mbar, uint32_t& phase) {
#ifndef DNLS_NO_TMA_STAGE
  if ((n & 1) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    bulk_load<NT>(dst, src, n, mbar, phase);
    return;
  }
#endif
  stage_in<NT>(dst, src, n);
}

// ---- level-wide dense kernels (all panels of a level at once)
// inverse pivots 1/L_jj of the D x D diagonal block at (c0, c0) live in its unused strict upper
// triangle: (c0+j, c0+j+1) for j < D-1 and (c0, c0+D-1) for j = D-1
template <int D>
__device__ __forceinline__ int ivpos(int c0, int j, int ld) {
  return j < D - 1 ? (c0 + j + 1) * ld + (c0 + j) : (c0 + D - 1) * ld + c0;
}
// single-block panel solves (w == D), one thread: forward y = L^-1 t / backward x = L^-T t
template <int D>
__device__ __forceinline__ void trsv_lower_block(const double* P, int ld, double* xs) {
  double y[D];
#pragma unroll
  for (int q = 0; q < D; ++q) {
    double s = xs[q];
#pragma unroll
    for (int k = 0; k < q; ++k) s = fma(-P[(size_t)k * ld + q], y[k], s);
    y[q] = s * P[ivpos<D>(0, q, ld)];
  }
#pragma unroll
  for (int q = 0; q < D; ++q) xs[q] = y[q];
}
template <int D>
__device__ __forceinline__ void trsv_upper_block(const double* P, int ld, double* xs) {
  double y[D];
#pragma unroll
  for (int q = D - 1; q >= 0; --q) {
    double s = xs[q];
#pragma unroll
    for (int k = q + 1; k < D; ++k) s = fma(-P[(size_t)q * ld + k], y[k], s);
    y[q] = s * P[ivpos<D>(0, q, ld)];
  }
#pragma unroll
  for (int q = 0; q < D; ++q) xs[q] = y[q];
}
// index of the panel owning flattened item it (prefix array pre[0..n], pre[0] = 0)
__device__ __forceinline__ int find_panel(const int* pre, int n, int it) {
  int lo = 0, hi = n;   // pre[lo] <= it < pre[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] <= it) lo = mid;
    else hi = mid;
  }
  return lo;
}

// ---- team-wise level factorisation (replaces the CTA-phase version above on the hot path)
// Redundant in-register Cholesky of the D x D diagonal block at (c0, c0): every lane of a team
// loads the lower triangle (a shared-memory broadcast) and factors it, so no barrier separates
// the diagonal factorisation from the TRSM rows that need it.  Same arithmetic and order as
// the former chol_block (bitwise identical factor).  Returns true if a pivot <= tol.
template <int D>
__device__ __forceinline__ bool chol_regs(const double* P, int ld, int c0, double tol, double (&a)[D][D],
                                          double (&iv)[D]) {
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int i = j; i < D; ++i) a[i][j] = P[(size_t)(c0 + j) * ld + c0 + i];
  bool bad = false;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double piv = a[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) piv = fma(-a[j][k], a[j][k], piv);
    if (!(piv > tol)) {
      bad = true;
      piv = 1.0;
    }
    const double inv = rsqrt(piv);
    iv[j] = inv;
    a[j][j] = piv * inv;
#pragma unroll
    for (int i = j + 1; i < D; ++i) {
      double s = a[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) s = fma(-a[i][k], a[j][k], s);
      a[i][j] = s * inv;
    }
  }
  return bad;
}
template <int D>
__device__ __forceinline__ void store_diag(double* P, int ld, int c0, const double (&a)[D][D], const double (&iv)[D]) {
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int i = j; i < D; ++i) P[(size_t)(c0 + j) * ld + c0 + i] = a[i][j];
#pragma unroll
  for (int j = 0; j < D; ++j) P[ivpos<D>(c0, j, ld)] = iv[j];
}
// row r below the diagonal block, L_jj from registers (same arithmetic as the former trsm_row)
template <int D>
__device__ __forceinline__ void trsm_row_regs(double* P, int ld, int c0, int r, const double (&a)[D][D],
                                              const double (&iv)[D]) {
  double x[D];
#pragma unroll
  for (int q = 0; q < D; ++q) x[q] = P[(size_t)(c0 + q) * ld + r];
#pragma unroll
  for (int q = 0; q < D; ++q) {
    double s = x[q];
#pragma unroll
    for (int k = 0; k < q; ++k) s = fma(-x[k], a[q][k], s);
    x[q] = s * iv[q];
  }
#pragma unroll
  for (int q = 0; q < D; ++q) P[(size_t)(c0 + q) * ld + r] = x[q];
}

struct TeamSync {
  int size, bar;
  unsigned mask;
  __device__ __forceinline__ void sync() const {
    if (size <= 32) __syncwarp(mask);
    else asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(size) : "memory");
  }
};

// Dense factorisation of every panel of a level by teams: sub-warp lane groups when the level
// has more panels than warps, groups of warps (named barriers) otherwise.  Per D-column block:
// redundant register Cholesky, TRSM rows split over the team, one team barrier, trailing update,
// one team barrier.  Single-block panels (the common case) need no barrier at all.  x != nullptr
// fuses the forward substitution of the panel's diagonal block (y_s = L_ss^-1 t_s).
// The caller places a CTA barrier after this function.
template <int D, int NT, int CL = 1>
__device__ void level_factor_teams(const Pk& P, const LView& V, double tol, int* fail, double* x) {
  constexpr int NW = NT / 32;
  const int nsn = P.nsn;
  if (nsn <= 0) return;
  if constexpr (CL > 1) {
    // wide panels of a sparse level (the separator supernodes of large problems; C3r's reach ~1554 columns):
    // a team of at most one CTA would leave the group's other CTAs waiting at the level barrier, so every
    // thread of the group works on one panel at a time -- per D-column block the redundant diagonal
    // Cholesky, the TRSM rows and the trailing update split over CL * NT threads, two group barriers.  The
    // same arithmetic per entry as the team path (identical factor).
    bool coop = nsn <= 2;
    if (coop) {
      bool wide = false;
      for (int i = 0; i < nsn; ++i) wide |= P.sna[i].w >= 8 * D;
      coop = wide;
    }
    if (coop) {
      const int gt = crank<CL>() * NT + threadIdx.x, GT = CL * NT;
      for (int i = 0; i < nsn; ++i) {
        const int4 sa = P.sna[i];
        double* Pn = V.at(sa.x);
        const int m = sa.y, ld = sa.z, w = sa.w;
        double* xs = x ? x + (size_t)D * P.snb[i].x : nullptr;
        for (int c0 = 0; c0 < w; c0 += D) {
          double a[D][D], iv[D];
          const bool bad = chol_regs<D>(Pn, ld, c0, tol, a, iv);
          for (int r = c0 + D + gt; r < m; r += GT) trsm_row_regs<D>(Pn, ld, c0, r, a, iv);
          gsync<CL>();   // every thread has read the unfactored diagonal block, the TRSM rows are written
          if (gt == 0) {
            store_diag<D>(Pn, ld, c0, a, iv);
            if (bad) *fail = 1;
          }
          const int r0 = c0 + D;
          if (r0 < w) {
            const int nc = w - r0, nr = m - r0, nit = nc * nr;
            for (int t = gt; t < nit; t += GT) {
              const int ci = t / nr, ri = t - ci * nr;
              if (ri < ci) continue;
              const int c = r0 + ci, r = r0 + ri;
              double s0 = 0.0, s1 = 0.0;
#pragma unroll
              for (int k = 0; k < D; k += 2) {
                s0 = fma(Pn[(size_t)(c0 + k) * ld + r], Pn[(size_t)(c0 + k) * ld + c], s0);
                if (k + 1 < D) s1 = fma(Pn[(size_t)(c0 + k + 1) * ld + r], Pn[(size_t)(c0 + k + 1) * ld + c], s1);
              }
              Pn[(size_t)c * ld + r] -= s0 + s1;
            }
          }
          gsync<CL>();
        }
        if (xs) {
          if (gt < 32) warp_trsv_lower_w<D>(Pn, ld, w, xs);
          gsync<CL>();
        }
      }
      return;
    }
  }
  const int nsc = (nsn + CL - 1) / CL;   // panels per CTA of the group
  int G;
  if (nsc >= NT) {
    G = 1;
  } else if (nsc > NW) {
    G = NT / nsc;
    while (G & (G - 1)) G &= G - 1;
    if (G > 32) G = 32;
  } else {
    int tw = NW / nsc;
    while (tw & (tw - 1)) tw &= tw - 1;
    G = 32 * tw;
  }
  const int nteams = NT / G;
  const int cr = crank<CL>();

  const int team = threadIdx.x / G, rank = threadIdx.x - team * G;
  TeamSync ts;
  ts.size = G;
  ts.bar = 1 + team;
  ts.mask = G >= 32 ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  // threads of a partial last team (NT need not be a multiple of G: 384 = 256 + 128) take no panel
  for (int i = (team < nteams ? team + cr * nteams : nsn); i < nsn; i += nteams * CL) {
    const int4 sa = P.sna[i];
    double* Pn = V.at(sa.x);
    const int m = sa.y, ld = sa.z, w = sa.w;
    double* xs = x ? x + (size_t)D * P.snb[i].x : nullptr;
    if (w == D) {
      // at most one warp factors redundantly and solves the TRSM rows (the fp64 pipe is shared); its
      // first lane stores L_jj and applies the forward substitution once every lane of the group has
      // read the unfactored diagonal block (warp sync: the store overwrites what the others read --
      // compute-sanitizer racecheck, profiles/r2_sanitizer.txt)
      const int Gr = G < 32 ? G : 32;
      if (rank >= Gr) continue;
      double a[D][D], iv[D];
      const bool bad = chol_regs<D>(Pn, ld, 0, tol, a, iv);
      for (int r = D + rank; r < m; r += Gr) trsm_row_regs<D>(Pn, ld, 0, r, a, iv);
      __syncwarp(ts.mask);
      if (rank == 0) {
        store_diag<D>(Pn, ld, 0, a, iv);
        if (bad) *fail = 1;
        if (xs) {
          double y[D];
#pragma unroll
          for (int q = 0; q < D; ++q) {
            double s = xs[q];
#pragma unroll
            for (int k = 0; k < q; ++k) s = fma(-a[q][k], y[k], s);
            y[q] = s * iv[q];
          }
#pragma unroll
          for (int q = 0; q < D; ++q) xs[q] = y[q];
        }
      }
      continue;
    }
    for (int c0 = 0; c0 < w; c0 += D) {
      double a[D][D], iv[D];
      const bool bad = chol_regs<D>(Pn, ld, c0, tol, a, iv);
      for (int r = c0 + D + rank; r < m; r += G) trsm_row_regs<D>(Pn, ld, c0, r, a, iv);
      ts.sync();   // every rank has read the unfactored diagonal block and written its TRSM rows
      if (rank == 0) {   // the trailing update below reads rows >= c0 + D only
        store_diag<D>(Pn, ld, c0, a, iv);
        if (bad) *fail = 1;
      }
      const int r0 = c0 + D;
      if (r0 < w) {
        const int nc = w - r0, nr = m - r0, nit = nc * nr;
        for (int t = rank; t < nit; t += G) {
          const int ci = t / nr, ri = t - ci * nr;
          if (ri < ci) continue;
          const int c = r0 + ci, r = r0 + ri;
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int k = 0; k < D; k += 2) {
            s0 = fma(Pn[(size_t)(c0 + k) * ld + r], Pn[(size_t)(c0 + k) * ld + c], s0);
            if (k + 1 < D) s1 = fma(Pn[(size_t)(c0 + k + 1) * ld + r], Pn[(size_t)(c0 + k + 1) * ld + c], s1);
          }
          Pn[(size_t)c * ld + r] -= s0 + s1;
        }
        ts.sync();
      }
    }
    if (xs) {
      ts.sync();   // the last diagonal block is stored
      if (G >= 32) {
        if (rank < 32) warp_trsv_lower_w<D>(Pn, ld, w, xs);
      } else if (rank == 0) {   // y = L_ss^-1 t, column-oriented, inverse pivots from ivpos
        for (int c = 0; c < w; ++c) {
          const int cb = c - c % D, j = c - cb;
          const double yc = xs[c] * Pn[ivpos<D>(cb, j, ld)];
          xs[c] = yc;
          const double* col = Pn + (size_t)c * ld;
          for (int r = c + 1; r < w; ++r) xs[r] = fma(-col[r], yc, xs[r]);
        }
      }
      ts.sync();
    }
  }
}

// y_s = L_ss^-1 t_s for every panel of a level (thread per single-block panel, warp otherwise)
template <int D, int NT>
__device__ void level_trsv_lower(const Pk& P, const LView& V, double* x) {
  for (int i = threadIdx.x; i < P.nsn; i += NT) {
    const int4 sa = P.sna[i];
    if (sa.w == D) trsv_lower_block<D>(V.at(sa.x), sa.z, x + (size_t)D * P.snb[i].x);
  }
  for (int i = threadIdx.x >> 5; i < P.nsn; i += NT / 32) {
    const int4 sa = P.sna[i];
    if (sa.w > D) warp_trsv_lower_w<D>(V.at(sa.x), sa.z, sa.w, x + (size_t)D * P.snb[i].x);
  }
}
template <int D, int NT, int CL = 1>
__device__ void level_trsv_upper(const Pk& P, const LView& V, double* x) {
  for (int i = crank<CL>() * NT + threadIdx.x; i < P.nsn; i += CL * NT) {
    const int4 sa = P.sna[i];
    if (sa.w == D) trsv_upper_block<D>(V.at(sa.x), sa.z, x + (size_t)D * P.snb[i].x);
  }
  for (int i = crank<CL>() * (NT / 32) + (threadIdx.x >> 5); i < P.nsn; i += CL * (NT / 32)) {
    const int4 sa = P.sna[i];
    if (sa.w > D) warp_trsv_upper_w<D>(V.at(sa.x), sa.z, sa.w, x + (size_t)D * P.snb[i].x);
  }
}
// backward gather of a level: item (panel, column c): x_c -= sum over below rows L[r][c] x_r
template <int D, int NT, int CL = 1>
__device__ void level_bwd_gather(const Pk& P, const LView& V, double* x) {
  const int total = P.snw[P.nsn];
  for (int it = crank<CL>() * NT + threadIdx.x; it < total; it += CL * NT) {
    const int i = find_panel(P.snw, P.nsn, it);
    const int4 sa = P.sna[i], sb = P.snb[i];
    const int c = it - P.snw[i];
    const double* col = V.at(sa.x) + (size_t)c * sa.z + sa.w;
    double s0 = 0.0, s1 = 0.0;
    for (int rr = sb.y; rr < sb.z; ++rr) {
      const double* xr = x + (size_t)D * P.snr[rr];
      const double* cr = col + (rr - sb.y) * D;
#pragma unroll
      for (int a = 0; a < D; a += 2) {
        s0 = fma(cr[a], xr[a], s0);
        if (a + 1 < D) s1 = fma(cr[a + 1], xr[a + 1], s1);
      }
    }
    x[(size_t)D * sb.x + c] -= s0 + s1;
  }
}

// partial rows a0 .. a0 + R - 1 of update task tk over the contributions ci = lane (mod G) of the task: the G
// lanes of a group take whole source panels, so their (independent) loads overlap; R rows per item share the
// loads of the target's column block (R + D loads per R * D FMAs).  Per accumulator the FMAs run over the
// source columns in order (the same sequence for any R).
template <int D, int R>
__device__ __forceinline__ void pk_task_rows_partial(const Pk& P, const LView& V, const int4 tk, int a0, int lane,
                                                     int G, double (&acc)[R * D]) {
  for (int ci = tk.z + lane; ci < tk.w; ci += G) {
    const int4 c = P.con4[ci];
    const double* A = V.at(c.x) + a0;
    const double* Bm = V.at(c.y);
    const size_t ld = c.z;
    int k = 0;
#ifndef DNLS_UK
#define DNLS_UK 3
#endif
    constexpr int UK = DNLS_UK;
    for (; k + UK <= c.w; k += UK) {   // UK source columns of loads in flight
      double av[UK][R], bv[UK][D];
#pragma unroll
      for (int u = 0; u < UK; ++u) {
#pragma unroll
        for (int r = 0; r < R; ++r) av[u][r] = A[(k + u) * ld + r];
#pragma unroll
        for (int q = 0; q < D; ++q) bv[u][q] = Bm[(k + u) * ld + q];
      }
#pragma unroll
      for (int u = 0; u < UK; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int q = 0; q < D; ++q) acc[r * D + q] = fma(av[u][r], bv[u][q], acc[r * D + q]);
    }
    for (; k < c.w; ++k) {
      double av[R], bv[D];
#pragma unroll
      for (int r = 0; r < R; ++r) av[r] = A[k * ld + r];
#pragma unroll
      for (int q = 0; q < D; ++q) bv[q] = Bm[k * ld + q];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int q = 0; q < D; ++q) acc[r * D + q] = fma(av[r], bv[q], acc[r * D + q]);
    }
  }
}

template <int D>
__device__ __forceinline__ double pk_fwd_row_partial(const Pk& P, const LView& V, const double* x, int4 rw, int a,
                                                     int lane, int G) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int ci = rw.y + lane; ci < rw.z; ci += G) {
    const int4 c = P.fcon4[ci];
    const double* A = V.at(c.x) + a;
    const double* y = x + c.w;
    const size_t ld = c.y;
    int k = 0;
    for (; k + 6 <= c.z; k += 6) {   // same accumulator assignment as two 3-column steps, loads hoisted
      double av[6], yv[6];
#pragma unroll
      for (int u = 0; u < 6; ++u) {
        av[u] = A[(k + u) * ld];
        yv[u] = y[k + u];
      }
      s0 = fma(av[0], yv[0], s0);
      s1 = fma(av[1], yv[1], s1);
      s2 = fma(av[2], yv[2], s2);
      s0 = fma(av[3], yv[3], s0);
      s1 = fma(av[4], yv[4], s1);
      s2 = fma(av[5], yv[5], s2);
    }
    for (; k + 3 <= c.z; k += 3) {
      s0 = fma(A[k * ld], y[k], s0);
      s1 = fma(A[(k + 1) * ld], y[k + 1], s1);
      s2 = fma(A[(k + 2) * ld], y[k + 2], s2);
    }
    for (; k < c.z; ++k) s0 = fma(A[k * ld], y[k], s0);
  }
  return (s0 + s1) + s2;
}

// forward-substitution gather of a level's pose rows (CTA-wide): x_pa -= sum L_d[p_a,:] y_d.
// Lane map (packet): each (row, component) item owns an aligned group of G lanes.
template <int D, int NT, int CL = 1>
__device__ void pk_fwd_rows(const Pk& P, const LView& V, double* x) {
  for (int base = crank<CL>() * NT; base < P.nfl; base += CL * NT) {
    const int L = base + threadIdx.x;
    const int e = L < P.nfl ? P.flane[L] : -1;
    const int G = e >= 0 ? 1 << ((e >> 5) & 7) : 1, sub = e >= 0 ? (e & 31) : 0;
    const int item = e >= 0 ? e >> 8 : 0;
    const int r = item / D, a = item - r * D;
    const int4 rw = P.row4[r];
    double acc[1] = {e >= 0 ? pk_fwd_row_partial<D>(P, V, x, rw, a, sub, G) : 0.0};
    group_reduce_var<1>(acc, G);
    if (e >= 0 && sub == 0) x[(size_t)D * rw.x + a] -= acc[0];
  }
}

// Full numeric factorisation, level-synchronous with packet prefetch.  xf != nullptr fuses the
// forward substitution (y = L^-1 x in place).
template <int D, int NT, int CL = 1>
__device__ void factor_phase(const DevGraph& g, const LView& L, double* stage, double tol, int* s_fail,
                             uint64_t* mbar, uint32_t& phase, double* xinv, double* xf, PkPipe& pp) {
  proxy_barrier();
  pk_issue(g, pp, 0);
  pk_issue(g, pp, 1);
  for (int k = 0; k < g.npk; ++k) {
    const Pk P = pk_wait(pp, k);
    const int lv = P.level;
    const int lo = g.level_off[lv];
    const bool resident = lo >= L.rlo;
    const int hi = (resident || CL > 1) ? lo : g.level_stage_hi[lv];   // groups work in global memory
    DNLS_TRACE_POINT(1000 + lv);
#ifndef DNLS_SKIP_STAGE
    if (P.first && !resident) stage_level<NT>(stage, L.g + lo, hi - lo, mbar, phase);
    DNLS_TRACE_POINT(1100 + lv);
#endif
    const LView V = L.level(stage, lo, hi);
    {   // (U) gather-form updates: item = (task, row a) owns an aligned group of G lanes (lane map)
      constexpr int R = CL == 1 ? UPD_ROWS : 1, IPT = D / R;   // rows per item, items per task
      const int nul = CL == 1 ? P.nul3 : P.nul;
      const int* ulane = CL == 1 ? P.ulane3 : P.ulane;
      for (int base = crank<CL>() * NT; base < nul; base += CL * NT) {
        const int Ln = base + threadIdx.x;
        const int e = Ln < nul ? ulane[Ln] : -1;
        const bool valid = e >= 0;
        const int G = valid ? 1 << ((e >> 5) & 7) : 1, lane = valid ? (e & 31) : 0;
        const int item = valid ? e >> 8 : 0;
        const int t = item / IPT, a0 = (item - t * IPT) * R;
        const int4 tk = P.ntasks > 0 ? P.task4[t] : make_int4(0, 0, 0, 0);
        double acc[R * D];
#pragma unroll
        for (int q = 0; q < R * D; ++q) acc[q] = 0.0;
#ifndef DNLS_SKIP_U
        if (valid) pk_task_rows_partial<D, R>(P, V, tk, a0, lane, G, acc);
#endif
        group_reduce_var<R * D>(acc, G);
        if (valid && lane == 0) {
          double* T = V.at(tk.x) + a0;
#pragma unroll
          for (int r = 0; r < R; ++r)
#pragma unroll
            for (int q = 0; q < D; ++q) T[(size_t)q * tk.y + r] -= acc[r * D + q];
        }
      }
    }
    DNLS_TRACE_POINT(1160 + lv);
    // forward-substitution rows read descendant panels and y of earlier levels only: no barrier
    // between them and the updates of this level's panels
#ifndef DNLS_SKIP_FWD
    if (xf) pk_fwd_rows<D, NT, CL>(P, V, xf);
#endif
    gsync<CL>();
    DNLS_TRACE_POINT(1200 + lv);
    // (F) dense factorisation of this packet's panels, level-wide
#ifndef DNLS_SKIP_F
    level_factor_teams<D, NT, CL>(P, V, tol, s_fail, xf);   // + fused y_s = L_ss^-1 t_s
#endif
    gsync<CL>();
    DNLS_TRACE_POINT(1300 + lv);
#ifndef DNLS_SKIP_STAGE
    if (P.last && !resident && hi > lo) copy_range<NT>(L.g + lo, stage, hi - lo);
#endif
    proxy_barrier();
    pk_issue(g, pp, k + 2);
  }
  DNLS_TRACE_POINT(1999);
}

// Solve with the factor: forward (unless fused into the factorisation) and backward
// substitution, level-synchronous with packet prefetch; warp per supernode for the dense parts.
template <int D, int NT, int CL = 1>
__device__ void solve_phase(const DevGraph& g, const LView& L, double* stage, double* x, uint64_t* mbar,
                            uint32_t& phase, PkPipe& pp, bool forward = true) {
  if (forward) {
    proxy_barrier();
    pk_issue(g, pp, 0);
    pk_issue(g, pp, 1);
    for (int k = 0; k < g.npk; ++k) {
      const Pk P = pk_wait(pp, k);
      const int lv = P.level;
      const int lo = g.level_off[lv];
      const bool resident = lo >= L.rlo;
      const int hi = resident ? lo : g.level_stage_hi[lv];
      if (P.first && !resident) stage_in<NT>(stage, L.g + lo, hi - lo);
      const LView V = L.level(stage, lo, hi);
      pk_fwd_rows<D, NT>(P, V, x);
      __syncthreads();
      level_trsv_lower<D, NT>(P, V, x);
      proxy_barrier();
      pk_issue(g, pp, k + 2);
    }
  }
  // backward: root to leaves (packets in reverse; a level's chunks are independent here)
  proxy_barrier();
  pk_issue(g, pp, g.npk - 1);
  pk_issue(g, pp, g.npk - 2);
  for (int k = g.npk - 1; k >= 0; --k) {
    const Pk P = pk_wait(pp, k);
    const int lv = P.level;
    const int lo = g.level_off[lv];
    const bool resident = lo >= L.rlo;
    const int hi = (resident || CL > 1) ? lo : g.level_stage_hi[lv];
    DNLS_TRACE_POINT(3000 + lv);
#ifndef DNLS_SKIP_STAGE
    if (P.last && !resident) stage_level<NT>(stage, L.g + lo, hi - lo, mbar, phase);
#endif
    DNLS_TRACE_POINT(3100 + lv);
    const LView V = L.level(stage, lo, hi);
#ifndef DNLS_SKIP_BS
    level_bwd_gather<D, NT, CL>(P, V, x);
#endif
    gsync<CL>();
#ifndef DNLS_SKIP_BS
    level_trsv_upper<D, NT, CL>(P, V, x);
#endif
    gsync<CL>();   // also orders the packet buffer reuse (proxy barrier)
    pk_issue(g, pp, k - 2);
  }
}

// ============================================================================= a5: retraction
// Tout[o] = Tin[o] Exp(-alpha delta_o), delta in permuted order
template <int D, int NT, int CL = 1>
__device__ void retract_phase(const DevGraph& g, const double* Tin, double* Tout, const double* x, double alpha) {
  constexpr int PS = GT<D>::PS;
  using namespace dev;
  for (int o = crank<CL>() * NT + threadIdx.x; o < g.N; o += CL * NT) {
    const double* dl = x + (size_t)D * g.iperm[o];
    double xi[D];
#pragma unroll
    for (int a = 0; a < D; ++a) xi[a] = -alpha * dl[a];
    if (D == 6) {
      SE3 T = se3_load(Tin + (size_t)o * PS);
      se3_store(se3_mul(T, se3_exp(xi)), Tout + (size_t)o * PS);
    } else {
      SE2 T = se2_load(Tin + (size_t)o * PS);
      se2_store(se2_mul(T, se2_exp(xi)), Tout + (size_t)o * PS);
    }
  }
}

}  // namespace dnls
