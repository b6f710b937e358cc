// Per-element device phases of one GN/LM iteration.  One CUDA block ("CTA") owns one batch
// element; every phase below is executed cooperatively by the CTA's NT threads
// (DESIGN.md "Kernels").  Phases:
//   jac_phase       a1: per-cost residual + weighted Jacobians -> per-element scratch
//   assemble_phase  a2: scatter-free H (+lambda damping) into the factor storage, b, S
//   factor_phase    a3: supernodal left-looking Cholesky, level-synchronous
//   solve_phase     a4: forward / backward substitution
//   retract_phase   a5: T <- T Exp(-alpha delta)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lie.cuh"

namespace dnls {

// device view of the symbolic analysis (all arrays int32, uploaded once per graph)
struct DevGraph {
  int D, N, E, P, S, L, storage, nblk, n;
  int x_smem;     // 1: the solution vector x lives in shared memory (offset 0, n_pad doubles)
  int n_pad;      // n rounded up to an even count (16-byte alignment of the staging area)
  int stage_n;    // doubles of the level-staging area (largest staged level prefix)
  const int *perm, *iperm, *edges, *prior_vars;
  const int *sn_first, *sn_ncols, *sn_m, *sn_w, *sn_off;
  const int *level_ptr, *level_sn, *level_off, *level_stage_hi;
  const int *ut_level_ptr, *ut_off, *ut_ld, *ut_cptr, *uc_a, *uc_b, *uc_ld, *uc_w;
  const int *fc_ptr, *fc_off, *fc_ld, *fc_w, *fc_x;
  const int *snr_ptr, *snr;
  const int *blk_off, *blk_ld, *blk_kind, *blk_cptr, *blk_con;
  const int *bc_ptr, *bc;
};

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
};

// per-call workspace views (device)
struct DevWs {
  double* L;      // [B][storage]
  double* x;      // [B][n]   rhs / solution (permuted order)
  double* jac;    // [B][E+P][JS]  weighted J_i, J_j, r per cost slot
  double* cost;   // [B][E+P]      1/2 |r|^2 per slot (or weight gradient in backward)
  double* trial;  // [B][N][PS]    LM trial poses
  double* S;      // [B] current objective
  double* Sprev;  // [B]
  double* lam;    // [B]
  double* maxd;   // [B] max diagonal of the matrix last assembled/imported
  int* st;        // [B] status
  int* it;        // [B] iterations
};

template <int D>
struct GT {
  static constexpr int PS = (D == 6) ? 12 : 6;   // doubles per pose
  static constexpr int JS = 2 * D * D + D;        // scratch doubles per cost slot
};

// Factor storage view: offsets >= lo live in shared memory (a suffix of the storage, the
// top of the elimination tree), the rest in global memory.  Generic pointers serve both.
struct LView {
  double* g;
  double* s;
  int lo, hi;
  __device__ __forceinline__ double* at(int off) const {
    return (off >= lo && off < hi) ? s + (off - lo) : g + off;
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

// ============================================================================= cost evaluation
// Unweighted cost c and Jacobians of slot `slot` (edge e < E, else prior slot - E) at poses Tb.
// Ci/Cj are row-major D x D.  For priors only Ci is written.
template <int D>
__device__ __forceinline__ void eval_slot(const DevGraph& g, const DevProb& pr, const double* Tb, int b,
                                          int slot, double* c, double* Ci, double* Cj, bool need_jac) {
  constexpr int PS = GT<D>::PS;
  using namespace dev;
  if (D == 6) {
    SE3 Eerr;
    if (slot < g.E) {
      const int i = g.edges[2 * slot], j = g.edges[2 * slot + 1];
      SE3 Ti = se3_load(Tb + (size_t)i * PS), Tj = se3_load(Tb + (size_t)j * PS);
      SE3 Z = se3_load(pr.meas + ((size_t)b * g.E + slot) * PS);
      SE3 X = se3_between(Ti, Tj);
      Eerr = se3_between(Z, X);
      se3_log(Eerr, c);
      if (!need_jac) return;
      M3 Ji, U;
      se3_jr_inv(c, Ji, U);
      // Cj = Jr^-1(c) = [[Ji, U], [0, Ji]]
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
    } else {
      const int k = slot - g.E;
      SE3 T = se3_load(Tb + (size_t)g.prior_vars[k] * PS);
      SE3 Z = se3_load(pr.prior_meas + (size_t)b * pr.pm_bstride + (size_t)k * PS);
      Eerr = se3_between(Z, T);
      se3_log(Eerr, c);
      if (!need_jac) return;
      M3 Ji, U;
      se3_jr_inv(c, Ji, U);
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          Ci[r * 6 + q] = Ji.m[r][q];
          Ci[r * 6 + q + 3] = U.m[r][q];
          Ci[(r + 3) * 6 + q] = 0.0;
          Ci[(r + 3) * 6 + q + 3] = Ji.m[r][q];
        }
    }
  } else {
    if (slot < g.E) {
      const int i = g.edges[2 * slot], j = g.edges[2 * slot + 1];
      SE2 Ti = se2_load(Tb + (size_t)i * PS), Tj = se2_load(Tb + (size_t)j * PS);
      SE2 Z = se2_load(pr.meas + ((size_t)b * g.E + slot) * PS);
      SE2 Eerr = se2_between(Z, se2_between(Ti, Tj));
      se2_log(Eerr, c);
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
    } else {
      const int k = slot - g.E;
      SE2 T = se2_load(Tb + (size_t)g.prior_vars[k] * PS);
      SE2 Z = se2_load(pr.prior_meas + (size_t)b * pr.pm_bstride + (size_t)k * PS);
      se2_log(se2_between(Z, T), c);
      if (!need_jac) return;
      double J[3][3];
      se2_jr_inv(c, J);
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int q = 0; q < 3; ++q) Ci[r * 3 + q] = J[r][q];
    }
  }
}

template <int D>
__device__ __forceinline__ double slot_weight(const DevGraph& g, const DevProb& pr, int b, int slot) {
  return slot < g.E ? pr.w_edge[(size_t)b * pr.we_bstride + slot]
                    : pr.w_prior[(size_t)b * pr.wp_bstride + (slot - g.E)];
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

// ============================================================================= a1: Jacobians
template <int D, int NT>
__device__ void jac_phase(const DevGraph& g, const DevProb& pr, const double* Tb, int b, double* jac_b,
                          double* cost_b) {
  constexpr int JS = GT<D>::JS;
  const int nslot = g.E + g.P;
  for (int slot = threadIdx.x; slot < nslot; slot += NT) {
    double c[D], Ci[D * D], Cj[D * D];
    eval_slot<D>(g, pr, Tb, b, slot, c, Ci, Cj, true);
    const double w = slot_weight<D>(g, pr, b, slot);
    double* o = jac_b + (size_t)slot * JS;
    double n2 = 0.0;
#pragma unroll
    for (int q = 0; q < D * D; ++q) o[q] = w * Ci[q];
    if (slot < g.E) {
#pragma unroll
      for (int q = 0; q < D * D; ++q) o[D * D + q] = w * Cj[q];
    }
#pragma unroll
    for (int q = 0; q < D; ++q) {
      double r = w * c[q];
      o[2 * D * D + q] = r;
      n2 += r * r;
    }
    cost_b[slot] = 0.5 * n2;
  }
}

// objective only (LM trial / final objective without implicit)
template <int D, int NT>
__device__ void objective_phase(const DevGraph& g, const DevProb& pr, const double* Tb, int b, double* cost_b) {
  const int nslot = g.E + g.P;
  for (int slot = threadIdx.x; slot < nslot; slot += NT) {
    double c[D];
    eval_slot<D>(g, pr, Tb, b, slot, c, nullptr, nullptr, false);
    const double w = slot_weight<D>(g, pr, b, slot);
    double n2 = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) n2 += (w * c[q]) * (w * c[q]);
    cost_b[slot] = 0.5 * n2;
  }
}

// ============================================================================= a2: assembly
// Every d x d block of the factor storage is written exactly once (scatter-free, single writer,
// fixed summation order over its contribution list).  Item = (block, row a) -> D outputs.
// lam < 0: undamped.  damping 0: Marquardt (diag *= 1 + lam), 1: identity (diag += lam).
template <int D, int NT>
__device__ void assemble_phase(const DevGraph& g, LView L, const double* jac_b, double* x_b, double lam,
                               int damping, double* s_red) {
  constexpr int JS = GT<D>::JS;
  double mymax = 0.0;
  const int nitems = g.nblk * D;
  for (int itm = threadIdx.x; itm < nitems; itm += NT) {
    const int blk = itm / D, a = itm - blk * D;
    double acc[D];
#pragma unroll
    for (int q = 0; q < D; ++q) acc[q] = 0.0;
    const int c0 = g.blk_cptr[blk], c1 = g.blk_cptr[blk + 1];
    for (int ci = c0; ci < c1; ++ci) {
      const int code = g.blk_con[ci];
      const int slot = code >> 2, rs = (code >> 1) & 1, cs = code & 1;
      const double* Jr = jac_b + (size_t)slot * JS + rs * D * D;
      const double* Jc = jac_b + (size_t)slot * JS + cs * D * D;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double jra = Jr[k * D + a];
#pragma unroll
        for (int q = 0; q < D; ++q) acc[q] = fma(jra, Jc[k * D + q], acc[q]);
      }
    }
    if (g.blk_kind[blk] == 1) {
      double v = acc[a];
      if (lam > 0.0) v = (damping == 0) ? v * (1.0 + lam) : v + lam;
      acc[a] = v;
      mymax = fmax(mymax, v);
    }
    double* T = L.at(g.blk_off[blk]);
    const int ld = g.blk_ld[blk];
#pragma unroll
    for (int q = 0; q < D; ++q) T[(size_t)q * ld + a] = acc[q];
  }
  // b = J^T r (permuted order)
  const int nb = g.N * D;
  for (int itm = threadIdx.x; itm < nb; itm += NT) {
    const int p = itm / D, a = itm - p * D;
    double acc = 0.0;
    for (int ci = g.bc_ptr[p]; ci < g.bc_ptr[p + 1]; ++ci) {
      const int code = g.bc[ci];
      const int slot = code >> 1, sd = code & 1;
      const double* J = jac_b + (size_t)slot * JS + sd * D * D;
      const double* r = jac_b + (size_t)slot * JS + 2 * D * D;
#pragma unroll
      for (int k = 0; k < D; ++k) acc = fma(J[k * D + a], r[k], acc);
    }
    x_b[itm] = acc;
  }
  // max diagonal (CTA reduce, max is order independent)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mymax = fmax(mymax, __shfl_xor_sync(0xffffffffu, mymax, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = mymax;
}

// ============================================================================= a3: factorisation
// A team is a warp, a group of warps synchronised by a named barrier, or the whole CTA.
struct Team {
  int rank, size, bar;
  __device__ __forceinline__ void sync() const {
    if (size == 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(size) : "memory");
  }
};

// Dense right-looking Cholesky of one supernode panel P (m rows, w columns, column-major,
// leading dim m), blocked by D columns.  Writes L in place (lower part of the diagonal block
// and the rows below).  *fail set if a pivot <= tol.
template <int D>
__device__ void panel_factor(double* P, int m, int w, double tol, const Team& tm, int* fail) {
  for (int c0 = 0; c0 < w; c0 += D) {
    if (tm.rank == 0) {
      double a[D][D];
#pragma unroll
      for (int j = 0; j < D; ++j)
#pragma unroll
        for (int i = j; i < D; ++i) a[i][j] = P[(size_t)(c0 + j) * m + c0 + i];
      bool bad = false;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double piv = a[j][j];
#pragma unroll
        for (int k = 0; k < j; ++k) piv -= a[j][k] * a[j][k];
        if (!(piv > tol)) {
          bad = true;
          piv = 1.0;
        }
        const double ljj = sqrt(piv);
        const double inv = 1.0 / ljj;
        a[j][j] = ljj;
#pragma unroll
        for (int i = j + 1; i < D; ++i) {
          double s = a[i][j];
#pragma unroll
          for (int k = 0; k < j; ++k) s -= a[i][k] * a[j][k];
          a[i][j] = s * inv;
        }
      }
#pragma unroll
      for (int j = 0; j < D; ++j)
#pragma unroll
        for (int i = j; i < D; ++i) P[(size_t)(c0 + j) * m + c0 + i] = a[i][j];
      if (bad) *fail = 1;
    }
    tm.sync();
    const int r0 = c0 + D;
    if (r0 < m) {
      double l[D][D], inv[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
#pragma unroll
        for (int i = j; i < D; ++i) l[i][j] = P[(size_t)(c0 + j) * m + c0 + i];
        inv[j] = 1.0 / l[j][j];
      }
      for (int r = r0 + tm.rank; r < m; r += tm.size) {
        double x[D];
#pragma unroll
        for (int q = 0; q < D; ++q) x[q] = P[(size_t)(c0 + q) * m + r];
#pragma unroll
        for (int q = 0; q < D; ++q) {
          double s = x[q];
#pragma unroll
          for (int k = 0; k < q; ++k) s -= x[k] * l[q][k];
          x[q] = s * inv[q];
        }
#pragma unroll
        for (int q = 0; q < D; ++q) P[(size_t)(c0 + q) * m + r] = x[q];
      }
      tm.sync();
      const int nc = w - r0;
      if (nc > 0) {
        const int nr = m - r0;
        const int nit = nc * nr;
        for (int it = tm.rank; it < nit; it += tm.size) {
          const int ci = it / nr, ri = it - ci * nr;
          if (ri < ci) continue;
          const int c = r0 + ci, r = r0 + ri;
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s = fma(P[(size_t)(c0 + k) * m + r], P[(size_t)(c0 + k) * m + c], s);
          P[(size_t)c * m + r] -= s;
        }
        tm.sync();
      }
    }
  }
}

// Split the CTA's warps into teams for `nsn` independent panels: warp per panel when there are
// at least NW panels, otherwise power-of-two groups of warps (named barriers 1..NW).
template <int NT>
__device__ __forceinline__ void team_of(int nsn, Team& tm, int& team, int& nteams) {
  constexpr int NW = NT / 32;
  const int warp = threadIdx.x >> 5;
  int tw = 1;
  if (nsn < NW) {
    tw = NW / nsn;
    while (tw & (tw - 1)) tw &= tw - 1;   // round down to a power of two
  }
  nteams = NW / tw;
  team = warp / tw;
  tm.rank = threadIdx.x - team * tw * 32;
  tm.size = tw * 32;
  tm.bar = 1 + team;
}

// Supernodal left-looking Cholesky, level-synchronous.  Each level's panels are one contiguous
// storage range; its prefix [level_off, level_stage_hi) is staged into shared memory `stage`,
// updated (gather form, from descendant panels in global memory), factored by teams, and
// written back.
template <int D, int NT>
__device__ void factor_phase(const DevGraph& g, double* Lg, double* stage, double tol, int* s_fail) {
  for (int lv = 0; lv < g.L; ++lv) {
    const int lo = g.level_off[lv], hi = g.level_stage_hi[lv];
    copy_range<NT>(stage, Lg + lo, hi - lo);
    __syncthreads();
    LView V{Lg, stage, lo, hi};
    // (U) gather-form updates from descendants into this level's panels
    const int t0 = g.ut_level_ptr[lv], t1 = g.ut_level_ptr[lv + 1];
    const int nitems = (t1 - t0) * D;
    for (int itm = threadIdx.x; itm < nitems; itm += NT) {
      const int t = t0 + itm / D, a = itm % D;
      double acc[D];
#pragma unroll
      for (int q = 0; q < D; ++q) acc[q] = 0.0;
      for (int ci = g.ut_cptr[t]; ci < g.ut_cptr[t + 1]; ++ci) {
        const double* A = Lg + g.uc_a[ci];
        const double* Bm = Lg + g.uc_b[ci];
        const int ld = g.uc_ld[ci], w = g.uc_w[ci];
        for (int k = 0; k < w; ++k) {
          const double av = A[(size_t)k * ld + a];
#pragma unroll
          for (int q = 0; q < D; ++q) acc[q] = fma(av, Bm[(size_t)k * ld + q], acc[q]);
        }
      }
      double* T = V.at(g.ut_off[t]);
      const int ld = g.ut_ld[t];
#pragma unroll
      for (int q = 0; q < D; ++q) T[(size_t)q * ld + a] -= acc[q];
    }
    __syncthreads();
    // (F) dense factorisation of the level's panels by teams
    const int s0 = g.level_ptr[lv], nsn = g.level_ptr[lv + 1] - s0;
    Team tm;
    int team, nteams;
    team_of<NT>(nsn, tm, team, nteams);
    for (int i = team; i < nsn; i += nteams) {
      const int s = g.level_sn[s0 + i];
      panel_factor<D>(V.at(g.sn_off[s]), g.sn_m[s], g.sn_w[s], tol, tm, s_fail);
    }
    __syncthreads();
    copy_range<NT>(Lg + lo, stage, hi - lo);
    __syncthreads();
  }
}

// ============================================================================= a4: solves
// Warp-level dense triangular solves on a panel's w x w diagonal block (P column-major, leading
// dim m), rows owned by lanes (row r = lane + 32 j), values held in registers, each step one
// shuffle broadcast.  MAXR = max ceil(w / 32).
template <int MAXR>
__device__ __forceinline__ void warp_trsv_lower(const double* P, int m, int w, double* xs) {
  const int lane = threadIdx.x & 31;
  double t[MAXR], inv[MAXR];
#pragma unroll
  for (int j = 0; j < MAXR; ++j) {
    const int r = lane + 32 * j;
    t[j] = (r < w) ? xs[r] : 0.0;
    inv[j] = (r < w) ? 1.0 / P[(size_t)r * m + r] : 0.0;
  }
#pragma unroll
  for (int sj = 0; sj < MAXR; ++sj) {
    if (32 * sj >= w) break;
    const int cend = min(32, w - 32 * sj);
    for (int cl = 0; cl < cend; ++cl) {
      const int c = 32 * sj + cl;
      const double xc = __shfl_sync(0xffffffffu, t[sj] * inv[sj], cl);
      if (lane == cl) t[sj] = xc;
      const double* col = P + (size_t)c * m;
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
__device__ __forceinline__ void warp_trsv_upper(const double* P, int m, int w, double* xs) {
  // solve L^T x = t : step c from w-1 down to 0, rows r < c updated with L[c][r] = P[r*m + c]
  const int lane = threadIdx.x & 31;
  double t[MAXR], inv[MAXR];
#pragma unroll
  for (int j = 0; j < MAXR; ++j) {
    const int r = lane + 32 * j;
    t[j] = (r < w) ? xs[r] : 0.0;
    inv[j] = (r < w) ? 1.0 / P[(size_t)r * m + r] : 0.0;
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
        if (r < c) t[j] = fma(-P[(size_t)r * m + c], xc, t[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < MAXR; ++j) {
    const int r = lane + 32 * j;
    if (r < w) xs[r] = t[j];
  }
}

// x (permuted, length n; shared or global memory) holds b on entry and H^-1 b on exit.
// Level ranges are staged into `stage` (read-only); warp per supernode.
template <int D, int NT>
__device__ void solve_phase(const DevGraph& g, double* Lg, double* stage, double* x) {
  constexpr int NW = NT / 32;
  constexpr int MAXR = (64 * D + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // forward: L y = b, leaves to root
  for (int lv = 0; lv < g.L; ++lv) {
    const int lo = g.level_off[lv], hi = g.level_stage_hi[lv];
    copy_range<NT>(stage, Lg + lo, hi - lo);
    __syncthreads();
    LView V{Lg, stage, lo, hi};
    const int s0 = g.level_ptr[lv], s1 = g.level_ptr[lv + 1];
    for (int i = s0 + warp; i < s1; i += NW) {
      const int s = g.level_sn[i];
      const int f = g.sn_first[s], w = g.sn_w[s], m = g.sn_m[s];
      const double* P = V.at(g.sn_off[s]);
      double* xs = x + (size_t)D * f;
      for (int r = lane; r < w; r += 32) {
        const int p = f + r / D, a = r % D;
        double t = xs[r];
        for (int ci = g.fc_ptr[p]; ci < g.fc_ptr[p + 1]; ++ci) {
          const double* A = Lg + g.fc_off[ci];
          const int ld = g.fc_ld[ci], ww = g.fc_w[ci];
          const double* y = x + g.fc_x[ci];
          for (int k = 0; k < ww; ++k) t = fma(-A[(size_t)k * ld + a], y[k], t);
        }
        xs[r] = t;
      }
      __syncwarp();
      warp_trsv_lower<MAXR>(P, m, w, xs);
    }
    __syncthreads();
  }
  // backward: L^T x = y, root to leaves
  for (int lv = g.L - 1; lv >= 0; --lv) {
    const int lo = g.level_off[lv], hi = g.level_stage_hi[lv];
    copy_range<NT>(stage, Lg + lo, hi - lo);
    __syncthreads();
    LView V{Lg, stage, lo, hi};
    const int s0 = g.level_ptr[lv], s1 = g.level_ptr[lv + 1];
    for (int i = s0 + warp; i < s1; i += NW) {
      const int s = g.level_sn[i];
      const int f = g.sn_first[s], w = g.sn_w[s], m = g.sn_m[s];
      const double* P = V.at(g.sn_off[s]);
      double* xs = x + (size_t)D * f;
      const int rb = g.snr_ptr[s], nbr = g.snr_ptr[s + 1] - rb;
      for (int c = lane; c < w; c += 32) {
        double t = xs[c];
        const double* col = P + (size_t)c * m + w;
        for (int rr = 0; rr < nbr; ++rr) {
          const double* xr = x + (size_t)D * g.snr[rb + rr];
#pragma unroll
          for (int a = 0; a < D; ++a) t = fma(-col[rr * D + a], xr[a], t);
        }
        xs[c] = t;
      }
      __syncwarp();
      warp_trsv_upper<MAXR>(P, m, w, xs);
    }
    __syncthreads();
  }
}

// ============================================================================= a5: retraction
// Tout[o] = Tin[o] Exp(-alpha delta_o), delta in permuted order
template <int D, int NT>
__device__ void retract_phase(const DevGraph& g, const double* Tin, double* Tout, const double* x, double alpha) {
  constexpr int PS = GT<D>::PS;
  using namespace dev;
  for (int o = threadIdx.x; o < g.N; o += NT) {
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
