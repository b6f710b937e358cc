// libdnls: C-ABI implementation (include/dnls.h) and the sm_100a kernels.
//
// Kernel design: one CTA owns one batch element for the whole solve.
// k_forward runs all K GN/LM iterations plus the final implicit linearisation+factorisation in
// ONE launch: the per-element phases (phases.cuh) are separated by __syncthreads only, so no
// grid-wide synchronisation and no per-iteration launches exist.  The stage-level entry points
// launch thin kernels around the same device phases.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dnls.h"
#include "phases.cuh"
#include "symbolic.h"

// every kernel launch of the library is counted (dnls_debug_launch_count; bench.py's gpu_launches)
namespace dnls {
extern std::atomic<long long> g_launches;
}
#define DNLS_KL ::dnls::g_launches.fetch_add(1, std::memory_order_relaxed),

using namespace dnls;

namespace {
#ifndef DNLS_NT
#define DNLS_NT 384
#endif
constexpr int NT = DNLS_NT;   // threads per CTA (one batch element per CTA)
#ifndef DNLS_MINB
#define DNLS_MINB 1
#endif
constexpr int MINB = DNLS_MINB;   // resident CTAs per SM the register allocation is sized for
constexpr int MAX_CL = 8;         // largest cluster (CTAs sharing one batch element)
constexpr int64_t SMEM_BYTES = 190 * 1024;   // dynamic shared memory per CTA (x + resident + staging); the rest of the 256 KB unified L1 caches the global panels (measured optimum, tools/smem_sweep.sh)
thread_local std::string g_err;

dnls_status fail(dnls_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
dnls_status cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DNLS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return DNLS_OK;
}
size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }
}  // namespace

namespace {
struct BLPlan;
void bl_plan_delete(BLPlan* p);
}  // namespace

struct dnls_graph {
  Symbolic sym;
  // batch-interleaved level-major plan (bl.cuh), built on first use
  BLPlan* bl = nullptr;
  std::string bl_err;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> phase_ev;   // factorisation phases of the last BL forward
  std::mutex bl_mu;
  int device = 0;
  int* dbuf = nullptr;
  size_t dbuf_bytes = 0;
  DevGraph dg{};
  std::mutex mu;
  // Factor cache registry (include/dnls.h "Ownership"): workspace base -> what its factor storage
  // holds for (graph, batch).  An implicit forward registers its workspace; every entry point that
  // writes the factor storage of a workspace drops it, so a backward on a workspace whose cached
  // factor was overwritten (or never made) returns DNLS_E_STATE.  Several workspaces may hold
  // cached factors of the same graph at once.
  struct FactorRecord {
    int batch;
    int kind;   // DNLS_BWD_* of the forward that wrote it
    int K;      // unroll: iterations whose factors are kept
    double alpha = 1.0;   // unroll: the GN step size of the recorded forward
    int layout = 0;       // 0: per-element storage, 1: batch-interleaved (bl.cuh)
  };
  std::map<const void*, FactorRecord> cached;
  void drop(const void* ws) {
    std::lock_guard<std::mutex> lk(mu);
    cached.erase(ws);
  }
  void keep(const void* ws, FactorRecord r) {
    std::lock_guard<std::mutex> lk(mu);
    cached[ws] = r;
  }
  bool get(const void* ws, FactorRecord& r) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cached.find(ws);
    if (it == cached.end()) return false;
    r = it->second;
    return true;
  }
};

namespace {
// the stage-level views read the per-element storage: a workspace whose last forward ran the batch-interleaved
// path holds its factor element-interleaved -- refused instead of read as garbage
dnls_status per_element_storage(const char* what, const dnls_graph* g, const void* ws) {
  dnls_graph::FactorRecord rec;
  if (const_cast<dnls_graph*>(g)->get(ws, rec) && rec.layout == 1)
    return fail(DNLS_E_UNSUPPORTED, std::string(what) + ": the workspace holds the batch-interleaved factor of the "
                                    "last dnls_forward (batch_interleave = 1 keeps the per-element layout)");
  return DNLS_OK;
}
// Runs the calling thread's CUDA calls on the graph's device and restores the previous one
// (the graph's index arrays and the caller's buffers live on that device).
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      prev = -1;
      cudaGetLastError();
    }
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    if (!ok) cudaGetLastError();
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

// ----------------------------------------------------------------------------- workspace layout
namespace {
struct WsLayout {
  size_t L, x, bsave, jac, cost, rgrad, trial, S, Sprev, lam, maxd, st, it, clred, hT, hd, hL, total;
  int keep;
};
// keep > 0: room for the unroll / truncated history of `keep` GN iterations per element
WsLayout ws_layout(const Symbolic& s, int B, int keep = 0) {
  const int D = s.D, PS = D == 6 ? 12 : 6, JS = D == 6 ? Scr<6>::SIZE : Scr<3>::SIZE;   // GT<D>::JS
  const size_t n = (size_t)s.N * D, slots = (size_t)s.E + s.P;
  WsLayout w{};
  size_t o = 0;
  w.L = o;     o = align_up(o + sizeof(double) * (size_t)B * s.storage);
  w.x = o;     o = align_up(o + sizeof(double) * (size_t)B * n);
  w.bsave = o; o = align_up(o + sizeof(double) * (size_t)B * n);
  w.jac = o;   o = align_up(o + sizeof(double) * (size_t)B * slots * JS);
  w.cost = o;  o = align_up(o + sizeof(double) * (size_t)B * slots);
  w.rgrad = o; o = align_up(o + sizeof(double) * (size_t)B * slots);
  w.trial = o; o = align_up(o + sizeof(double) * (size_t)B * s.N * PS);
  w.S = o;     o = align_up(o + sizeof(double) * B);
  w.Sprev = o; o = align_up(o + sizeof(double) * B);
  w.lam = o;   o = align_up(o + sizeof(double) * B);
  w.maxd = o;  o = align_up(o + sizeof(double) * B);
  w.st = o;    o = align_up(o + sizeof(int) * B);
  w.it = o;    o = align_up(o + sizeof(int) * B);
  w.clred = o; o = align_up(o + sizeof(double) * B * 2 * MAX_CL);
  w.keep = keep;
  w.hT = o;    o = align_up(o + sizeof(double) * (size_t)B * keep * s.N * PS);
  w.hd = o;    o = align_up(o + sizeof(double) * (size_t)B * keep * n);
  w.hL = o;    o = align_up(o + sizeof(double) * (size_t)B * keep * s.storage);
  w.total = o;
  return w;
}
// iterations an unroll / truncated forward records (0 for the other modes)
int history_keep(const dnls_options* opt) {
  if (!opt) return 0;
  if (opt->backward_mode == DNLS_BWD_UNROLL) return std::max(0, (int)opt->max_iterations);
  if (opt->backward_mode == DNLS_BWD_TRUNCATED)
    return std::max(0, std::min((int)opt->max_iterations, (int)opt->backward_steps));
  return 0;
}
DevWs ws_views(const WsLayout& l, void* base) {
  char* p = (char*)base;
  DevWs w;
  w.L = (double*)(p + l.L);
  w.x = (double*)(p + l.x);
  w.bsave = (double*)(p + l.bsave);
  w.jac = (double*)(p + l.jac);
  w.cost = (double*)(p + l.cost);
  w.rgrad = (double*)(p + l.rgrad);
  w.trial = (double*)(p + l.trial);
  w.S = (double*)(p + l.S);
  w.Sprev = (double*)(p + l.Sprev);
  w.lam = (double*)(p + l.lam);
  w.maxd = (double*)(p + l.maxd);
  w.st = (int*)(p + l.st);
  w.it = (int*)(p + l.it);
  w.clred = (double*)(p + l.clred);
  w.keep = l.keep;
  w.hT = (double*)(p + l.hT);
  w.hd = (double*)(p + l.hd);
  w.hL = (double*)(p + l.hL);
  return w;
}
DevProb dev_prob(const dnls_problem* p) {
  DevProb d;
  d.poses = p->poses;
  d.meas = p->meas;
  d.prior_meas = p->prior_meas;
  d.pm_bstride = p->prior_meas_bstride;
  d.w_edge = p->w_edge;
  d.we_bstride = p->w_edge_bstride;
  d.w_prior = p->w_prior;
  d.wp_bstride = p->w_prior_bstride;
  d.radius = p->radius;
  d.r_bstride = p->radius_bstride;
  return d;
}
}  // namespace

// ============================================================================= kernels
namespace dnls {
struct FwdParams {
  int K;
  int lm;
  double alpha;
  double lam0, lam_min, lam_max, lam_down, lam_up;
  int damping;
  int early_stop;
  double abs_tol, rel_tol;
  int implicit;
  int dogleg;
  double dl0, dl_max, dl_min;   // trust radius
  double* objective;
  int* status;
  int* iterations;
};
// k_forward with clusters of CL CTAs per element, compiled in its own translation unit
// (dnls_cluster.cu: instantiating it here changes the inlining of the shared device phases and
// makes the one-CTA kernel spill).  Returns the launch error.
cudaError_t launch_forward_cluster(int CL, int D, const DevGraph& g, DevProb pr, DevWs ws, FwdParams fp, int batch,
                                   cudaStream_t s);
}  // namespace dnls

namespace {

size_t smem_bytes(const DevGraph& g) {
  return sizeof(double) * ((g.x_smem ? (size_t)g.n_pad : 0) + (size_t)g.res_n + (size_t)g.stage_n) +
         sizeof(int) * 2 * (size_t)g.pk_max;
}
size_t smem_bytes_grouped(const DevGraph& g) { return sizeof(int) * 2 * (size_t)g.pk_max; }

template <class F>
dnls_status set_smem(F* kernel, size_t bytes, const char* what) {
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return fail(DNLS_E_CUDA, std::string(what) + ": cudaFuncSetAttribute: " + cudaGetErrorString(cudaGetLastError()));
  return DNLS_OK;
}

// per-CTA shared memory views
struct Smem {
  double* x;        // solution vector (shared or global)
  double* res;      // resident top levels of the factor storage
  double* stage;    // level staging area / per-warp forest slices
  double* xinv;     // per-team D x D scratch (inverse diagonal of the current diagonal block)
  PkPipe pp;        // double-buffered descriptor packets
  uint64_t* mbar;   // mbarrier of the bulk (TMA) loads
  uint32_t phase;
};
// must be called by every thread at kernel start (initialises the mbarrier, one barrier).
// grouped == true (a cluster shares the element): x, the factor and the staging stay in global
// memory; shared memory holds only the descriptor packets.
__device__ __forceinline__ Smem smem_views(const DevGraph& g, double* xg, bool grouped = false) {
  extern __shared__ __align__(16) double smem[];
  __shared__ uint64_t s_mbar, s_mbpk[2];
  __shared__ double s_xinv[(NT / 32) * 36];
  Smem v;
  const bool xs = g.x_smem && !grouped;
  v.x = xs ? smem : xg;
  v.res = smem + (xs ? g.n_pad : 0);
  v.stage = v.res + (grouped ? 0 : g.res_n);
  v.pp.buf[0] = reinterpret_cast<int*>(v.stage + (grouped ? 0 : g.stage_n));
  v.pp.buf[1] = v.pp.buf[0] + g.pk_max;
  v.pp.mb[0] = &s_mbpk[0];
  v.pp.mb[1] = &s_mbpk[1];
  v.pp.ph[0] = v.pp.ph[1] = 0;
  v.xinv = s_xinv;
  v.mbar = &s_mbar;
  v.phase = 0;
  if (threadIdx.x == 0) {
    mbar_init(&s_mbar);
    mbar_init(&s_mbpk[0]);
    mbar_init(&s_mbpk[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");   // visible to the async proxy
  }
  __syncthreads();
  return v;
}
__device__ __forceinline__ LView full_view(const DevGraph& g, double* Lg, const Smem& sm) {
  return LView{Lg, sm.res, g.res_lo, nullptr, 0, 0};
}
__device__ __forceinline__ LView global_view(const DevGraph& g, double* Lg) {
  return LView{Lg, nullptr, g.storage, nullptr, 0, 0};
}


// group-wide: S = sum(cost) (fixed order, identical in every CTA of the group), maxdiag = max
// over warps (and over the group's CTAs through the global scratch clr[CL]).  Returns via shared
// variables.
template <int D, int CL = 1>
__device__ void finish_assembly(const DevGraph& g, const double* cost_b, double* s_red, double* sh_S,
                                double* sh_max, double* clr = nullptr) {
  DNLS_PROBE_NOW(q0);
  gsync<CL>();
  DNLS_PROBE_NOW(q1);
  DNLS_PROBE_ADD(4, q0, q1);
  {   // S: every thread one strided share, fixed shuffle tree, warps in order (deterministic and
      // identical in every CTA of a group, which all sum the whole array)
    __shared__ double s_part[NT / 32];
    double part = 0.0;
    for (int i = threadIdx.x; i < g.E + g.P; i += NT) part += cost_b[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      double sum = 0.0, m = 0.0;
      for (int i = 0; i < NT / 32; ++i) {
        sum += s_part[i];
        m = fmax(m, s_red[i]);
      }
      *sh_S = sum;
      if (CL > 1) clr[crank<CL>()] = m;
      else *sh_max = m;
    }
  }
  if (CL > 1) {
    gsync<CL>();
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int i = 0; i < CL; ++i) m = fmax(m, clr[i]);
      *sh_max = m;
    }
  }
  __syncthreads();
  DNLS_PROBE_NOW(q2);
  DNLS_PROBE_ADD(5, q1, q2);
}
// group-wide OR of the per-CTA factorisation failure flags (after a group barrier)
template <int CL>
__device__ void group_fail(int* sh_fail, double* clr) {
  if constexpr (CL > 1) {
    if (threadIdx.x == 0) clr[CL + crank<CL>()] = (double)*sh_fail;
    gsync<CL>();
    if (threadIdx.x == 0) {
      int f = 0;
      for (int i = 0; i < CL; ++i) f |= clr[CL + i] != 0.0;
      *sh_fail = f;
    }
  }
  __syncthreads();
}

// CTA-wide deterministic sum (fixed shuffle tree, warps summed in order); every thread gets it
__device__ __forceinline__ double cta_sum(double v, double* s_tmp) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_tmp[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < NT / 32; ++i) t += s_tmp[i];
  __syncthreads();
  return t;
}
// CTA-wide deterministic sum of v[0..n): strided per-thread shares, fixed shuffle tree, warps in
// order; every thread of the CTA gets the value (identical in every CTA of a group)
__device__ __forceinline__ double cta_sum_array(const double* v, int n, double* s_tmp) {
  double part = 0.0;
  for (int i = threadIdx.x; i < n; i += NT) part += v[i];
  return cta_sum(part, s_tmp);
}
// packed lower-triangular quadratic form u^T H u (H symmetric, lower triangle packed column-wise)
template <int D>
__device__ __forceinline__ double quad_lower(const double* h, const double* u) {
  double v = 0.0;
  int e = 0;
#pragma unroll
  for (int q = 0; q < D; ++q)
#pragma unroll
    for (int a = q; a < D; ++a) {
      const double t = h[e++] * u[a] * u[q];
      v += (a == q) ? t : 2.0 * t;
    }
  return v;
}
// b^T H_s b of one cost slot from its H contributions (scratch diagonal parts, the off-diagonal
// block in the factor storage -- before the factorisation overwrites it -- or in the scratch for
// parallel edges).  x_b holds b (permuted order).  Dogleg's Cauchy point needs sum_s b^T H_s b.
template <int D>
__device__ double slot_bHb(const DevGraph& g, const LView& L, const double* x_b, const double* scr, int slot) {
  using SC = Scr<D>;
  const int4 d0 = g.slot_desc[3 * slot], d1 = g.slot_desc[3 * slot + 1], d2 = g.slot_desc[3 * slot + 2];
  const double* o = scr + (size_t)slot * SC::SIZE;
  const double* bi = x_b + (size_t)D * d2.x;
  double v = quad_lower<D>(o + SC::H0, bi);
  if (d0.y >= 0) {
    const double* bj = x_b + (size_t)D * d2.y;
    v += quad_lower<D>(o + SC::H1, bj);
    const double* O = d2.z ? L.at(d0.z) : o + SC::HIJ;
    const int ld = d2.z ? d1.z : D;
    const double* br = d0.w ? bj : bi;   // block rows: pose P (j if d0.w), columns: the other pose
    const double* bc = d0.w ? bi : bj;
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q)
#pragma unroll
      for (int a = 0; a < D; ++a) t += br[a] * O[(size_t)q * ld + a] * bc[q];
    v += 2.0 * t;
  }
  return v;
}

// CL > 1: a cluster of CL CTAs shares element blockIdx.x / CL (few large problems)
template <int D, int CL>
__global__ void __launch_bounds__(NT, MINB) k_forward(DevGraph g, DevProb pr, DevWs ws, FwdParams fp) {
  constexpr int PS = GT<D>::PS, JS = GT<D>::JS;
  const int b = blockIdx.x / CL;
  const int cr = crank<CL>();
  double* const clr = CL > 1 ? ws.clred + (size_t)b * 2 * CL : nullptr;   // no live register at CL == 1
  __shared__ double s_red[NT / 32];
  __shared__ double sh_S, sh_max, sh_Stry;
  __shared__ int sh_fail;
  const size_t slots = (size_t)g.E + g.P;
  double* Tb = pr.poses + (size_t)b * g.N * PS;
  double* Ttr = ws.trial + (size_t)b * g.N * PS;
  double* jac_b = ws.jac + (size_t)b * slots * JS;
  double* cost_b = ws.cost + (size_t)b * slots;
  double* Lg = ws.L + (size_t)b * g.storage;
  Smem sm = smem_views(g, ws.x + (size_t)b * g.n, CL > 1);
  double* x_b = sm.x;
  const LView L = CL > 1 ? global_view(g, Lg) : full_view(g, Lg, sm);

  int status = DNLS_ST_OK, iters = 0;
  double lam = fp.lam0, Sprev = 0.0;
  // Dogleg state in shared memory (not live in registers across the factorisation):
  // [0] trust radius, [1] b.b, [2] b.Hb, [3] y.y
  __shared__ double s_tmp[NT / 32], sh_dl[4];
  if (threadIdx.x == 0) sh_dl[0] = fp.dl0;
  bool have_prev = false;
  for (int k = 0; k < fp.K; ++k) {
    // a1 + a2 at theta_k
    DNLS_TRACE_POINT(100);
    DNLS_TRACE_POINT(200);
#ifndef DNLS_SKIP_LIN
    linearize_phase<D, NT, CL>(g, pr, Tb, b, L, x_b, cost_b, jac_b, fp.lm ? lam : -1.0, fp.damping, s_red);
#endif
    finish_assembly<D, CL>(g, cost_b, s_red, &sh_S, &sh_max, clr);
    DNLS_TRACE_POINT(300);
    const double S = sh_S;
    if (fp.early_stop && have_prev && fabs(S - Sprev) < fp.abs_tol + fp.rel_tol * Sprev) {
      status = DNLS_ST_CONVERGED;
      break;
    }
    if (CL == 1 && fp.dogleg) {   // b = J^T r (saved), b.b and b.Hb before the factor overwrites H
      double* bs = ws.bsave + (size_t)b * g.n;
      double pb = 0.0, ph = 0.0;
      for (int i = threadIdx.x; i < g.n; i += NT) {
        const double v = x_b[i];
        bs[i] = v;
        pb = fma(v, v, pb);
      }
      for (int sl = threadIdx.x; sl < g.E + g.P; sl += NT) ph += slot_bHb<D>(g, L, x_b, jac_b, sl);
      const double bb = cta_sum(pb, s_tmp), bHb = cta_sum(ph, s_tmp);
      if (threadIdx.x == 0) {
        sh_dl[1] = bb;
        sh_dl[2] = bHb;
      }
    }
    if (threadIdx.x == 0) sh_fail = 0;
    __syncthreads();
    factor_phase<D, NT, CL>(g, L, sm.stage, 1e-13 * sh_max, &sh_fail, sm.mbar, sm.phase, sm.xinv, x_b, sm.pp);
    group_fail<CL>(&sh_fail, clr);
    const bool ok = sh_fail == 0;
    __syncthreads();
    if (CL == 1 && fp.dogleg && ok) {   // y = L^-1 b: b^T H^-1 b = y.y
      double py = 0.0;
      for (int i = threadIdx.x; i < g.n; i += NT) py = fma(x_b[i], x_b[i], py);
      const double yy = cta_sum(py, s_tmp);
      if (threadIdx.x == 0) sh_dl[3] = yy;
    }
    if (CL == 1 && fp.dogleg) {   // Powell's dogleg (reading DL1)
      ++iters;
      if (!ok) {
        status = DNLS_ST_NOT_SPD;
        break;
      }
      solve_phase<D, NT, CL>(g, L, sm.stage, x_b, sm.mbar, sm.phase, sm.pp, false);   // x_b = d_gn = H^-1 b
      double pg = 0.0;
      for (int i = threadIdx.x; i < g.n; i += NT) pg = fma(x_b[i], x_b[i], pg);
      const double gg = cta_sum(pg, s_tmp);
      const double delta = sh_dl[0], bb = sh_dl[1], bHb = sh_dl[2], yy = sh_dl[3];
      const double* bs = ws.bsave + (size_t)b * g.n;
      // step d = alpha b + beta d_gn; scalars from H d_gn = b, d_gn.b = y.y (identical in all threads)
      double alpha, beta;
      if (sqrt(gg) <= delta) {
        alpha = 0.0;
        beta = 1.0;
      } else {
        const double kappa = bb / bHb;   // Cauchy point d_c = kappa b
        if (kappa * sqrt(bb) >= delta) {
          alpha = delta / sqrt(bb);
          beta = 0.0;
        } else {   // |d_c + tau (d_gn - d_c)| = delta
          const double uu = gg - 2.0 * kappa * yy + kappa * kappa * bb;
          const double qb = 2.0 * (kappa * yy - kappa * kappa * bb), qc = kappa * kappa * bb - delta * delta;
          const double tau = (-qb + sqrt(qb * qb - 4.0 * uu * qc)) / (2.0 * uu);
          alpha = (1.0 - tau) * kappa;
          beta = tau;
        }
      }
      const double pred = (alpha * bb + beta * yy) - 0.5 * (alpha * alpha * bHb + 2.0 * alpha * beta * bb +
                                                            beta * beta * yy);
      for (int i = threadIdx.x; i < g.n; i += NT) x_b[i] = alpha * bs[i] + beta * x_b[i];
      __syncthreads();
      retract_phase<D, NT, CL>(g, Tb, Ttr, x_b, 1.0);
      __syncthreads();
      objective_phase<D, NT, CL>(g, pr, Ttr, b, cost_b);
      __syncthreads();
      {
        const double st = cta_sum_array(cost_b, g.E + g.P, s_tmp);
        if (threadIdx.x == 0) sh_Stry = st;
      }
      __syncthreads();
      const double rho = pred > 0.0 ? (S - sh_Stry) / pred : 0.0;
      const double delta_new = rho > 0.75 ? fmin(2.0 * delta, fp.dl_max) : (rho < 0.25 ? 0.5 * delta : delta);
      __syncthreads();
      if (threadIdx.x == 0) sh_dl[0] = delta_new;
      if (rho > 0.0) {
        for (int i = threadIdx.x; i < g.N * PS; i += NT) Tb[i] = Ttr[i];
        __syncthreads();
        Sprev = S;
        have_prev = true;
      } else if (delta_new < fp.dl_min) {
        status = DNLS_ST_SATURATED;
        break;
      }
    } else if (!fp.lm) {
#ifndef DNLS_ABLATE   // development builds that skip a phase (timing ablation) must not stop early
      if (!ok) {
        status = DNLS_ST_NOT_SPD;
        break;
      }
#endif
      solve_phase<D, NT, CL>(g, L, sm.stage, x_b, sm.mbar, sm.phase, sm.pp, false);
      DNLS_TRACE_POINT(400);
      if (CL == 1 && ws.keep > 0) {   // unroll / truncated history: theta_k, delta_k, the factor of H(theta_k)
        const size_t hs = (size_t)b * ws.keep + (k % ws.keep);
        double* hT = ws.hT + hs * g.N * PS;
        for (int i = threadIdx.x; i < g.N * PS; i += NT) hT[i] = Tb[i];
        double* hd = ws.hd + hs * g.n;
        for (int i = threadIdx.x; i < g.n; i += NT) hd[i] = x_b[i];
        double* hL = ws.hL + hs * g.storage;
        copy_range<NT>(hL, Lg, g.res_lo);
        copy_range<NT>(hL + g.res_lo, sm.res, g.storage - g.res_lo);
        __syncthreads();
      }
      retract_phase<D, NT, CL>(g, Tb, Tb, x_b, fp.alpha);
      gsync<CL>();
      DNLS_TRACE_POINT(500);
      ++iters;
      Sprev = S;
      have_prev = true;
    } else {
      ++iters;
      bool accept = false;
      if (ok) {
        solve_phase<D, NT, CL>(g, L, sm.stage, x_b, sm.mbar, sm.phase, sm.pp, false);
        retract_phase<D, NT, CL>(g, Tb, Ttr, x_b, fp.alpha);
        gsync<CL>();
        objective_phase<D, NT, CL>(g, pr, Ttr, b, cost_b);
        gsync<CL>();
        {
          const double st = cta_sum_array(cost_b, g.E + g.P, s_tmp);
          if (threadIdx.x == 0) sh_Stry = st;
        }
        __syncthreads();
        accept = sh_Stry < S;
      }
      if (accept) {
        for (int i = cr * NT + threadIdx.x; i < g.N * PS; i += CL * NT) Tb[i] = Ttr[i];
        gsync<CL>();
        lam = fmax(lam / fp.lam_down, fp.lam_min);
        Sprev = S;
        have_prev = true;
      } else {
        if (lam >= fp.lam_max) {
          status = DNLS_ST_SATURATED;
          break;
        }
        lam = fmin(lam * fp.lam_up, fp.lam_max);
      }
    }
  }
  __syncthreads();
  // final objective S(theta_K); implicit: undamped H(theta_K) and its factor stay in ws
  if (fp.implicit) {
    linearize_phase<D, NT, CL>(g, pr, Tb, b, L, x_b, cost_b, jac_b, -1.0, 0, s_red);
    finish_assembly<D, CL>(g, cost_b, s_red, &sh_S, &sh_max, clr);
    if (threadIdx.x == 0) sh_fail = 0;
    __syncthreads();
    factor_phase<D, NT, CL>(g, L, sm.stage, 1e-13 * sh_max, &sh_fail, sm.mbar, sm.phase, sm.xinv, nullptr, sm.pp);
    group_fail<CL>(&sh_fail, clr);
    // a failed final factor takes precedence over CONVERGED / SATURATED: the backward must not use it
    if (sh_fail) status = DNLS_ST_NOT_SPD;
    // Prop. 1 assumes theta* optimal: warn (not fail) when the last accepted step still
    // changed the objective by more than the early-stop tolerance
    else if (have_prev && !(fabs(sh_S - Sprev) < fp.abs_tol + fp.rel_tol * Sprev)) status |= DNLS_ST_WARN_NOT_CONVERGED;
    // the cached factor must be complete in global memory for dnls_backward_implicit
    if (CL == 1) copy_range<NT>(Lg + g.res_lo, sm.res, g.storage - g.res_lo);
  } else {
    objective_phase<D, NT, CL>(g, pr, Tb, b, cost_b);
    gsync<CL>();
    {
      const double st = cta_sum_array(cost_b, g.E + g.P, s_tmp);
      if (threadIdx.x == 0) sh_S = st;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && cr == 0) {
    if (fp.objective) fp.objective[b] = sh_S;
    if (fp.status) fp.status[b] = status;
    if (fp.iterations) fp.iterations[b] = iters;
    ws.S[b] = sh_S;
    ws.lam[b] = fp.dogleg ? sh_dl[0] : lam;
    ws.st[b] = status;
    ws.it[b] = iters;
  }
}

#ifndef DNLS_CLUSTER_TU
template <int D>
__global__ void __launch_bounds__(NT, MINB) k_linearize(DevGraph g, DevProb pr, DevWs ws, const double* lam,
                                                      int damping, double* objective) {
  constexpr int PS = GT<D>::PS, JS = GT<D>::JS;
  const int b = blockIdx.x;
  __shared__ double s_red[NT / 32];
  __shared__ double sh_S, sh_max;
  const size_t slots = (size_t)g.E + g.P;
  const double* Tb = pr.poses + (size_t)b * g.N * PS;
  double* jac_b = ws.jac + (size_t)b * slots * JS;
  double* cost_b = ws.cost + (size_t)b * slots;
  const LView L = global_view(g, ws.L + (size_t)b * g.storage);
  double* xg = ws.x + (size_t)b * g.n;
  Smem sm = smem_views(g, xg);
  linearize_phase<D, NT>(g, pr, Tb, b, L, sm.x, cost_b, jac_b, lam ? lam[b] : -1.0, damping, s_red);
  finish_assembly<D>(g, cost_b, s_red, &sh_S, &sh_max);
  if (g.x_smem)
    for (int i = threadIdx.x; i < g.n; i += NT) xg[i] = sm.x[i];
  if (threadIdx.x == 0) {
    if (objective) objective[b] = sh_S;
    ws.S[b] = sh_S;
    ws.maxd[b] = sh_max;
  }
}

template <int D>
__global__ void __launch_bounds__(NT, MINB) k_factorize(DevGraph g, DevWs ws, int* status) {
  const int b = blockIdx.x;
  __shared__ int sh_fail;
  if (threadIdx.x == 0) sh_fail = 0;
  __syncthreads();
  Smem sm = smem_views(g, ws.x + (size_t)b * g.n);
  double* Lg = ws.L + (size_t)b * g.storage;
  bulk_load<NT>(sm.res, Lg + g.res_lo, g.storage - g.res_lo, sm.mbar, sm.phase);
  factor_phase<D, NT>(g, full_view(g, Lg, sm), sm.stage, 1e-13 * ws.maxd[b], &sh_fail, sm.mbar, sm.phase, sm.xinv,
                      nullptr, sm.pp);
  copy_range<NT>(Lg + g.res_lo, sm.res, g.storage - g.res_lo);
  __syncthreads();
  if (threadIdx.x == 0 && status) status[b] = sh_fail ? DNLS_ST_NOT_SPD : DNLS_ST_OK;
}

// rhs/x in original order [B][N][D]
template <int D>
__global__ void __launch_bounds__(NT, MINB) k_solve(DevGraph g, DevWs ws, const double* rhs, double* xout) {
  const int b = blockIdx.x;
  Smem sm = smem_views(g, ws.x + (size_t)b * g.n);
  double* x_b = sm.x;
  for (int i = threadIdx.x; i < g.n; i += NT) {
    const int o = i / D, a = i - o * D;
    x_b[(size_t)g.iperm[o] * D + a] = rhs[(size_t)b * g.n + i];
  }
  double* Lg = ws.L + (size_t)b * g.storage;
  bulk_load<NT>(sm.res, Lg + g.res_lo, g.storage - g.res_lo, sm.mbar, sm.phase);
  solve_phase<D, NT>(g, full_view(g, Lg, sm), sm.stage, x_b, sm.mbar, sm.phase, sm.pp);
  __syncthreads();
  for (int i = threadIdx.x; i < g.n; i += NT) {
    const int o = i / D, a = i - o * D;
    xout[(size_t)b * g.n + i] = x_b[(size_t)g.iperm[o] * D + a];
  }
}

// upstream gradient of pose o (original order) in right-tangent coordinates: given directly
// (DNLS_GRAD_TANGENT) or projected from the Euclidean gradient on the matrix entries (App. D)
template <int D>
__device__ __forceinline__ void tangent_grad(const double* Tb, const double* gpose, int grad_kind, int b, int N,
                                             int o, double (&v)[D]) {
  constexpr int PS = GT<D>::PS;
  if (grad_kind == DNLS_GRAD_TANGENT) {
#pragma unroll
    for (int a = 0; a < D; ++a) v[a] = gpose[((size_t)b * N + o) * D + a];
  } else {
    // v_a = < dL/dT , T G_a >  (top rows), G_a the Lie-algebra generators
    const double* G = gpose + ((size_t)b * N + o) * PS;
    const double* T = Tb + (size_t)o * PS;
    if (D == 6) {
      // T G_a for translation generators: column 3 = R e_a ; rotation generators: R [e_a]x in the
      // 3x3 block.   <G, R[e]x> = sum_ij G_ij (R[e]x)_ij
#pragma unroll
      for (int a = 0; a < 3; ++a) v[a] = G[0 * 4 + 3] * T[0 * 4 + a] + G[1 * 4 + 3] * T[1 * 4 + a] + G[2 * 4 + 3] * T[2 * 4 + a];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double e[3] = {0.0, 0.0, 0.0};
        e[a] = 1.0;
        // [e]x columns: col0 = (0, e2, -e1), col1 = (-e2, 0, e0), col2 = (e1, -e0, 0)
        double Ex[3][3] = {{0.0, -e[2], e[1]}, {e[2], 0.0, -e[0]}, {-e[1], e[0], 0.0}};
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            double rex = T[i * 4 + 0] * Ex[0][j] + T[i * 4 + 1] * Ex[1][j] + T[i * 4 + 2] * Ex[2][j];
            acc += G[i * 4 + j] * rex;
          }
        v[3 + a] = acc;
      }
    } else {
      v[0] = G[2] * T[0] + G[5] * T[3];
      v[1] = G[2] * T[1] + G[5] * T[4];
      // rotation generator [[0,-1],[1,0]]: R*Gen = [[R01, -R00], [R11, -R10]]
      v[2] = G[0] * T[1] - G[1] * T[0] + G[3] * T[4] - G[4] * T[3];
    }
  }
}

// implicit backward, per element: v -> lambda = H^-1 v (cached factor) -> per-slot weight grads
template <int D>
__global__ void __launch_bounds__(NT, MINB) k_backward(DevGraph g, DevProb pr, DevWs ws, const double* gpose,
                                                     int grad_kind) {
  constexpr int PS = GT<D>::PS;
  const int b = blockIdx.x;
  const size_t slots = (size_t)g.E + g.P;
  const double* Tb = pr.poses + (size_t)b * g.N * PS;
  Smem sm = smem_views(g, ws.x + (size_t)b * g.n);
  double* x_b = sm.x;
  double* out_b = ws.cost + (size_t)b * slots;
  double* rg_b = ws.rgrad + (size_t)b * slots;
  if (ws.st[b] == DNLS_ST_NOT_SPD) {   // no valid factor: zero gradient contribution
    for (int s = threadIdx.x; s < (int)slots; s += NT) out_b[s] = rg_b[s] = 0.0;
    return;
  }
  // v (original order) -> permuted
  for (int o = threadIdx.x; o < g.N; o += NT) {
    double v[D];
    tangent_grad<D>(Tb, gpose, grad_kind, b, g.N, o, v);
#pragma unroll
    for (int a = 0; a < D; ++a) x_b[(size_t)g.iperm[o] * D + a] = v[a];
  }
  double* Lg = ws.L + (size_t)b * g.storage;
  bulk_load<NT>(sm.res, Lg + g.res_lo, g.storage - g.res_lo, sm.mbar, sm.phase);
  solve_phase<D, NT>(g, full_view(g, Lg, sm), sm.stage, x_b, sm.mbar, sm.phase, sm.pp);
  __syncthreads();
  // dL/dw = -2 w (C lambda) . c  (unweighted C, c at theta_K)
  for (int slot = threadIdx.x; slot < (int)slots; slot += NT) {
    double c[D], Ci[D * D], Cj[D * D];
    eval_slot<D>(g, pr, Tb, b, slot, c, Ci, Cj, true);
    const double w = slot_weight<D>(g, pr, b, slot);
    double dot = 0.0;
    if (slot < g.E) {
      const double* li = x_b + (size_t)D * g.iperm[g.edges[2 * slot]];
      const double* lj = x_b + (size_t)D * g.iperm[g.edges[2 * slot + 1]];
#pragma unroll
      for (int r = 0; r < D; ++r) {
        double cl = 0.0;
#pragma unroll
        for (int q = 0; q < D; ++q) cl += Ci[r * D + q] * li[q] + Cj[r * D + q] * lj[q];
        dot += cl * c[r];
      }
    } else {
      const double* lp = x_b + (size_t)D * g.iperm[g.prior_vars[slot - g.E]];
#pragma unroll
      for (int r = 0; r < D; ++r) {
        double cl = 0.0;
#pragma unroll
        for (int q = 0; q < D; ++q) cl += Ci[r * D + q] * lp[q];
        dot += cl * c[r];
      }
    }
    // Welsch edge (W1-W2): g_e = psi w^2 C^T c  =>  d/dw = 2 w psi (1 - s/k^2),  d/dk = (2 s/k^3) psi w^2
    double n2 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) n2 = fma(c[a], c[a], n2);
    double psi;
    const double sq = w * w * n2;
    slot_cost(g, pr, b, slot, sq, psi);
    double fw = 1.0, rg = 0.0;
    if (pr.radius != nullptr && slot < g.E) {
      const double k = pr.radius[(size_t)b * pr.r_bstride];
      fw = psi * (1.0 - sq / (k * k));
      rg = -2.0 * sq / (k * k * k) * psi * w * w * dot;
    }
    out_b[slot] = -2.0 * w * fw * dot;
    rg_b[slot] = rg;
  }
}

// DLM backward (PAPER.md :259-271, App. :897-934; readings B1-B3), per element:
//   linearise at theta*, H_a = J^T J + 2 eps^2 I (identity damping), rhs = J^T r - eps v,
//   factor + solve (one extra factorisation), theta_direct = theta* [+] (-delta_a)  (one GN step),
//   per slot  g = (w / eps) (||c(theta*)||^2 - ||c(theta_direct)||^2)  -> k_reduce_wgrad.
template <int D>
__global__ void __launch_bounds__(NT, MINB) k_backward_dlm(DevGraph g, DevProb pr, DevWs ws, const double* gpose,
                                                         int grad_kind, double eps) {
  constexpr int PS = GT<D>::PS, JS = GT<D>::JS;
  const int b = blockIdx.x;
  __shared__ double s_red[NT / 32];
  __shared__ double sh_S, sh_max;
  __shared__ int sh_fail;
  const size_t slots = (size_t)g.E + g.P;
  const double* Tb = pr.poses + (size_t)b * g.N * PS;
  double* Tdir = ws.trial + (size_t)b * g.N * PS;
  double* jac_b = ws.jac + (size_t)b * slots * JS;
  double* cost_b = ws.cost + (size_t)b * slots;
  double* Lg = ws.L + (size_t)b * g.storage;
  Smem sm = smem_views(g, ws.x + (size_t)b * g.n);
  double* x_b = sm.x;
  const LView L = full_view(g, Lg, sm);
  linearize_phase<D, NT>(g, pr, Tb, b, L, x_b, cost_b, jac_b, 2.0 * eps * eps, DNLS_DAMP_IDENTITY, s_red);
  finish_assembly<D>(g, cost_b, s_red, &sh_S, &sh_max);
  for (int o = threadIdx.x; o < g.N; o += NT) {   // rhs = J^T r - eps v  (permuted order)
    double v[D];
    tangent_grad<D>(Tb, gpose, grad_kind, b, g.N, o, v);
#pragma unroll
    for (int a = 0; a < D; ++a) x_b[(size_t)g.iperm[o] * D + a] -= eps * v[a];
  }
  if (threadIdx.x == 0) sh_fail = 0;
  __syncthreads();
  factor_phase<D, NT>(g, L, sm.stage, 1e-13 * sh_max, &sh_fail, sm.mbar, sm.phase, sm.xinv, x_b, sm.pp);
  __syncthreads();
  const bool ok = sh_fail == 0;
  if (ok) {
    solve_phase<D, NT>(g, L, sm.stage, x_b, sm.mbar, sm.phase, sm.pp, false);
    retract_phase<D, NT>(g, Tb, Tdir, x_b, 1.0);
  }
  __syncthreads();
  double* rg_b = ws.rgrad + (size_t)b * slots;
  for (int slot = threadIdx.x; slot < (int)slots; slot += NT) {
    double gw = 0.0, gr = 0.0;
    if (ok) {
      double c0[D], c1[D];
      eval_slot<D>(g, pr, Tb, b, slot, c0, nullptr, nullptr, false);
      eval_slot<D>(g, pr, Tdir, b, slot, c1, nullptr, nullptr, false);
      double n0 = 0.0, n1 = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        n0 = fma(c0[a], c0[a], n0);
        n1 = fma(c1[a], c1[a], n1);
      }
      const double w = slot_weight<D>(g, pr, b, slot);
      double p0, p1;   // dS/dw = psi w ||c||^2 (psi = 1 for quadratic costs)
      slot_cost(g, pr, b, slot, w * w * n0, p0);
      slot_cost(g, pr, b, slot, w * w * n1, p1);
      gw = w * (p0 * n0 - p1 * n1) / eps;
      if (pr.radius != nullptr && slot < g.E) {   // dS/dk = k (1 - psi) - (s/k) psi
        const double k = pr.radius[(size_t)b * pr.r_bstride];
        const double s0 = w * w * n0, s1 = w * w * n1;
        const double d0 = -k * expm1(-s0 / (k * k)) - s0 / k * p0, d1 = -k * expm1(-s1 / (k * k)) - s1 / k * p1;
        gr = (d0 - d1) / eps;
      }
    }
    cost_b[slot] = gw;
    rg_b[slot] = gr;
  }
}

// ---------------------------------------------------------------------------- unroll / truncated backward
// Retraction adjoint of theta_{k+1} = theta_k Exp(-alpha delta) for one pose (oracle/unroll.py):
//   u = -alpha Jr(-alpha delta)^T v  (dL/d delta),   v <- Ad(Exp(alpha delta))^T v  (direct part).
__device__ __forceinline__ void retract_adjoint(const double* dl, double alpha, double* v, double* u, dev::SE3*) {
  using namespace dev;
  double x[6], y[6];
#pragma unroll
  for (int a = 0; a < 6; ++a) x[a] = -alpha * dl[a];
  // Jr(x) = [[Jr(w), Q], [0, Jr(w)]] = inverse of Jr^-1(x) = [[Ji, U], [0, Ji]]:  Jr(w) = Ji^-1, Q = -Jr(w) U Jr(w)
  M3 Ji, U;
  se3_jr_inv(x, Ji, U);
  const double th = sqrt(x[3] * x[3] + x[4] * x[4] + x[5] * x[5]);
  const Coef k = coefs(th);
  const M3 Jw = poly_hat(1.0, -k.B, k.C, x + 3);   // Jr(w) = Jl(-w) = I - B W + C W^2
  const M3 Q0 = mul(mul(Jw, U), Jw);
  // Jr^T v = (Jw^T v_r, -Q0^T v_r + Jw^T v_w)
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    y[a] = Jw.m[0][a] * v[0] + Jw.m[1][a] * v[1] + Jw.m[2][a] * v[2];
    y[3 + a] = -(Q0.m[0][a] * v[0] + Q0.m[1][a] * v[1] + Q0.m[2][a] * v[2]) +
               Jw.m[0][a] * v[3] + Jw.m[1][a] * v[4] + Jw.m[2][a] * v[5];
  }
#pragma unroll
  for (int a = 0; a < 6; ++a) u[a] = -alpha * y[a];
  // Ad(T)^T v with T = Exp(alpha delta) = [R | t]:  (R^T v_r, -R^T (t x v_r) + R^T v_w)
#pragma unroll
  for (int a = 0; a < 6; ++a) x[a] = alpha * dl[a];
  const SE3 T = se3_exp(x);
  const double tx[3] = {T.t[1] * v[2] - T.t[2] * v[1], T.t[2] * v[0] - T.t[0] * v[2], T.t[0] * v[1] - T.t[1] * v[0]};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    y[a] = T.R[0][a] * v[0] + T.R[1][a] * v[1] + T.R[2][a] * v[2];
    y[3 + a] = -(T.R[0][a] * tx[0] + T.R[1][a] * tx[1] + T.R[2][a] * tx[2]) +
               T.R[0][a] * v[3] + T.R[1][a] * v[4] + T.R[2][a] * v[5];
  }
#pragma unroll
  for (int a = 0; a < 6; ++a) v[a] = y[a];
}
__device__ __forceinline__ void retract_adjoint(const double* dl, double alpha, double* v, double* u, dev::SE2*) {
  using namespace dev;
  // Jr(x) = [[A, wB, wC r1 - B r2], [-wB, A, B r1 + wC r2], [0, 0, 1]] at x = -alpha delta
  const double r1 = -alpha * dl[0], r2 = -alpha * dl[1], w = -alpha * dl[2];
  const Coef k = coefs(fabs(w));
  const double a = k.A, bb = w * k.B, v0 = w * k.C * r1 - k.B * r2, v1 = k.B * r1 + w * k.C * r2;
  u[0] = -alpha * (a * v[0] - bb * v[1]);
  u[1] = -alpha * (bb * v[0] + a * v[1]);
  u[2] = -alpha * (v0 * v[0] + v1 * v[1] + v[2]);
  // Ad(T)^T v, T = Exp(alpha delta) = [R | t], Ad = [[R, (t_y, -t_x)^T], [0, 1]]
  double x[3] = {alpha * dl[0], alpha * dl[1], alpha * dl[2]};
  const SE2 T = se2_exp(x);
  const double y0 = T.R[0][0] * v[0] + T.R[1][0] * v[1], y1 = T.R[0][1] * v[0] + T.R[1][1] * v[1];
  const double y2 = T.t[1] * v[0] - T.t[0] * v[1] + v[2];
  v[0] = y0;
  v[1] = y1;
  v[2] = y2;
}
__device__ __forceinline__ dev::SE3 pose_retract(const dev::SE3& T, const double* e) { return dev::se3_mul(T, dev::se3_exp(e)); }
__device__ __forceinline__ dev::SE2 pose_retract(const dev::SE2& T, const double* e) { return dev::se2_mul(T, dev::se2_exp(e)); }

// (C(theta) lam).p - (C(theta) del).q of one cost term at the given poses (reading U1's contraction)
template <int D, class PT>
__device__ __forceinline__ double jac_contract(bool edge, const PT& Ti, const PT& Tj, const PT& Z, const double* li,
                                               const double* lj, const double* di, const double* dj, const double* p,
                                               const double* q) {
  double c[D], Ci[D * D], Cj[D * D];
  if (edge) edge_eval(Ti, Tj, Z, c, Ci, Cj, true);
  else prior_eval(Ti, Z, c, Ci, true);
  double v = 0.0;
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double cl = 0.0, cd = 0.0;
#pragma unroll
    for (int t = 0; t < D; ++t) {
      cl = fma(Ci[r * D + t], li[t], cl);
      cd = fma(Ci[r * D + t], di[t], cd);
      if (edge) {
        cl = fma(Cj[r * D + t], lj[t], cl);
        cd = fma(Cj[r * D + t], dj[t], cd);
      }
    }
    v += cl * p[r] - cd * q[r];
  }
  return v;
}

constexpr double UNROLL_FD_STEP = 1e-5;   // reading U1 (oracle/unroll.py FD_STEP)

// Unroll / Truncated backward, one CTA per element (oracle/unroll.py, dnls.h dnls_backward_unroll):
// reverse the recorded GN iterations k = it-1 .. it-Tw.  v (original pose order) lives in ws.bsave, the
// per-slot weight gradients accumulate in ws.cost, the per-slot pose-gradient contributions go to the slot
// scratch and are gathered per pose in the fixed order of the symbolic list bc (deterministic).
template <int D>
__global__ void __launch_bounds__(NT, MINB) k_backward_unroll(DevGraph g, DevProb pr, DevWs ws, const double* gpose,
                                                            int grad_kind, int Tw, double alpha, double* gpose0) {
  constexpr int PS = GT<D>::PS, JS = GT<D>::JS;
  using PT = typename PoseT<D>::T;
  const int b = blockIdx.x;
  const size_t slots = (size_t)g.E + g.P;
  Smem sm = smem_views(g, ws.x + (size_t)b * g.n);
  double* x_b = sm.x;
  double* v = ws.bsave + (size_t)b * g.n;
  double* gw = ws.cost + (size_t)b * slots;
  double* pg = ws.jac + (size_t)b * slots * JS;
  const double* TK = pr.poses + (size_t)b * g.N * PS;
  const int iters = ws.it[b];
  for (int o = threadIdx.x; o < g.N; o += NT) {
    double vv[D];
    tangent_grad<D>(TK, gpose, grad_kind, b, g.N, o, vv);
#pragma unroll
    for (int a = 0; a < D; ++a) v[(size_t)o * D + a] = vv[a];
  }
  for (int sl = threadIdx.x; sl < (int)slots; sl += NT) gw[sl] = 0.0;
  __syncthreads();
  const int kend = max(0, iters - Tw);
  for (int k = iters - 1; k >= kend; --k) {
    const size_t hs = (size_t)b * ws.keep + (k % ws.keep);
    const double* Tk = ws.hT + hs * g.N * PS;
    const double* dk = ws.hd + hs * g.n;
    double* Lk = ws.hL + hs * g.storage;
    // (a) retraction adjoint: rhs u (permuted order) and the direct part of v
    for (int o = threadIdx.x; o < g.N; o += NT) {
      const int pp = g.iperm[o];
      double u[D];
      retract_adjoint(dk + (size_t)D * pp, alpha, v + (size_t)o * D, u, (PT*)nullptr);
#pragma unroll
      for (int a = 0; a < D; ++a) x_b[(size_t)D * pp + a] = u[a];
    }
    // (b) lambda = H_k^-1 u on the iteration's cached factor
    bulk_load<NT>(sm.res, Lk + g.res_lo, g.storage - g.res_lo, sm.mbar, sm.phase);
    solve_phase<D, NT>(g, full_view(g, Lk, sm), sm.stage, x_b, sm.mbar, sm.phase, sm.pp);
    __syncthreads();
    // (c) per cost term: weight gradient and the pose-gradient contributions
    for (int slot = threadIdx.x; slot < (int)slots; slot += NT) {
      const bool edge = slot < g.E;
      const int vi = edge ? g.edges[2 * slot] : g.prior_vars[slot - g.E];
      const int vj = edge ? g.edges[2 * slot + 1] : vi;
      const double* li = x_b + (size_t)D * g.iperm[vi];
      const double* lj = x_b + (size_t)D * g.iperm[vj];
      const double* di = dk + (size_t)D * g.iperm[vi];
      const double* dj = dk + (size_t)D * g.iperm[vj];
      double c[D], Ci[D * D], Cj[D * D];
      eval_slot<D>(g, pr, Tk, b, slot, c, Ci, Cj, true);
      const double w = slot_weight<D>(g, pr, b, slot);
      double q[D], p[D], qc = 0.0, qd = 0.0;
#pragma unroll
      for (int r = 0; r < D; ++r) {
        double cl = 0.0, cd = 0.0;
#pragma unroll
        for (int t = 0; t < D; ++t) {
          cl = fma(Ci[r * D + t], li[t], cl);
          cd = fma(Ci[r * D + t], di[t], cd);
          if (edge) {
            cl = fma(Cj[r * D + t], lj[t], cl);
            cd = fma(Cj[r * D + t], dj[t], cd);
          }
        }
        q[r] = cl;
        p[r] = c[r] - cd;
        qc = fma(cl, c[r], qc);
        qd = fma(cl, cd, qd);
      }
      gw[slot] += 2.0 * w * (qc - qd);
      // w^2 [C_s^T q + grad_eta contraction] for each endpoint s
      const PT Ti = PoseT<D>::load(Tk + (size_t)vi * PS);
      const PT Tj = PoseT<D>::load(Tk + (size_t)vj * PS);
      const PT Z = edge ? PoseT<D>::load(pr.meas + ((size_t)b * g.E + slot) * PS)
                        : PoseT<D>::load(pr.prior_meas + (size_t)b * pr.pm_bstride + (size_t)(slot - g.E) * PS);
      for (int side = 0; side < (edge ? 2 : 1); ++side) {
        const double* Cs = side == 0 ? Ci : Cj;
        double gr[D];
#pragma unroll
        for (int t = 0; t < D; ++t) {
          double a = 0.0;
#pragma unroll
          for (int r = 0; r < D; ++r) a = fma(Cs[r * D + t], q[r], a);
          gr[t] = a;
        }
        for (int t = 0; t < D; ++t) {
          double e[D];
#pragma unroll
          for (int a = 0; a < D; ++a) e[a] = a == t ? UNROLL_FD_STEP : 0.0;
          const PT Tp = pose_retract(side == 0 ? Ti : Tj, e);
#pragma unroll
          for (int a = 0; a < D; ++a) e[a] = -e[a];
          const PT Tm = pose_retract(side == 0 ? Ti : Tj, e);
          const double fp_ = side == 0 ? jac_contract<D>(edge, Tp, Tj, Z, li, lj, di, dj, p, q)
                                       : jac_contract<D>(edge, Ti, Tp, Z, li, lj, di, dj, p, q);
          const double fm_ = side == 0 ? jac_contract<D>(edge, Tm, Tj, Z, li, lj, di, dj, p, q)
                                       : jac_contract<D>(edge, Ti, Tm, Z, li, lj, di, dj, p, q);
          gr[t] += (fp_ - fm_) / (2.0 * UNROLL_FD_STEP);
        }
        double* o = pg + (size_t)slot * JS + side * 8;
#pragma unroll
        for (int t = 0; t < D; ++t) o[t] = w * w * gr[t];
      }
    }
    __syncthreads();
    // (d) v_o += sum of its slots' contributions (fixed order of bc)
    for (int pp = threadIdx.x; pp < g.N; pp += NT) {
      double acc[D];
      const int o = g.perm[pp];
#pragma unroll
      for (int a = 0; a < D; ++a) acc[a] = v[(size_t)o * D + a];
      for (int cidx = g.bc_ptr[pp]; cidx < g.bc_ptr[pp + 1]; ++cidx) {
        const int code = g.bc[cidx];
        const double* src = pg + (size_t)(code >> 1) * JS + (code & 1) * 8;
#pragma unroll
        for (int a = 0; a < D; ++a) acc[a] += src[a];
      }
#pragma unroll
      for (int a = 0; a < D; ++a) v[(size_t)o * D + a] = acc[a];
    }
    __syncthreads();
  }
  if (gpose0)
    for (int i = threadIdx.x; i < g.n; i += NT) gpose0[(size_t)b * g.n + i] = kend == 0 ? v[i] : 0.0;
}

// radius gradient: per element the fixed-order sum over edge slots, then, for a shared radius
// (radius_bstride == 0), over the batch in order; per-element radii get per-element gradients; one warp
__global__ void k_reduce_radius(int B, int E, int slots, const double* src, double* out, long long bstride) {
  const int lane = threadIdx.x;
  double tot = 0.0;
  for (int b = 0; b < B; ++b) {
    double s = 0.0;
    for (int e = lane; e < E; e += 32) s += src[(size_t)b * slots + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (bstride > 0) {
      if (lane == 0) out[b] = s;
    } else {
      tot += s;
    }
  }
  if (bstride == 0 && lane == 0) out[0] = tot;
}

// fixed-order batch reduction (or per-element copy) of the per-slot weight gradients
__global__ void k_reduce_wgrad(int B, int E, int P, const double* src, double* ge, double* gp,
                               long long bstride) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  const int slots = E + P;
  if (slot >= slots) return;
  double* dst = slot < E ? ge : gp;
  const int idx = slot < E ? slot : slot - E;
  if (!dst) return;
  if (bstride == 0) {
    double s = 0.0;
    for (int b = 0; b < B; ++b) s += src[(size_t)b * slots + slot];
    dst[idx] = s;
  } else {
    for (int b = 0; b < B; ++b) dst[(size_t)b * bstride + idx] = src[(size_t)b * slots + slot];
  }
}

template <int D>
__global__ void k_export_factor(DevGraph g, DevWs ws, double* dense) {
  const int b = blockIdx.x;
  const size_t n = g.n;
  double* Db = dense + (size_t)b * n * n;
  const double* Lb = ws.L + (size_t)b * g.storage;
  for (size_t i = threadIdx.x; i < n * n; i += NT) Db[i] = 0.0;
  __syncthreads();
  // iterate storage panels: (row, col) scalar within panel -> permuted global indices
  for (int s = 0; s < g.S; ++s) {
    const int f = g.sn_first[s], w = g.sn_w[s], m = g.sn_m[s], ld = g.sn_ld[s], off = g.sn_off[s];
    const int rb = g.snr_ptr[s];
    for (int it = threadIdx.x; it < m * w; it += NT) {
      const int c = it / m, r = it - c * m;
      int gr;
      if (r < w) {
        if (r < c) continue;
        gr = D * f + r;
      } else {
        const int rr = (r - w) / D, a = (r - w) % D;
        gr = D * g.snr[rb + rr] + a;
      }
      Db[(size_t)gr * n + (size_t)D * f + c] = Lb[off + (size_t)c * ld + r];
    }
  }
}

template <int D>
__global__ void k_import_matrix(DevGraph g, DevWs ws, const double* dense) {
  const int b = blockIdx.x;
  const size_t n = g.n;
  const double* Db = dense + (size_t)b * n * n;
  double* Lb = ws.L + (size_t)b * g.storage;
  __shared__ double s_red[NT / 32];
  double mymax = 0.0;
  for (int s = 0; s < g.S; ++s) {
    const int f = g.sn_first[s], w = g.sn_w[s], m = g.sn_m[s], ld = g.sn_ld[s], off = g.sn_off[s];
    const int rb = g.snr_ptr[s];
    for (int it = threadIdx.x; it < m * w; it += NT) {
      const int c = it / m, r = it - c * m;
      double v = 0.0;
      const int pc = f + c / D, ac = c % D;
      if (r >= c) {
        int pr_, ar;
        if (r < w) {
          pr_ = f + r / D;
          ar = r % D;
        } else {
          pr_ = g.snr[rb + (r - w) / D];
          ar = (r - w) % D;
        }
        v = Db[((size_t)g.perm[pr_] * D + ar) * n + (size_t)g.perm[pc] * D + ac];
        if (r == c) mymax = fmax(mymax, v);
      }
      Lb[off + (size_t)c * ld + r] = v;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mymax = fmax(mymax, __shfl_xor_sync(0xffffffffu, mymax, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = mymax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < NT / 32; ++i) m = fmax(m, s_red[i]);
    ws.maxd[b] = m;
  }
}

template <int D>
__global__ void k_export_rhs(DevGraph g, DevWs ws, double* out) {
  const int b = blockIdx.x;
  const double* x_b = ws.x + (size_t)b * g.n;
  for (int i = threadIdx.x; i < g.n; i += NT) {
    const int o = i / D, a = i - o * D;
    out[(size_t)b * g.n + i] = x_b[(size_t)g.iperm[o] * D + a];
  }
}

#include "bl.cuh"
void bl_plan_delete(BLPlan* p) { delete p; }
#endif  // !DNLS_CLUSTER_TU
}  // namespace

// ============================================================================= C ABI
#ifdef DNLS_CLUSTER_TU
namespace dnls {
cudaError_t launch_forward_cluster(int CL, int D, const DevGraph& g, DevProb pr, DevWs ws, FwdParams fp, int batch,
                                   cudaStream_t s) {
  const size_t smem = smem_bytes_grouped(g);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * CL));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#define DNLS_LAUNCH_CL(DD, CC)                                                                         \
  {                                                                                                  \
    cudaError_t e = cudaFuncSetAttribute(k_forward<DD, CC>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         (int)smem);                                                 \
    if (e != cudaSuccess) return e;                                                                  \
    g_launches.fetch_add(1, std::memory_order_relaxed);                                              \
    return cudaLaunchKernelEx(&cfg, k_forward<DD, CC>, g, pr, ws, fp);                               \
  }
  if (D == 6 && CL == 2) DNLS_LAUNCH_CL(6, 2)
  if (D == 6 && CL == 4) DNLS_LAUNCH_CL(6, 4)
  if (D == 6 && CL == 8) DNLS_LAUNCH_CL(6, 8)
  if (D == 3 && CL == 2) DNLS_LAUNCH_CL(3, 2)
  if (D == 3 && CL == 4) DNLS_LAUNCH_CL(3, 4)
  if (D == 3 && CL == 8) DNLS_LAUNCH_CL(3, 8)
#undef DNLS_LAUNCH_CL
  return cudaErrorInvalidValue;
}
}  // namespace dnls
#else  // the main translation unit: host API

namespace dnls {
std::atomic<long long> g_launches{0};
}

namespace {
// batch-interleaved level-major path (bl.cuh): Gauss-Newton with the
// implicit (or no) backward and quadratic costs; chosen explicitly (batch_interleave == 32) or automatically
bool bl_supported(const dnls_options* opt, const dnls_problem* prob) {
  return opt->optimizer == DNLS_GN &&
         (opt->backward_mode == DNLS_BWD_NONE || opt->backward_mode == DNLS_BWD_IMPLICIT) &&
         (prob == nullptr || prob->radius == nullptr);
}
bool bl_choose(const dnls_graph* g, int batch, const dnls_options* opt, const dnls_problem* prob) {
  if (!opt || opt->batch_interleave == 1 || !bl_supported(opt, prob)) return false;
  if (opt->batch_interleave == 32) return true;
  // automatic: many problems per GPU (measured crossover); below it one CTA
  // per element (k_forward) keeps each problem's factor on chip
  // (profiles/r3q: C4 graph, 1024 poses: B = 256 132k vs 112k problem-iter/s, B = 128 73k vs 112k; C2 graph, 256
  // poses: B = 256 317k vs 555k, B = 512 568k vs 550k): batch >= 256 and batch x poses >= 256 x 1024
  static const int min_batch = std::getenv("DNLS_BL_MIN_BATCH") ? std::atoi(std::getenv("DNLS_BL_MIN_BATCH")) : 256;
  return batch >= min_batch && (long long)batch * g->sym.N >= 262144LL;
}
size_t bl_ws_bytes(const dnls_graph* g, int batch) {
  const Symbolic& s = g->sym;
  return bl_layout_sizes(s.D, s.N, s.E, s.P, s.nnz_L_blocks, batch).total;
}
dnls_status bl_plan_for(dnls_graph* g, BLPlan** out) {
  std::lock_guard<std::mutex> lk(g->bl_mu);
  if (!g->bl) {
    BLPlan* pl = new BLPlan();
    DeviceGuard dguard(g->device);
    const std::string e = bl_build(g->sym, g->device, *pl);
    if (!e.empty()) {
      delete pl;
      return fail(DNLS_E_CUDA, e);
    }
    g->bl = pl;
  }
  *out = g->bl;
  return DNLS_OK;
}
// CTAs per batch element for dnls_forward: a cluster when the
// batch leaves most SMs idle and the graph has enough work per level to share
int forward_cluster(const dnls_graph* g, int batch, int req) {
  if (req == 1 || req == 2 || req == 4 || req == 8) return req;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // measured on C3 (4096 poses, B = 16; profiles/r2u_c3_cl*.json): 1 CTA 2.40k, 2 CTAs 2.67k, 4 CTAs 2.99k,
  // 8 CTAs 1.60k problem-iter/s -- beyond 4 the cluster barriers and the all-global working set outweigh the
  // wider levels
  if (g->sym.N < 1024) return 1;
  if (batch * 4 <= sms) return 4;
  if (batch * 2 <= sms) return 2;
  return 1;
}
}  // namespace

extern "C" {

DNLS_API const char* dnls_version_string(void) {
  return "libdnls 1 (sm_100a, fp64; one CTA per batch element; supernodal Cholesky)";
}

DNLS_API const char* dnls_last_error(void) { return g_err.c_str(); }

DNLS_API dnls_status dnls_debug_trace(int64_t* out, int32_t capacity, int32_t* count) {
#ifdef DNLS_TRACE
  if (!out || !count) return fail(DNLS_E_INVALID, "dnls_debug_trace: NULL argument");
  int n = 0;
  cudaMemcpyFromSymbol(&n, g_trace_n, sizeof(int));
  n = std::min(n, (int)capacity);
  if (n > 0) cudaMemcpyFromSymbol(out, g_trace, sizeof(long long) * 2 * n);
  *count = n;
  int zero = 0;
  cudaMemcpyToSymbol(g_trace_n, &zero, sizeof(int));
  return cuda_check("dnls_debug_trace");
#else
  (void)out;
  (void)capacity;
  if (count) *count = 0;
  return fail(DNLS_E_UNSUPPORTED, "dnls_debug_trace: library built without -DDNLS_TRACE");
#endif
}

DNLS_API dnls_status dnls_debug_launch_count(int64_t* count, int32_t reset) {
  if (!count) return fail(DNLS_E_INVALID, "dnls_debug_launch_count: NULL argument");
  *count = reset ? (int64_t)dnls::g_launches.exchange(0) : (int64_t)dnls::g_launches.load();
  return DNLS_OK;
}

DNLS_API dnls_status dnls_debug_phase_times(const dnls_graph* g, double* ms, int32_t capacity, int32_t* count) {
  if (!g || !count) return fail(DNLS_E_INVALID, "dnls_debug_phase_times: NULL argument");
  dnls_graph* gm = const_cast<dnls_graph*>(g);
  std::lock_guard<std::mutex> lk(gm->bl_mu);
  int n = 0;
  for (auto& e : gm->phase_ev) {
    float t = 0.f;
    if (cudaEventSynchronize(e.second) == cudaSuccess && cudaEventElapsedTime(&t, e.first, e.second) == cudaSuccess &&
        ms && n < capacity)
      ms[n] = t;
    ++n;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  gm->phase_ev.clear();
  *count = std::min(n, (int)capacity);
  return cuda_check("dnls_debug_phase_times");
}

#ifdef DNLS_LIN_PROBE
DNLS_API int dnls_debug_probe(unsigned long long* out8, int reset) {
  if (cudaMemcpyFromSymbol(out8, g_probe, sizeof(unsigned long long) * 8) != cudaSuccess) return 7;
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_probe, z, sizeof(z));
  }
  return 0;
}
#endif

DNLS_API void dnls_options_default(dnls_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->optimizer = DNLS_GN;
  o->max_iterations = 10;
  o->step_size = 1.0;
  o->lambda0 = 1e-3;
  o->lambda_min = 1e-8;
  o->lambda_max = 1e5;
  o->lambda_down = 3.0;
  o->lambda_up = 2.0;
  o->damping = DNLS_DAMP_MARQUARDT;
  o->early_stop = 0;
  o->abs_tol = 1e-10;
  o->rel_tol = 1e-8;
  o->backward_mode = DNLS_BWD_NONE;
  o->trust_radius0 = 1.0;
  o->trust_radius_max = 1e4;
  o->trust_radius_min = 1e-10;
}

DNLS_API dnls_status dnls_graph_create(int32_t group, int32_t num_vars, int32_t num_edges,
                                       const int32_t* edges_ij, int32_t num_priors,
                                       const int32_t* prior_vars, int32_t device, dnls_graph** out) {
  if (!out) return fail(DNLS_E_INVALID, "dnls_graph_create: out is NULL");
  *out = nullptr;
  dnls_graph* g = new dnls_graph();
  int code = 0;
  SymbolicOptions sopt;
  int64_t smem_total = 0;
  {
    // shared-memory plan: x (n doubles) in shared memory when it fits in 64 KB, the rest of
    // SMEM_BYTES holds the resident top levels + the staging buffer of the lower levels
    const int64_t n = (int64_t)num_vars * group;
    const int64_t xb = (n * 8 <= 65536) ? ((n + 1) & ~int64_t(1)) * 8 : 0;
    int64_t smem = SMEM_BYTES;
    if (const char* env = std::getenv("DNLS_SMEM_KB")) smem = std::min<int64_t>(SMEM_BYTES, std::atoll(env) * 1024);
    sopt.smem_cap_doubles = std::max<int64_t>(0, smem - xb - 2 * 4 * (int64_t)sopt.packet_ints) / 8;   // packets
    sopt.cta_threads = NT;
    smem_total = smem - xb;
  }
  if (const char* env = std::getenv("DNLS_RELAX")) {   // tuning override: "a,sc,sf,mc,mf,max,bf"
    std::sscanf(env, "%d,%d,%lf,%d,%lf,%d,%lf", &sopt.relax_always_cols, &sopt.relax_small_cols,
                &sopt.relax_small_frac, &sopt.relax_mid_cols, &sopt.relax_mid_frac, &sopt.relax_max_cols,
                &sopt.relax_big_frac);
  }
  std::string msg = analyze(group, num_vars, num_edges, edges_ij, num_priors, prior_vars, sopt, g->sym, &code);
  if (msg.empty() && g->sym.pk_max != sopt.packet_ints) {   // re-plan the residency for the actual packets
    sopt.smem_cap_doubles = std::max<int64_t>(0, smem_total - 8 * (int64_t)g->sym.pk_max - 64) / 8;
    msg = analyze(group, num_vars, num_edges, edges_ij, num_priors, prior_vars, sopt, g->sym, &code);
  }
  if (!msg.empty()) {
    delete g;
    return fail((dnls_status)code, msg);
  }
  const Symbolic& s = g->sym;
  // pack all int32 arrays into one device buffer
  std::vector<int32_t> buf;
  std::vector<size_t> offs;
  auto add = [&](const std::vector<int32_t>& v) {
    while (buf.size() % 4) buf.push_back(0);   // 16-byte aligned arrays (int4 loads)
    offs.push_back(buf.size());
    buf.insert(buf.end(), v.begin(), v.end());
    buf.push_back(0);   // never empty
  };
  std::vector<int32_t> sn_off32(s.sn_off.begin(), s.sn_off.end());
  add(s.perm); add(s.iperm); add(s.edges); add(s.prior_vars);
  add(s.sn_first); add(s.sn_m); add(s.sn_ld); add(s.sn_w); add(sn_off32);
  add(s.level_off); add(s.level_stage_hi);
  add(s.pk); add(s.pk_off);
  add(s.slot_desc); add(s.col_sn);
  add(s.snr_ptr); add(s.snr);
  add(s.blk_off); add(s.blk_ld); add(s.blk_cptr); add(s.blk_con);
  add(s.bc_ptr); add(s.bc);
  add(s.dup_blk);
  if (std::getenv("DNLS_VERBOSE")) {
    int64_t maxlev = 0;
    for (int l = 0; l < s.num_levels; ++l) maxlev = std::max<int64_t>(maxlev, s.level_off[l + 1] - s.level_off[l]);
    std::fprintf(stderr,
                 "[dnls] N=%d levels=%d storage=%lld res_lo=%d res_n=%lld stage_cap=%lld max_level=%lld "
                 "max_stage=%lld pk_max=%d ints packets=%d\n",
                 s.N, s.num_levels, (long long)s.storage, s.res_lo, (long long)s.res_n, (long long)s.stage_cap,
                 (long long)maxlev, (long long)s.max_level_stage, s.pk_max, s.npk);
    if (std::atoi(std::getenv("DNLS_VERBOSE")) > 1)
      for (int k = 0; k < s.npk; ++k) {
        const int32_t* h = s.pk.data() + s.pk_off[k];
        const int lv = h[9];
        std::fprintf(stderr, "  packet %d level %d res %d: tasks %d cons %d rows %d fcons %d sn %d ulanes %d flanes %d maxb %d\n",
                     k, lv, s.level_off[lv] >= s.res_lo ? 1 : 0, h[0], h[1], h[2], h[3], h[4], h[6], h[7], h[8]);
      }
  }
  g->device = device;
  while (buf.size() % 4) buf.push_back(0);
  g->dbuf_bytes = buf.size() * sizeof(int32_t);
  if (device < 0) {   // host-only symbolic analysis (no device arrays; compute calls refuse it)
    *out = g;
    return DNLS_OK;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    delete g;
    return fail(DNLS_E_CUDA, "dnls_graph_create: cudaSetDevice(" + std::to_string(device) + ") failed");
  }
  g->device = device;
  if (cudaMalloc(&g->dbuf, buf.size() * sizeof(int32_t)) != cudaSuccess ||
      cudaMemcpy(g->dbuf, buf.data(), buf.size() * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
    std::string e = cudaGetErrorString(cudaGetLastError());
    if (g->dbuf) cudaFree(g->dbuf);
    cudaSetDevice(prev);
    delete g;
    return fail(DNLS_E_CUDA, "dnls_graph_create: device upload failed: " + e);
  }
  cudaSetDevice(prev);
  const int* d = g->dbuf;
  int k = 0;
  DevGraph& dg = g->dg;
  dg.D = s.D; dg.N = s.N; dg.E = s.E; dg.P = s.P; dg.S = s.S;
  dg.storage = (int)s.storage; dg.n = s.N * s.D;
  dg.res_lo = s.res_lo;
  dg.res_n = (int)((s.res_n + 1) & ~int64_t(1));
  dg.x_smem = (int64_t)dg.n * 8 <= 65536 ? 1 : 0;
  dg.n_pad = (dg.n + 1) & ~1;
  dg.stage_n = (int)((s.max_level_stage + 1) & ~int64_t(1));
  dg.stage_n = std::max<int>(dg.stage_n, (int)(((s.stage_cap > 0 ? s.stage_cap : 0)) & ~int64_t(1)));
  dg.perm = d + offs[k++]; dg.iperm = d + offs[k++]; dg.edges = d + offs[k++]; dg.prior_vars = d + offs[k++];
  dg.sn_first = d + offs[k++]; dg.sn_m = d + offs[k++]; dg.sn_ld = d + offs[k++]; dg.sn_w = d + offs[k++];
  dg.sn_off = d + offs[k++];
  dg.level_off = d + offs[k++]; dg.level_stage_hi = d + offs[k++];
  dg.pk = d + offs[k++];
  dg.pk_off = d + offs[k++];
  dg.pk_max = s.pk_max;
  dg.npk = s.npk;
  dg.slot_desc = reinterpret_cast<const int4*>(d + offs[k++]);
  dg.pose_sn = d + offs[k++];
  dg.snr_ptr = d + offs[k++]; dg.snr = d + offs[k++];
  dg.blk_off = d + offs[k++]; dg.blk_ld = d + offs[k++]; dg.blk_cptr = d + offs[k++]; dg.blk_con = d + offs[k++];
  dg.bc_ptr = d + offs[k++]; dg.bc = d + offs[k++];
  dg.dup_blk = d + offs[k++];
  dg.ndup = (int)s.dup_blk.size();
  *out = g;
  return DNLS_OK;
}

DNLS_API void dnls_graph_destroy(dnls_graph* g) {
  if (!g) return;
  if (g->bl) bl_plan_delete(g->bl);
  if (g->dbuf) cudaFree(g->dbuf);
  delete g;
}

DNLS_API dnls_status dnls_graph_stats(const dnls_graph* g, dnls_stats* o) {
  if (!g || !o) return fail(DNLS_E_INVALID, "dnls_graph_stats: NULL argument");
  const Symbolic& s = g->sym;
  std::memset(o, 0, sizeof(*o));
  o->group = s.D;
  o->num_vars = s.N;
  o->num_edges = s.E;
  o->num_priors = s.P;
  o->num_supernodes = s.S;
  o->num_levels = s.num_levels;
  o->etree_height = s.etree_height;
  o->max_supernode_cols = s.max_sn_cols_sc;
  o->max_panel_rows = s.max_panel_rows;
  o->nnz_H_blocks = s.nnz_H_blocks;
  o->nnz_L_blocks = s.nnz_L_blocks;
  o->nnz_L = s.nnz_L;
  o->storage_doubles = s.storage;
  o->factor_flops = s.factor_flops;
  o->solve_flops = 4.0 * (double)s.nnz_L;
  const double pose_b = s.D == 6 ? 96.0 : 48.0;
  const double nvec = 8.0 * s.N * s.D;
  o->bytes_linearize = pose_b * (s.N + s.E + s.P) + 8.0 * s.nnz_L + nvec;
  o->bytes_factor = 16.0 * s.nnz_L;
  o->bytes_solve = 16.0 * s.nnz_L + 2.0 * nvec;
  o->bytes_update = 2.0 * pose_b * s.N + nvec;
  o->bytes_backward = 16.0 * s.nnz_L + pose_b * (s.N + s.E + s.P) + 2.0 * nvec;
  o->index_bytes = (int64_t)g->dbuf_bytes;
  o->smem_bytes = g->dbuf ? (int64_t)smem_bytes(g->dg) : 0;
  o->resident_doubles = (int64_t)(s.storage - s.res_lo);
  return DNLS_OK;
}

DNLS_API dnls_status dnls_block_offsets(const dnls_graph* g, int32_t* edge_desc, int32_t* prior_desc) {
  if (!g) return fail(DNLS_E_INVALID, "dnls_block_offsets: graph is NULL");
  const Symbolic& s = g->sym;
  for (int sl = 0; sl < s.E + s.P; ++sl) {
    const int32_t* d = &s.slot_desc[12 * (size_t)sl];
    if (sl < s.E) {
      if (!edge_desc) continue;
      int32_t* o = edge_desc + 7 * (size_t)sl;
      o[0] = d[0]; o[1] = d[4]; o[2] = d[1]; o[3] = d[5]; o[4] = d[2]; o[5] = d[6]; o[6] = d[3];
    } else if (prior_desc) {
      int32_t* o = prior_desc + 2 * (size_t)(sl - s.E);
      o[0] = d[0]; o[1] = d[4];
    }
  }
  return DNLS_OK;
}

DNLS_API dnls_status dnls_status_summary(const int32_t* status, int32_t batch, int32_t* n_failed, int32_t* n_warned,
                                         void* stream) {
  if (batch < 0 || (batch > 0 && !status)) return fail(DNLS_E_INVALID, "dnls_status_summary: bad arguments");
  std::vector<int32_t> h((size_t)batch);
  if (batch > 0) {
    if (cudaMemcpyAsync(h.data(), status, sizeof(int32_t) * batch, cudaMemcpyDeviceToHost, (cudaStream_t)stream) !=
            cudaSuccess ||
        cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
      return fail(DNLS_E_CUDA, std::string("dnls_status_summary: ") + cudaGetErrorString(cudaGetLastError()));
  }
  int nf = 0, nw = 0;
  for (int32_t v : h) {
    const int c = v & DNLS_ST_CODE_MASK;
    nf += (c == DNLS_ST_NOT_SPD || c == DNLS_ST_SATURATED);
    nw += (v & DNLS_ST_WARN_NOT_CONVERGED) != 0;
  }
  if (n_failed) *n_failed = nf;
  if (n_warned) *n_warned = nw;
  if (batch > 0 && nf == batch)
    return fail(DNLS_E_ALL_FAILED, "dnls_status_summary: all " + std::to_string(batch) + " elements failed");
  return DNLS_OK;
}

DNLS_API dnls_status dnls_graph_perm(const dnls_graph* g, int32_t* perm) {
  if (!g || !perm) return fail(DNLS_E_INVALID, "dnls_graph_perm: NULL argument");
  std::copy(g->sym.perm.begin(), g->sym.perm.end(), perm);
  return DNLS_OK;
}

DNLS_API dnls_status dnls_graph_etree(const dnls_graph* g, int32_t* parent) {
  if (!g || !parent) return fail(DNLS_E_INVALID, "dnls_graph_etree: NULL argument");
  std::copy(g->sym.parent.begin(), g->sym.parent.end(), parent);
  return DNLS_OK;
}

DNLS_API dnls_status dnls_graph_pattern(const dnls_graph* g, int32_t* colptr, int32_t* rowidx) {
  if (!g || !colptr || !rowidx) return fail(DNLS_E_INVALID, "dnls_graph_pattern: NULL argument");
  const Symbolic& s = g->sym;
  int32_t k = 0;
  for (int c = 0; c < s.N; ++c) {
    colptr[c] = k;
    rowidx[k++] = c;
    for (int r : s.colstruct[c]) rowidx[k++] = r;
  }
  colptr[s.N] = k;
  return DNLS_OK;
}

DNLS_API dnls_status dnls_graph_supernodes(const dnls_graph* g, int32_t* first, int32_t* ncols, int32_t* level) {
  if (!g) return fail(DNLS_E_INVALID, "dnls_graph_supernodes: NULL graph");
  const Symbolic& s = g->sym;
  if (first) std::copy(s.sn_first.begin(), s.sn_first.end(), first);
  if (ncols) std::copy(s.sn_ncols.begin(), s.sn_ncols.end(), ncols);
  if (level) std::copy(s.sn_level.begin(), s.sn_level.end(), level);
  return DNLS_OK;
}

DNLS_API dnls_status dnls_workspace_bytes(const dnls_graph* g, int32_t batch, const dnls_options* opt,
                                          size_t* bytes) {
  if (!g || !bytes) return fail(DNLS_E_INVALID, "dnls_workspace_bytes: NULL argument");
  if (batch < 0) return fail(DNLS_E_SHAPE, "dnls_workspace_bytes: batch < 0");
  *bytes = ws_layout(g->sym, batch, history_keep(opt)).total;
  if (opt && opt->batch_interleave != 1 && bl_supported(opt, nullptr)) *bytes = std::max(*bytes, bl_ws_bytes(g, batch));
  return DNLS_OK;
}

namespace {
dnls_status check_common(const char* fn, const dnls_graph* g, int32_t batch, const void* ws, size_t ws_bytes,
                         int keep = 0) {
  if (!g) return fail(DNLS_E_INVALID, std::string(fn) + ": graph is NULL");
  if (!g->dbuf) return fail(DNLS_E_INVALID, std::string(fn) + ": graph was created host-only (device < 0)");
  if (batch < 0) return fail(DNLS_E_SHAPE, std::string(fn) + ": batch < 0");
  if (!ws && batch > 0) return fail(DNLS_E_INVALID, std::string(fn) + ": workspace is NULL");
  if (((uintptr_t)ws) % 256) return fail(DNLS_E_INVALID, std::string(fn) + ": workspace not 256-byte aligned");
  size_t need = ws_layout(g->sym, batch, keep).total;
  if (ws_bytes < need)
    return fail(DNLS_E_WORKSPACE, std::string(fn) + ": workspace has " + std::to_string(ws_bytes) +
                                      " bytes, needs " + std::to_string(need));
  return DNLS_OK;
}
dnls_status check_problem(const char* fn, const dnls_graph* g, const dnls_problem* p) {
  if (!p) return fail(DNLS_E_INVALID, std::string(fn) + ": problem is NULL");
  if (!p->poses) return fail(DNLS_E_INVALID, std::string(fn) + ": problem.poses is NULL");
  if (g->sym.E > 0 && (!p->meas || !p->w_edge))
    return fail(DNLS_E_INVALID, std::string(fn) + ": problem.meas / w_edge is NULL with num_edges > 0");
  if (g->sym.P > 0 && (!p->prior_meas || !p->w_prior))
    return fail(DNLS_E_INVALID, std::string(fn) + ": problem.prior_meas / w_prior is NULL with num_priors > 0");
  if (p->prior_meas_bstride < 0 || p->w_edge_bstride < 0 || p->w_prior_bstride < 0 || p->radius_bstride < 0)
    return fail(DNLS_E_INVALID, std::string(fn) + ": negative batch stride");
  return DNLS_OK;
}
#define DISPATCH_D(D_, ...)            \
  if ((D_) == 6) {                     \
    constexpr int DD = 6;              \
    __VA_ARGS__;                       \
  } else {                             \
    constexpr int DD = 3;              \
    __VA_ARGS__;                       \
  }
}  // namespace


DNLS_API dnls_status dnls_forward(const dnls_graph* g, int32_t batch, const dnls_options* opt,
                                  const dnls_problem* prob, void* workspace, size_t ws_bytes, void* stream) {
  if (!opt) return fail(DNLS_E_INVALID, "dnls_forward: options is NULL");
  const int keep = history_keep(opt);
  dnls_status st = check_common("dnls_forward", g, batch, workspace, ws_bytes, keep);
  if (st) return st;
  if ((st = check_problem("dnls_forward", g, prob))) return st;
  if (opt->optimizer != DNLS_GN && opt->optimizer != DNLS_LM && opt->optimizer != DNLS_DOGLEG)
    return fail(DNLS_E_INVALID, "dnls_forward: unknown optimizer " + std::to_string(opt->optimizer));
  if (opt->max_iterations < 0) return fail(DNLS_E_INVALID, "dnls_forward: max_iterations < 0");
  if (!(opt->step_size > 0.0 && opt->step_size <= 1.0))
    return fail(DNLS_E_INVALID, "dnls_forward: step_size must be in (0, 1]");
  if (opt->backward_mode < DNLS_BWD_NONE || opt->backward_mode > DNLS_BWD_TRUNCATED)
    return fail(DNLS_E_INVALID, "dnls_forward: unknown backward_mode " + std::to_string(opt->backward_mode));
  const bool unroll = opt->backward_mode == DNLS_BWD_UNROLL || opt->backward_mode == DNLS_BWD_TRUNCATED;
  if (unroll && (opt->optimizer != DNLS_GN || prob->radius != nullptr))
    return fail(DNLS_E_UNSUPPORTED, "dnls_forward: UNROLL / TRUNCATED backward modes support Gauss-Newton with "
                                    "quadratic costs only");
  if (opt->backward_mode == DNLS_BWD_TRUNCATED && opt->backward_steps < 1)
    return fail(DNLS_E_INVALID, "dnls_forward: TRUNCATED needs backward_steps >= 1");
  if (opt->optimizer == DNLS_LM &&
      !(opt->lambda0 > 0 && opt->lambda_min > 0 && opt->lambda_max >= opt->lambda_min && opt->lambda_down > 1 &&
        opt->lambda_up > 1))
    return fail(DNLS_E_INVALID, "dnls_forward: invalid LM damping schedule");
  if (opt->optimizer == DNLS_DOGLEG &&
      !(opt->trust_radius0 > 0 && opt->trust_radius_min > 0 && opt->trust_radius_max >= opt->trust_radius0))
    return fail(DNLS_E_INVALID, "dnls_forward: invalid Dogleg trust radii");
  if (opt->damping != DNLS_DAMP_MARQUARDT && opt->damping != DNLS_DAMP_IDENTITY)
    return fail(DNLS_E_INVALID, "dnls_forward: unknown damping");
  if (opt->cluster_ctas != 0 && opt->cluster_ctas != 1 && opt->cluster_ctas != 2 && opt->cluster_ctas != 4 &&
      opt->cluster_ctas != 8)
    return fail(DNLS_E_INVALID, "dnls_forward: cluster_ctas must be 0 (automatic), 1, 2, 4 or 8");
  dnls_graph* gm = const_cast<dnls_graph*>(g);
  gm->drop(workspace);
  if (batch == 0) return DNLS_OK;
  DeviceGuard dguard(g->device);
  if (!dguard.ok) return fail(DNLS_E_CUDA, "dnls_forward: cannot select the graph's device");
  WsLayout l = ws_layout(g->sym, batch, keep);
  DevWs ws = ws_views(l, workspace);
  FwdParams fp;
  fp.K = opt->max_iterations;
  fp.lm = opt->optimizer == DNLS_LM;
  fp.alpha = opt->step_size;
  fp.lam0 = opt->lambda0;
  fp.lam_min = opt->lambda_min;
  fp.lam_max = opt->lambda_max;
  fp.lam_down = opt->lambda_down;
  fp.lam_up = opt->lambda_up;
  fp.damping = opt->damping;
  fp.early_stop = opt->early_stop;
  fp.abs_tol = opt->abs_tol;
  fp.rel_tol = opt->rel_tol;
  fp.implicit = opt->backward_mode == DNLS_BWD_IMPLICIT;
  fp.dogleg = opt->optimizer == DNLS_DOGLEG;
  fp.dl0 = opt->trust_radius0;
  fp.dl_max = opt->trust_radius_max;
  fp.dl_min = opt->trust_radius_min;
  fp.objective = prob->objective;
  fp.status = prob->status;
  fp.iterations = prob->iterations;
  cudaStream_t s = (cudaStream_t)stream;
  if (bl_choose(g, batch, opt, prob)) {
    if (ws_bytes < bl_ws_bytes(g, batch))
      return fail(DNLS_E_WORKSPACE, "dnls_forward: workspace too small for the batch-interleaved path (" +
                                        std::to_string(bl_ws_bytes(g, batch)) + " bytes)");
    BLPlan* pl = nullptr;
    if ((st = bl_plan_for(gm, &pl))) return st;
    const BLWs bw = bl_views(bl_layout(*pl, batch), workspace);
    BLPhaseTimer tm;
    tm.on = std::getenv("DNLS_PHASE_TIMING") != nullptr;
    DISPATCH_D(g->sym.D, bl_forward<DD>(*pl, batch, dev_prob(prob), bw, fp.K, fp.alpha, fp.early_stop, fp.abs_tol,
                                        fp.rel_tol, fp.implicit != 0, prob->objective, prob->status, prob->iterations,
                                        tm, s));
    if ((st = cuda_check("dnls_forward: batch-interleaved launches"))) return st;
    {
      std::lock_guard<std::mutex> lk(gm->bl_mu);
      for (auto& e : gm->phase_ev) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
      }
      gm->phase_ev = tm.ev;
    }
    if (fp.implicit) gm->keep(workspace, dnls_graph::FactorRecord{batch, DNLS_BWD_IMPLICIT, 0, 1.0, 1});
    return DNLS_OK;
  }
  const int cl = (opt->optimizer == DNLS_DOGLEG || unroll) ? 1 : forward_cluster(g, batch, opt->cluster_ctas);
  if (cl == 1) {
    DISPATCH_D(g->sym.D, if ((st = set_smem(k_forward<DD, 1>, smem_bytes(g->dg), "k_forward"))) return st; (DNLS_KL k_forward<DD, 1><<<batch, NT, smem_bytes(g->dg), s>>>(g->dg, dev_prob(prob), ws, fp)));
  } else if (launch_forward_cluster(cl, g->sym.D, g->dg, dev_prob(prob), ws, fp, batch, s) != cudaSuccess) {
    return fail(DNLS_E_CUDA, std::string("dnls_forward: cluster launch: ") + cudaGetErrorString(cudaGetLastError()));
  }
  if ((st = cuda_check("dnls_forward: k_forward launch"))) return st;
  if (fp.implicit) gm->keep(workspace, dnls_graph::FactorRecord{batch, DNLS_BWD_IMPLICIT, 0});
  if (unroll && keep > 0) gm->keep(workspace, dnls_graph::FactorRecord{batch, opt->backward_mode, keep, opt->step_size});
  return DNLS_OK;
}

DNLS_API dnls_status dnls_backward_implicit(const dnls_graph* g, int32_t batch, const dnls_problem* prob,
                                            const double* grad_poses, int32_t grad_kind, double* grad_w_edge,
                                            double* grad_w_prior, double* grad_radius, int64_t grad_bstride,
                                            void* workspace, size_t ws_bytes, void* stream) {
  dnls_status st = check_common("dnls_backward_implicit", g, batch, workspace, ws_bytes);
  if (st) return st;
  if ((st = check_problem("dnls_backward_implicit", g, prob))) return st;
  if (!grad_poses && batch > 0) return fail(DNLS_E_INVALID, "dnls_backward_implicit: grad_poses is NULL");
  if (grad_kind != DNLS_GRAD_TANGENT && grad_kind != DNLS_GRAD_MATRIX)
    return fail(DNLS_E_INVALID, "dnls_backward_implicit: unknown grad_kind");
  if (grad_bstride < 0) return fail(DNLS_E_INVALID, "dnls_backward_implicit: grad_bstride < 0");
  if (grad_bstride > 0 && grad_bstride < std::max(g->sym.E, g->sym.P))
    return fail(DNLS_E_SHAPE, "dnls_backward_implicit: grad_bstride smaller than num_edges/num_priors");
  dnls_graph::FactorRecord rec{};
  if (!const_cast<dnls_graph*>(g)->get(workspace, rec) || rec.batch != batch || rec.kind != DNLS_BWD_IMPLICIT)
    return fail(DNLS_E_STATE,
                "dnls_backward_implicit: no implicit-mode dnls_forward on this workspace/batch "
                "(factor cache missing or overwritten)");
  if (batch == 0) return DNLS_OK;
  DeviceGuard dguard(g->device);
  if (!dguard.ok) return fail(DNLS_E_CUDA, "dnls_backward_implicit: cannot select the graph's device");
  if (rec.layout == 1) {   // factor of the batch-interleaved path
    if (grad_radius && prob->radius)
      return fail(DNLS_E_UNSUPPORTED, "dnls_backward_implicit: no radius gradient on the batch-interleaved path");
    BLPlan* pl = nullptr;
    if ((st = bl_plan_for(const_cast<dnls_graph*>(g), &pl))) return st;
    const BLWs bw = bl_views(bl_layout(*pl, batch), workspace);
    DISPATCH_D(g->sym.D, bl_backward_implicit<DD>(*pl, batch, dev_prob(prob), bw, grad_poses, grad_kind, grad_w_edge,
                                                  grad_w_prior, (long long)grad_bstride, (cudaStream_t)stream));
    return cuda_check("dnls_backward_implicit: batch-interleaved launches");
  }
  WsLayout l = ws_layout(g->sym, batch);
  DevWs ws = ws_views(l, workspace);
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH_D(g->sym.D, if ((st = set_smem(k_backward<DD>, smem_bytes(g->dg), "k_backward"))) return st; (DNLS_KL k_backward<DD><<<batch, NT, smem_bytes(g->dg), s>>>(g->dg, dev_prob(prob), ws, grad_poses, grad_kind)));
  if ((st = cuda_check("dnls_backward_implicit: k_backward launch"))) return st;
  const int slots = g->sym.E + g->sym.P;
  if (slots > 0 && (grad_w_edge || grad_w_prior)) {
    DNLS_KL k_reduce_wgrad<<<(slots + 127) / 128, 128, 0, s>>>(batch, g->sym.E, g->sym.P, ws.cost, grad_w_edge,
                                                        grad_w_prior, (long long)grad_bstride);
    if ((st = cuda_check("dnls_backward_implicit: k_reduce_wgrad launch"))) return st;
  }
  if (grad_radius && prob->radius) {
    DNLS_KL k_reduce_radius<<<1, 32, 0, s>>>(batch, g->sym.E, slots, ws.rgrad, grad_radius, (long long)prob->radius_bstride);
    if ((st = cuda_check("dnls_backward_implicit: k_reduce_radius launch"))) return st;
  }
  return DNLS_OK;
}

DNLS_API dnls_status dnls_backward_dlm(const dnls_graph* g, int32_t batch, const dnls_problem* prob,
                                       const double* grad_poses, int32_t grad_kind, double epsilon,
                                       double* grad_w_edge, double* grad_w_prior, double* grad_radius,
                                       int64_t grad_bstride, void* workspace, size_t ws_bytes, void* stream) {
  dnls_status st = check_common("dnls_backward_dlm", g, batch, workspace, ws_bytes);
  if (st) return st;
  if ((st = check_problem("dnls_backward_dlm", g, prob))) return st;
  if (!grad_poses && batch > 0) return fail(DNLS_E_INVALID, "dnls_backward_dlm: grad_poses is NULL");
  if (grad_kind != DNLS_GRAD_TANGENT && grad_kind != DNLS_GRAD_MATRIX)
    return fail(DNLS_E_INVALID, "dnls_backward_dlm: unknown grad_kind");
  if (!(epsilon > 0.0) || !std::isfinite(epsilon))
    return fail(DNLS_E_INVALID, "dnls_backward_dlm: epsilon must be finite and > 0");
  if (grad_bstride < 0) return fail(DNLS_E_INVALID, "dnls_backward_dlm: grad_bstride < 0");
  if (grad_bstride > 0 && grad_bstride < std::max(g->sym.E, g->sym.P))
    return fail(DNLS_E_SHAPE, "dnls_backward_dlm: grad_bstride smaller than num_edges/num_priors");
  // the augmented factorisation overwrites any factor cached in this workspace
  const_cast<dnls_graph*>(g)->drop(workspace);
  if (batch == 0) return DNLS_OK;
  DeviceGuard dguard(g->device);
  if (!dguard.ok) return fail(DNLS_E_CUDA, "dnls_backward_dlm: cannot select the graph's device");
  WsLayout l = ws_layout(g->sym, batch);
  DevWs ws = ws_views(l, workspace);
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH_D(g->sym.D, if ((st = set_smem(k_backward_dlm<DD>, smem_bytes(g->dg), "k_backward_dlm"))) return st; (DNLS_KL k_backward_dlm<DD><<<batch, NT, smem_bytes(g->dg), s>>>(g->dg, dev_prob(prob), ws, grad_poses, grad_kind, epsilon)));
  if ((st = cuda_check("dnls_backward_dlm: k_backward_dlm launch"))) return st;
  const int slots = g->sym.E + g->sym.P;
  if (slots > 0 && (grad_w_edge || grad_w_prior)) {
    DNLS_KL k_reduce_wgrad<<<(slots + 127) / 128, 128, 0, s>>>(batch, g->sym.E, g->sym.P, ws.cost, grad_w_edge,
                                                        grad_w_prior, (long long)grad_bstride);
    if ((st = cuda_check("dnls_backward_dlm: k_reduce_wgrad launch"))) return st;
  }
  if (grad_radius && prob->radius) {
    DNLS_KL k_reduce_radius<<<1, 32, 0, s>>>(batch, g->sym.E, slots, ws.rgrad, grad_radius, (long long)prob->radius_bstride);
    if ((st = cuda_check("dnls_backward_dlm: k_reduce_radius launch"))) return st;
  }
  return DNLS_OK;
}

DNLS_API dnls_status dnls_backward_unroll(const dnls_graph* g, int32_t batch, const dnls_problem* prob,
                                          const double* grad_poses, int32_t grad_kind, double* grad_w_edge,
                                          double* grad_w_prior, double* grad_poses0, int64_t grad_bstride,
                                          void* workspace, size_t ws_bytes, void* stream) {
  if (!g) return fail(DNLS_E_INVALID, "dnls_backward_unroll: graph is NULL");
  dnls_graph::FactorRecord rec{};
  if (!const_cast<dnls_graph*>(g)->get(workspace, rec) || rec.batch != batch ||
      (rec.kind != DNLS_BWD_UNROLL && rec.kind != DNLS_BWD_TRUNCATED))
    return fail(DNLS_E_STATE, "dnls_backward_unroll: no unroll/truncated dnls_forward on this workspace/batch "
                              "(history missing or overwritten)");
  dnls_status st = check_common("dnls_backward_unroll", g, batch, workspace, ws_bytes, rec.K);
  if (st) return st;
  if ((st = check_problem("dnls_backward_unroll", g, prob))) return st;
  if (!grad_poses && batch > 0) return fail(DNLS_E_INVALID, "dnls_backward_unroll: grad_poses is NULL");
  if (grad_kind != DNLS_GRAD_TANGENT && grad_kind != DNLS_GRAD_MATRIX)
    return fail(DNLS_E_INVALID, "dnls_backward_unroll: unknown grad_kind");
  if (grad_bstride < 0) return fail(DNLS_E_INVALID, "dnls_backward_unroll: grad_bstride < 0");
  if (grad_bstride > 0 && grad_bstride < std::max(g->sym.E, g->sym.P))
    return fail(DNLS_E_SHAPE, "dnls_backward_unroll: grad_bstride smaller than num_edges/num_priors");
  if (batch == 0) return DNLS_OK;
  DeviceGuard dguard(g->device);
  if (!dguard.ok) return fail(DNLS_E_CUDA, "dnls_backward_unroll: cannot select the graph's device");
  DevWs ws = ws_views(ws_layout(g->sym, batch, rec.K), workspace);
  cudaStream_t s = (cudaStream_t)stream;
  // UNROLL differentiates every recorded iteration; TRUNCATED the last rec.K (= min(T, K)) of them
  const int Tw = rec.K;
  DISPATCH_D(g->sym.D, if ((st = set_smem(k_backward_unroll<DD>, smem_bytes(g->dg), "k_backward_unroll"))) return st;
             (DNLS_KL k_backward_unroll<DD><<<batch, NT, smem_bytes(g->dg), s>>>(g->dg, dev_prob(prob), ws, grad_poses,
                                                                         grad_kind, Tw, rec.alpha, grad_poses0)));
  if ((st = cuda_check("dnls_backward_unroll: k_backward_unroll launch"))) return st;
  const int slots = g->sym.E + g->sym.P;
  if (slots > 0 && (grad_w_edge || grad_w_prior)) {
    DNLS_KL k_reduce_wgrad<<<(slots + 127) / 128, 128, 0, s>>>(batch, g->sym.E, g->sym.P, ws.cost, grad_w_edge,
                                                        grad_w_prior, (long long)grad_bstride);
    if ((st = cuda_check("dnls_backward_unroll: k_reduce_wgrad launch"))) return st;
  }
  return DNLS_OK;
}

DNLS_API dnls_status dnls_linearize(const dnls_graph* g, int32_t batch, const dnls_problem* prob,
                                    const double* lambda, int32_t damping, void* workspace, size_t ws_bytes,
                                    void* stream) {
  dnls_status st = check_common("dnls_linearize", g, batch, workspace, ws_bytes);
  if (st) return st;
  if ((st = check_problem("dnls_linearize", g, prob))) return st;
  if (damping != DNLS_DAMP_MARQUARDT && damping != DNLS_DAMP_IDENTITY)
    return fail(DNLS_E_INVALID, "dnls_linearize: unknown damping");
  const_cast<dnls_graph*>(g)->drop(workspace);   // the factor storage is overwritten
  if (batch == 0) return DNLS_OK;
  DeviceGuard dguard(g->device);
  if (!dguard.ok) return fail(DNLS_E_CUDA, "dnls_linearize: cannot select the graph's device");
  DevWs ws = ws_views(ws_layout(g->sym, batch), workspace);
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH_D(g->sym.D, if ((st = set_smem(k_linearize<DD>, smem_bytes(g->dg), "k_linearize"))) return st;
             (DNLS_KL k_linearize<DD><<<batch, NT, smem_bytes(g->dg), s>>>(g->dg, dev_prob(prob), ws, lambda, damping, prob->objective)));
  return cuda_check("dnls_linearize: launch");
}

DNLS_API dnls_status dnls_factorize(const dnls_graph* g, int32_t batch, void* workspace, size_t ws_bytes,
                                    int32_t* status, void* stream) {
  dnls_status st = check_common("dnls_factorize", g, batch, workspace, ws_bytes);
  if (st) return st;
  const_cast<dnls_graph*>(g)->drop(workspace);   // the factor storage is overwritten
  if (batch == 0) return DNLS_OK;
  DeviceGuard dguard(g->device);
  if (!dguard.ok) return fail(DNLS_E_CUDA, "dnls_factorize: cannot select the graph's device");
  DevWs ws = ws_views(ws_layout(g->sym, batch), workspace);
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH_D(g->sym.D, if ((st = set_smem(k_factorize<DD>, smem_bytes(g->dg), "k_factorize"))) return st; (DNLS_KL k_factorize<DD><<<batch, NT, smem_bytes(g->dg), s>>>(g->dg, ws, status)));
  return cuda_check("dnls_factorize: launch");
}

DNLS_API dnls_status dnls_solve_factored(const dnls_graph* g, int32_t batch, void* workspace, size_t ws_bytes,
                                         const double* rhs, double* x, void* stream) {
  dnls_status st = check_common("dnls_solve_factored", g, batch, workspace, ws_bytes);
  if (st) return st;
  if ((st = per_element_storage("dnls_solve_factored", g, workspace))) return st;
  if (batch > 0 && (!rhs || !x)) return fail(DNLS_E_INVALID, "dnls_solve_factored: rhs/x is NULL");
  if (batch == 0) return DNLS_OK;
  DeviceGuard dguard(g->device);
  if (!dguard.ok) return fail(DNLS_E_CUDA, "dnls_solve_factored: cannot select the graph's device");
  DevWs ws = ws_views(ws_layout(g->sym, batch), workspace);
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH_D(g->sym.D, if ((st = set_smem(k_solve<DD>, smem_bytes(g->dg), "k_solve"))) return st; (DNLS_KL k_solve<DD><<<batch, NT, smem_bytes(g->dg), s>>>(g->dg, ws, rhs, x)));
  return cuda_check("dnls_solve_factored: launch");
}

DNLS_API dnls_status dnls_export_factor(const dnls_graph* g, int32_t batch, const void* workspace, size_t ws_bytes,
                                        double* dense, void* stream) {
  dnls_status st = check_common("dnls_export_factor", g, batch, workspace, ws_bytes);
  if (st) return st;
  if ((st = per_element_storage("dnls_export_factor", g, workspace))) return st;
  if (batch > 0 && !dense) return fail(DNLS_E_INVALID, "dnls_export_factor: dense is NULL");
  if (batch == 0) return DNLS_OK;
  DeviceGuard dguard(g->device);
  if (!dguard.ok) return fail(DNLS_E_CUDA, "dnls_export_factor: cannot select the graph's device");
  DevWs ws = ws_views(ws_layout(g->sym, batch), const_cast<void*>(workspace));
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH_D(g->sym.D, (DNLS_KL k_export_factor<DD><<<batch, NT, 0, s>>>(g->dg, ws, dense)));
  return cuda_check("dnls_export_factor: launch");
}

DNLS_API dnls_status dnls_import_matrix(const dnls_graph* g, int32_t batch, const double* dense, void* workspace,
                                        size_t ws_bytes, void* stream) {
  dnls_status st = check_common("dnls_import_matrix", g, batch, workspace, ws_bytes);
  if (st) return st;
  if (batch > 0 && !dense) return fail(DNLS_E_INVALID, "dnls_import_matrix: dense is NULL");
  const_cast<dnls_graph*>(g)->drop(workspace);   // the factor storage is overwritten
  if (batch == 0) return DNLS_OK;
  DeviceGuard dguard(g->device);
  if (!dguard.ok) return fail(DNLS_E_CUDA, "dnls_import_matrix: cannot select the graph's device");
  DevWs ws = ws_views(ws_layout(g->sym, batch), workspace);
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH_D(g->sym.D, (DNLS_KL k_import_matrix<DD><<<batch, NT, 0, s>>>(g->dg, ws, dense)));
  return cuda_check("dnls_import_matrix: launch");
}

DNLS_API dnls_status dnls_export_rhs(const dnls_graph* g, int32_t batch, const void* workspace, size_t ws_bytes,
                                     double* b, void* stream) {
  dnls_status st = check_common("dnls_export_rhs", g, batch, workspace, ws_bytes);
  if (st) return st;
  if ((st = per_element_storage("dnls_export_rhs", g, workspace))) return st;
  if (batch > 0 && !b) return fail(DNLS_E_INVALID, "dnls_export_rhs: b is NULL");
  if (batch == 0) return DNLS_OK;
  DeviceGuard dguard(g->device);
  if (!dguard.ok) return fail(DNLS_E_CUDA, "dnls_export_rhs: cannot select the graph's device");
  DevWs ws = ws_views(ws_layout(g->sym, batch), const_cast<void*>(workspace));
  cudaStream_t s = (cudaStream_t)stream;
  DISPATCH_D(g->sym.D, (DNLS_KL k_export_rhs<DD><<<batch, NT, 0, s>>>(g->dg, ws, b)));
  return cuda_check("dnls_export_rhs: launch");
}

}  // extern "C"
#endif  // DNLS_CLUSTER_TU
