// Batch-interleaved, level-major path ("BL") for many problems per GPU
// (BASELINE.json C4 / C5: 1024 poses x 256..2048 problems).  Included by dnls.cu inside its anonymous
// namespace (it reuses the per-cost device math of phases.cuh and the helpers of dnls.cu).
//
// The one-CTA-per-element kernel (k_forward) runs the elimination tree of ONE element level by level, so
// every level costs a barrier-separated latency chain while the SM is mostly idle.  Here the batch is the
// innermost dimension instead:
//   * storage is element-interleaved: entry i of the factor of element b lives at L[i * Bp + b]
//     (Bp = B rounded up to 32), so the 32 lanes of a warp -- 32 consecutive elements doing the SAME
//     item -- move 256 contiguous bytes per access (fully coalesced, no divergence, no shuffles);
//   * the factorisation is pose-level left-looking block Cholesky (every block d x d, stored column-major
//     36 / 9 doubles): per elimination-tree level one launch gathers the updates of the level's target
//     blocks (T_pk -= sum_s L_ps L_ks^T, one thread per (element, target block)) and the forward-substitution
//     rows, one launch factors the level's columns (redundant register Cholesky of L_kk per thread, one
//     TRSM block row per thread, fused y_k = L_kk^-1 x_k);
//   * every phase of the GN iteration (linearise, assemble, factor, solve, retract) is a grid of
//     (element, item) threads; the host enqueues the launches of all K iterations on the stream.
// Same arithmetic as the per-element path up to summation order (parity against the oracle, tests).
// Gauss-Newton (and the implicit backward) with quadratic or Welsch costs; LM / Dogleg / DLM / unroll
// use the per-element path.

constexpr int BL_TPB = 128;

// Programmatic dependent launch (PDL): every BL kernel is launched with programmatic stream serialisation, so
// the next kernel on the stream is scheduled while this one drains; it waits (griddepcontrol.wait: the previous
// grid has completed and its memory is visible) before touching any data, then lets its own dependent launch.
// g_bl_pdl = 0 (DNLS_PDL=0) launches without the attribute (the wait is then a no-op).
__device__ __forceinline__ void bl_pdl() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
inline int bl_pdl_on() {
  static const int on = [] {
    const char* e = std::getenv("DNLS_PDL");
    return e ? std::atoi(e) : 1;
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline void bl_launch_smem(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  ::dnls::g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = bl_pdl_on() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
inline void bl_launch(void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  bl_launch_smem(k, grid, block, 0, s, args...);
}
   // threads per block of the BL kernels (4 warps = 4 items x 32 elements)

struct BLDev {
  int D, N, E, P, n, nblk, Bp, B;
  int gmajor;            // bl_update_rb: group-major warp order (DNLS_BL_GMAJOR)
  const int *perm, *iperm, *edges, *prior_vars;
  const int* colptr;     // [N+1] blocks of permuted column k (diagonal block first, then rows ascending)
  const int* blkrow;     // [nblk] row pose of each block
  const int4* tsk;       // update tasks: (target block, con begin, con end, diagonal flag)
  const int2* con;       // contributions: (block (p, s), block (k, s))
  const int* fwdp;       // [N+1] per column: forward-substitution contributions
  const int2* fwd;       // (block (k, s), s)
  const int2* fac;       // factor items: (column k, block)
  const int4* slotd;     // per slot: (off-diagonal block or -1, row pose is j, unique flag, 0)
  const int *bc_ptr, *bc;   // per permuted pose: slot * 2 + side (fixed gather order)
  const int *dup_ptr, *dup_blk, *dup_con;   // off-diagonal blocks shared by several edges: their slots
  const int* fill;       // blocks no cost writes (fill-in), zeroed before assembly
  int nfill, ndup;
};

// per-call device views of the BL workspace
struct BLWs {
  double* L;       // [nblk * DD][Bp]   assembled H blocks; below-diagonal blocks become L (diagonal blocks keep
                   //                   the updated T_kk: the column's TRSM threads read it while L_kk is written)
  double* Ld;      // [N * DD][Bp]     L_kk of every column (lower triangle) + inverse pivots (upper triangle)
  double* x;       // [n][Bp]        rhs / solution (permuted order)
  double* scr;     // [slots * SW][Bp] per-slot assembly contributions
  double* cost;    // [slots][Bp]    per-slot objective (weight gradients in the backward)
  double* S;       // [Bp]
  double* Sprev;   // [Bp]
  unsigned long long* maxd;   // [Bp] max diagonal (bits of a non-negative double: integer max == double max)
  int* fail;       // [Bp] factorisation failure flag
  int* st;         // [Bp] status
  int* it;         // [Bp] iterations
  int* stf;        // [Bp] final status (the iteration status is parked here during the final linearisation)
};

template <int D>
struct BLC {
  static constexpr int DD = D * D, NL = D * (D + 1) / 2;
  // slot scratch fields (doubles): H_i (lower, NL), H_j (lower, NL), b_i (D), b_j (D), H_ij (DD)
  static constexpr int H0 = 0, H1 = NL, B0 = 2 * NL, B1 = 2 * NL + D, HIJ = 2 * NL + 2 * D, SW = 2 * NL + 2 * D + DD;
};

__device__ __forceinline__ bool bl_item(const BLDev& g, long long nitems, int& b, long long& item) {
  const long long t = (long long)blockIdx.x * BL_TPB + threadIdx.x;
  b = (int)(t % g.Bp);
  item = t / g.Bp;
  return item < nitems;
}
__device__ __forceinline__ bool bl_frozen(const BLWs& w, int b) { return w.st[b] != DNLS_ST_OK; }
// group-major variant: consecutive warps take the items of one group of 32 elements, so the CTAs resident at
// a time work on few groups and share their source blocks through L2 (g.gmajor)
__device__ __forceinline__ bool bl_item_gm(const BLDev& g, long long nitems, int& b, long long& item) {
  const long long t = (long long)blockIdx.x * BL_TPB + threadIdx.x;
  const long long wp = t >> 5;
  const long long grp = wp / nitems;
  item = wp - grp * nitems;
  b = (int)(grp * 32 + (t & 31));
  return grp < (g.Bp >> 5);
}

// DevGraph with only the fields the per-cost device math (slot_jac / eval_slot / slot_cost) reads
__device__ __forceinline__ DevGraph bl_cost_graph(const BLDev& g) {
  DevGraph d{};
  d.D = g.D;
  d.N = g.N;
  d.E = g.E;
  d.P = g.P;
  d.edges = g.edges;
  d.prior_vars = g.prior_vars;
  return d;
}

// ---------------------------------------------------------------------------- assembly (a1 + a2)
__global__ void __launch_bounds__(BL_TPB) bl_zero_fill(BLDev g, BLWs w, int DD, const int* fill, int nfill) {
  bl_pdl();
  int b;
  long long it;
  if (!bl_item(g, (long long)nfill * DD, b, it)) return;
  if (b >= g.B || bl_frozen(w, b)) return;
  const int k = (int)(it / DD), e = (int)(it - (long long)k * DD);
  w.L[((size_t)fill[k] * DD + e) * g.Bp + b] = 0.0;
}

// thread per (element, cost slot): compact Jacobian in registers, objective term, the slot's off-diagonal
// block stored straight into the factor storage (single edge between its poses) or into the scratch,
// the diagonal contributions and J^T r parts into the scratch (PAPER.md:64 J^T J, J^T r)
template <int D>
__global__ void __launch_bounds__(BL_TPB) bl_lin_slots(BLDev g, DevProb pr, BLWs w) {
  bl_pdl();
  using C = BLC<D>;
  int b;
  long long it;
  const int slots = g.E + g.P;
  if (!bl_item(g, slots, b, it)) return;
  if (b >= g.B || bl_frozen(w, b)) return;
  const int slot = (int)it;
  const DevGraph cg = bl_cost_graph(g);
  const double* Tb = pr.poses + (size_t)b * g.N * GT<D>::PS;
  SlotJ<D> J;
  slot_jac<D>(cg, pr, Tb, b, slot, J);
  double n2 = 0.0;
#pragma unroll
  for (int q = 0; q < D; ++q) n2 = fma(J.c[q], J.c[q], n2);
  double psi;
  w.cost[(size_t)slot * g.Bp + b] = slot_cost(cg, pr, b, slot, J.ww * n2, psi);
  J.ww *= psi;   // IRLS rescaling (reading W2)
  const size_t Bp = g.Bp;
  double* o = w.scr + (size_t)slot * C::SW * Bp + b;
  const bool edge = slot < g.E;
  // H_i / b_i: pose i (a prior's pose plays C_j's role: block 0 / rhs side 0, as in linearize_phase)
  int e = 0;
#pragma unroll
  for (int q = 0; q < D; ++q)
#pragma unroll
    for (int a = q; a < D; ++a, ++e) {
      o[(C::H0 + e) * Bp] = edge ? blk<D>(J, 1, a, q) : blk<D>(J, 0, a, q);
      if (edge) o[(C::H1 + e) * Bp] = blk<D>(J, 0, a, q);
    }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    o[(C::B0 + a) * Bp] = edge ? rhs<D>(J, 1, a) : rhs<D>(J, 0, a);
    if (edge) o[(C::B1 + a) * Bp] = rhs<D>(J, 0, a);
  }
  if (edge) {
    const int4 sd = g.slotd[slot];
    double* T = sd.z ? w.L + (size_t)sd.x * C::DD * Bp + b : o + C::HIJ * Bp;
#pragma unroll
    for (int q = 0; q < D; ++q)
#pragma unroll
      for (int a = 0; a < D; ++a) T[(q * D + a) * Bp] = sd.y ? blk<D>(J, 3, a, q) : blk<D>(J, 2, a, q);
  }
}

// thread per (element, permuted pose): its diagonal block and b segment are the sums of its slots'
// contributions in the fixed order of bc (deterministic, no atomics on values), damped, written once;
// the element's max diagonal by an integer atomicMax on the bits of a non-negative double
template <int D>
__global__ void __launch_bounds__(BL_TPB) bl_lin_poses(BLDev g, BLWs w, double lam, int damping) {
  bl_pdl();
  using C = BLC<D>;
  int b;
  long long it;
  if (!bl_item(g, g.N + g.ndup, b, it)) return;
  if (b >= g.B || bl_frozen(w, b)) return;
  const size_t Bp = g.Bp;
  if (it >= g.N) {   // an off-diagonal block shared by several (parallel) edges
    const int k = (int)it - g.N;
    double h[C::DD];
#pragma unroll
    for (int i = 0; i < C::DD; ++i) h[i] = 0.0;
    for (int c = g.dup_ptr[k]; c < g.dup_ptr[k + 1]; ++c) {
      const double* o = w.scr + ((size_t)g.dup_con[c] * C::SW + C::HIJ) * Bp + b;
#pragma unroll
      for (int i = 0; i < C::DD; ++i) h[i] += o[i * Bp];
    }
    double* T = w.L + (size_t)g.dup_blk[k] * C::DD * Bp + b;
#pragma unroll
    for (int i = 0; i < C::DD; ++i) T[i * Bp] = h[i];
    return;
  }
  const int p = (int)it;
  double h[C::NL], r[D];
#pragma unroll
  for (int i = 0; i < C::NL; ++i) h[i] = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) r[a] = 0.0;
  const int cb0 = g.bc_ptr[p], cb1 = g.bc_ptr[p + 1];
  int nxc = cb0 < cb1 ? __ldg(&g.bc[cb0]) : 0;
  for (int c = cb0; c < cb1; ++c) {
    const int code = nxc;
    nxc = __ldg(&g.bc[c + 1 < cb1 ? c + 1 : c]);
    const int side = code & 1;
    const double* o = w.scr + (size_t)(code >> 1) * C::SW * Bp + b;
    const double* oh = o + (side ? C::H1 : C::H0) * Bp;
    const double* orr = o + (side ? C::B1 : C::B0) * Bp;
#pragma unroll
    for (int i = 0; i < C::NL; ++i) h[i] += oh[i * Bp];
#pragma unroll
    for (int a = 0; a < D; ++a) r[a] += orr[a * Bp];
  }
  double* T = w.L + (size_t)g.colptr[p] * C::DD * Bp + b;
  double mymax = 0.0;
  int e = 0;
#pragma unroll
  for (int q = 0; q < D; ++q)
#pragma unroll
    for (int a = q; a < D; ++a, ++e) {
      double v = h[e];
      if (a == q) {
        if (lam > 0.0) v = (damping == 0) ? v * (1.0 + lam) : v + lam;
        mymax = fmax(mymax, v);
      }
      T[(q * D + a) * Bp] = v;
      if (a != q) T[(a * D + q) * Bp] = 0.0;   // upper triangle: the inverse pivots go there later
    }
#pragma unroll
  for (int a = 0; a < D; ++a) w.x[((size_t)p * D + a) * Bp + b] = r[a];
  if (mymax > 0.0) atomicMax(&w.maxd[b], (unsigned long long)__double_as_longlong(mymax));
}

// S = sum of the slot terms (fixed order: BL_SW warps each sum a contiguous slot range for the same 32
// elements, then the partials in warp order); final == 0: early stop (reading A14) and S_prev update,
// final == 1: S(theta_K) only
constexpr int BL_SW = 32;
__global__ void __launch_bounds__(BL_SW * 32) bl_objective(BLDev g, BLWs w, int early_stop, double abs_tol,
                                                          double rel_tol, int have_prev, int set_prev, int final) {
  bl_pdl();
  __shared__ double part[BL_SW][33];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int b = blockIdx.x * 32 + lane;
  const int slots = g.E + g.P, chunk = (slots + BL_SW - 1) / BL_SW;
  const int s0 = wp * chunk, s1 = min(slots, s0 + chunk);
  double acc = 0.0;
  if (b < g.B)
    for (int sl = s0; sl < s1; ++sl) acc += w.cost[(size_t)sl * g.Bp + b];
  part[wp][lane] = acc;
  __syncthreads();
  if (wp != 0 || b >= g.B) return;
  double S = 0.0;
#pragma unroll 8
  for (int q = 0; q < BL_SW; ++q) S += part[q][lane];
  if (final) {
    w.S[b] = S;
    return;
  }
  if (w.st[b] != DNLS_ST_OK) return;
  if (early_stop && have_prev && fabs(S - w.Sprev[b]) < abs_tol + rel_tol * w.Sprev[b]) w.st[b] = DNLS_ST_CONVERGED;
  w.S[b] = S;
  if (set_prev) w.Sprev[b] = S;
}
__global__ void __launch_bounds__(BL_TPB) bl_reset_iter(BLDev g, BLWs w) {
  bl_pdl();
  const int b = blockIdx.x * BL_TPB + threadIdx.x;
  if (b >= g.Bp) return;
  w.maxd[b] = 0ull;
  w.fail[b] = 0;
}

// ---------------------------------------------------------------------------- factorisation (a3 + fused a4 forward)
// Row-split items: one CTA = D warps x 32 consecutive elements works on one item; warp r owns row r of the
// item's d x d block (or component r of a vector), so every thread issues all loads of one source block
// before its FMAs (one memory round trip per contribution) and the d row threads share the column data
// through L1.  blockIdx.x = item * (Bp / 32) + element group.
__device__ __forceinline__ bool bl_row_item(const BLDev& g, long long nitems, int& b, long long& item, int& r) {
  const int groups = g.Bp >> 5;
  item = blockIdx.x / groups;
  b = ((blockIdx.x - (int)(item * groups)) << 5) + (threadIdx.x & 31);
  r = threadIdx.x >> 5;
  return item < nitems;
}
inline unsigned bl_grid_rows(long long items, int Bp) { return (unsigned)(items * (Bp >> 5)); }
// compiler fence between a batch of independent loads and their consumers: every load of the batch is
// issued before the first FMA (one memory round trip per batch instead of one per few loads)
__device__ __forceinline__ void bl_issue_fence() { asm volatile("" ::: "memory"); }

// level l: update tasks T_pk -= sum_s L_ps L_ks^T (items [0, ntask)) and forward-substitution rows
// x_k -= sum_s L_ks y_s of the level's columns (items [ntask, ntask + ncol)); warp r = row r
template <int D>
__global__ void __launch_bounds__(D * 32, 3) bl_update(BLDev g, BLWs w, int t0, int ntask, const int* cols, int ncol,
                                                    int fused_fwd) {
  bl_pdl();
  using C = BLC<D>;
  int b, r;
  long long it;
  if (!bl_row_item(g, (long long)ntask + (fused_fwd ? ncol : 0), b, it, r)) return;
  if (b >= g.B || bl_frozen(w, b)) return;
  const size_t Bp = g.Bp;
  if (it < ntask) {
    const int4 tk = g.tsk[t0 + it];
    double acc[D];
#pragma unroll
    for (int j = 0; j < D; ++j) acc[j] = 0.0;
    for (int ci = tk.y; ci < tk.z; ++ci) {
      const int2 cn = g.con[ci];
      const double* Pp = w.L + ((size_t)cn.x * C::DD + r) * Bp + b;   // row r of L_ps: stride D entries
      const double* Kp = w.L + (size_t)cn.y * C::DD * Bp + b;
      double pv[D], kv[D][D];
#pragma unroll
      for (int c = 0; c < D; ++c) pv[c] = Pp[(size_t)c * D * Bp];
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int j = 0; j < D; ++j) kv[c][j] = (!(tk.w & 1) || j <= r) ? Kp[(c * D + j) * Bp] : 0.0;
      bl_issue_fence();
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int j = 0; j < D; ++j) acc[j] = fma(pv[c], kv[c][j], acc[j]);
    }
    double* T = w.L + ((size_t)tk.x * C::DD + r) * Bp + b;
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (!(tk.w & 1) || r >= j) T[(size_t)j * D * Bp] -= acc[j];
    return;
  }
  const int k = cols[it - ntask];
  double acc = 0.0;
  for (int ci = g.fwdp[k]; ci < g.fwdp[k + 1]; ++ci) {
    const int2 f = g.fwd[ci];
    const double* Kp = w.L + ((size_t)f.x * C::DD + r) * Bp + b;
    const double* y = w.x + (size_t)f.y * D * Bp + b;
    double kv[D], yv[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      kv[c] = Kp[(size_t)c * D * Bp];
      yv[c] = y[c * Bp];
    }
    bl_issue_fence();
#pragma unroll
    for (int c = 0; c < D; ++c) acc = fma(kv[c], yv[c], acc);
  }
  w.x[((size_t)k * D + r) * Bp + b] -= acc;
}

// level l, register-blocked: thread = (element, item); an update task accumulates the WHOLE d x d target
// block in registers (acc[i][j] = sum_s sum_c L_ps[i][c] L_ks[j][c]), streaming the two source blocks
// column by column (half a block pair per memory round trip): 2 d^2 loads per d^3 FMAs instead of the
// row-split kernel's d (d + d^2).  A diagonal target (p == k) reads its single source block once and keeps
// the lower triangle.  Fill targets (tk.w & 2: no cost writes them) are stored as -acc, so they need no
// zeroing pass.  Warps enumerate (item, group of 32 elements) item-major.
template <int D>
#ifndef DNLS_RB_MINB
#define DNLS_RB_MINB 3
#endif
__global__ void __launch_bounds__(BL_TPB, DNLS_RB_MINB) bl_update_rb(BLDev g, BLWs w, int t0, int ntask, const int* cols, int ncol,
                                                       int fused_fwd) {
  bl_pdl();
  using C = BLC<D>;
#ifndef DNLS_RB_HD
#define DNLS_RB_HD 1
#endif
  constexpr int H = D / DNLS_RB_HD;   // source columns per round trip
  int b;
  long long it;
  const long long nit = (long long)ntask + (fused_fwd ? ncol : 0);
  if (!(g.gmajor ? bl_item_gm(g, nit, b, it) : bl_item(g, nit, b, it))) return;
  if (b >= g.B || bl_frozen(w, b)) return;
  const size_t Bp = g.Bp;
  if (it < ntask) {
    const int4 tk = g.tsk[t0 + it];
    double acc[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) acc[i][j] = 0.0;
    if (tk.w & 1) {   // diagonal target: T_kk -= sum_s L_ks L_ks^T (lower triangle)
      for (int ci = tk.y; ci < tk.z; ++ci) {
        const double* Kp = w.L + (size_t)g.con[ci].y * C::DD * Bp + b;
#pragma unroll
        for (int h = 0; h < D; h += H) {
          double kv[H][D];
#pragma unroll
          for (int c = 0; c < H; ++c)
#pragma unroll
            for (int j = 0; j < D; ++j) kv[c][j] = Kp[((h + c) * D + j) * Bp];
          bl_issue_fence();
#pragma unroll
          for (int c = 0; c < H; ++c)
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
              for (int j = 0; j <= i; ++j) acc[i][j] = fma(kv[c][i], kv[c][j], acc[i][j]);
        }
      }
    } else {
      for (int ci = tk.y; ci < tk.z; ++ci) {
        const int2 cn = g.con[ci];
        const double* Pp = w.L + (size_t)cn.x * C::DD * Bp + b;
        const double* Kp = w.L + (size_t)cn.y * C::DD * Bp + b;
#pragma unroll
        for (int h = 0; h < D; h += H) {
          double pv[H][D], kv[H][D];
#pragma unroll
          for (int c = 0; c < H; ++c)
#pragma unroll
            for (int j = 0; j < D; ++j) {
              pv[c][j] = Pp[((h + c) * D + j) * Bp];
              kv[c][j] = Kp[((h + c) * D + j) * Bp];
            }
          bl_issue_fence();
#pragma unroll
          for (int c = 0; c < H; ++c)
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
              for (int j = 0; j < D; ++j) acc[i][j] = fma(pv[c][i], kv[c][j], acc[i][j]);
        }
      }
    }
    double* T = w.L + (size_t)tk.x * C::DD * Bp + b;
    const bool diag = tk.w & 1, fill = tk.w & 2;
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int i = 0; i < D; ++i) {
        if (diag && i < j) continue;
        double* t = T + (size_t)(j * D + i) * Bp;
        *t = fill ? -acc[i][j] : *t - acc[i][j];
      }
    return;
  }
  // forward-substitution row of column k: x_k -= sum_s L_ks y_s
  const int k = cols[it - ntask];
  double acc[D];
#pragma unroll
  for (int i = 0; i < D; ++i) acc[i] = 0.0;
  for (int ci = g.fwdp[k]; ci < g.fwdp[k + 1]; ++ci) {
    const int2 f = g.fwd[ci];
    const double* Kp = w.L + (size_t)f.x * C::DD * Bp + b;
    const double* y = w.x + (size_t)f.y * D * Bp + b;
    double kv[D][D], yv[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      yv[c] = y[c * Bp];
#pragma unroll
      for (int i = 0; i < D; ++i) kv[c][i] = Kp[(c * D + i) * Bp];
    }
    bl_issue_fence();
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int i = 0; i < D; ++i) acc[i] = fma(kv[c][i], yv[c], acc[i]);
  }
  double* xk = w.x + (size_t)k * D * Bp + b;
#pragma unroll
  for (int i = 0; i < D; ++i) xk[i * Bp] -= acc[i];
}

// ---------------------------------------------------------------------------- persistent factorisation
// One launch per factorisation.  One CTA = one group of GW consecutive elements for ALL levels; units of GW
// threads (thread = element) take a level's work round robin and levels are separated by __syncthreads, so a
// group's separator chain at the top of the elimination tree is worked by all units of its CTA instead of one
// thread per (target, element) behind a per-level launch.
//   * wide levels (>= coltask_min columns): a unit takes a whole column k -- the diagonal target's updates,
//     L_kk in registers, the forward-substitution row and y_k = L_kk^-1 x_k, then every below target's updates
//     solved straight from the accumulators (L_pk = (T_pk - acc) L_kk^-T): each block is read once and
//     written once, T_kk is never stored.  Same arithmetic (and rounding) as bl_update_rb + bl_factor.
//   * narrow levels: the contribution lists are split into chunks over all units (partial sums in the slot
//     scratch, idle during the factorisation, subtracted in chunk order), then the level's blocks are factored
//     unit by unit (bl_factor's arithmetic: redundant register Cholesky of L_kk per block).
constexpr int BLP_NT = 256;
#ifndef DNLS_PT_HD
#define DNLS_PT_HD 1   // bl_acc_target: source columns per round trip = D / DNLS_PT_HD
#endif

struct BLPDev {
  const int4* bcon;     // [nblk] per block: (contribution begin, end, flags (bit 0 diagonal, bit 1 fill), 0)
  const int* it_lvl;    // [L+1] narrow levels: their work items
  const int4* items;    // (target block or -1 = forward row, begin, end, flags | (partial slot + 1) << 8)
  const int* rd_lvl;    // [L+1] narrow levels: their split reductions
  const int4* red;      // (target block or -1, first slot, count, flags)
  const int* lvl_ptr;   // [L+1] columns of each level in lvl_col
  const int* lvl_col;
  const int* fac_lvl;   // [L+1] factor items (g.fac) of each level
  int L, coltask_min;
};

template <int D>
__device__ __forceinline__ void bl_chol(double (&a)[D][D], double (&iv)[D], double tol, bool& bad) {
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double piv = a[j][j];
#pragma unroll
    for (int q = 0; q < j; ++q) piv = fma(-a[j][q], a[j][q], piv);
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
      for (int q = 0; q < j; ++q) s = fma(-a[i][q], a[j][q], s);
      a[i][j] = s * inv;
    }
  }
}

// acc[i][j] = sum over the contributions [c0, c1) of (L_ps L_ks^T)(i, j) (diag: lower triangle, L_ks == L_ps),
// register-blocked, a whole block pair per memory round trip.  init != nullptr (the in-place form): acc starts from
// the target block T (entry (i, j) at init[(j D + i) Bp]) and the products are subtracted, acc = T - sum -- the
// target's loads then share the first contribution's round trip instead of costing one after the loop.
template <int D>
__device__ __forceinline__ void bl_acc_target(const BLDev& g, const BLWs& w, int b, int c0, int c1, bool diag,
                                              double (&acc)[D][D], const double* init = nullptr) {
  using C = BLC<D>;
  constexpr int H = D / DNLS_PT_HD;
  const size_t Bp = g.Bp;
  const double sg = init ? -1.0 : 1.0;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) acc[i][j] = (init && (!diag || j <= i)) ? init[(j * D + i) * Bp] : 0.0;
  // the next contribution's block indices are loaded in the same memory round trip as this one's blocks
  int2 cn = c0 < c1 ? __ldg(&g.con[c0]) : make_int2(0, 0);
  if (diag) {
    for (int ci = c0; ci < c1; ++ci) {
      const int2 nx = __ldg(&g.con[ci + 1 < c1 ? ci + 1 : ci]);
      const double* Kp = w.L + (size_t)cn.y * C::DD * Bp + b;
#pragma unroll
      for (int h = 0; h < D; h += H) {
        double kv[H][D];
#pragma unroll
        for (int c = 0; c < H; ++c)
#pragma unroll
          for (int j = 0; j < D; ++j) kv[c][j] = Kp[((h + c) * D + j) * Bp];
        bl_issue_fence();
#pragma unroll
        for (int c = 0; c < H; ++c)
#pragma unroll
          for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j) acc[i][j] = fma(sg * kv[c][i], kv[c][j], acc[i][j]);
      }
      cn = nx;
    }
  } else {
    for (int ci = c0; ci < c1; ++ci) {
      const int2 nx = __ldg(&g.con[ci + 1 < c1 ? ci + 1 : ci]);
      const double* Pp = w.L + (size_t)cn.x * C::DD * Bp + b;
      const double* Kp = w.L + (size_t)cn.y * C::DD * Bp + b;
#pragma unroll
      for (int h = 0; h < D; h += H) {
        double pv[H][D], kv[H][D];
#pragma unroll
        for (int c = 0; c < H; ++c)
#pragma unroll
          for (int j = 0; j < D; ++j) {
            pv[c][j] = Pp[((h + c) * D + j) * Bp];
            kv[c][j] = Kp[((h + c) * D + j) * Bp];
          }
        bl_issue_fence();
#pragma unroll
        for (int c = 0; c < H; ++c)
#pragma unroll
          for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) acc[i][j] = fma(sg * pv[c][i], kv[c][j], acc[i][j]);
      }
      cn = nx;
    }
  }
}

// forward-substitution sum of column k over [f0, f1): acc = sum_s L_ks y_s; init != nullptr: acc = x_k - sum
template <int D>
__device__ __forceinline__ void bl_acc_fwd(const BLDev& g, const BLWs& w, int b, int f0, int f1, double (&acc)[D],
                                           const double* init = nullptr) {
  using C = BLC<D>;
  const size_t Bp = g.Bp;
  const double sg = init ? -1.0 : 1.0;
#pragma unroll
  for (int i = 0; i < D; ++i) acc[i] = init ? init[i * Bp] : 0.0;
  int2 f = f0 < f1 ? __ldg(&g.fwd[f0]) : make_int2(0, 0);
  for (int q = f0; q < f1; ++q) {
    const int2 nx = __ldg(&g.fwd[q + 1 < f1 ? q + 1 : q]);
    const double* Kp = w.L + (size_t)f.x * C::DD * Bp + b;
    const double* y = w.x + (size_t)f.y * D * Bp + b;
    double kv[D][D], yv[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      yv[c] = y[c * Bp];
#pragma unroll
      for (int i = 0; i < D; ++i) kv[c][i] = Kp[(c * D + i) * Bp];
    }
    bl_issue_fence();
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int i = 0; i < D; ++i) acc[i] = fma(sg * kv[c][i], yv[c], acc[i]);
    f = nx;
  }
}

// L_kk + inverse pivots -> Ld, failure flag, fused y_k = L_kk^-1 x_k
template <int D>
__device__ __forceinline__ void bl_store_diag(const BLDev& g, const BLWs& w, int b, int k, const double (&a)[D][D],
                                              const double (&iv)[D], bool bad, bool fused_fwd) {
  using C = BLC<D>;
  const size_t Bp = g.Bp;
  double* Lk = w.Ld + (size_t)k * C::DD * Bp + b;
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int i = j; i < D; ++i) Lk[(j * D + i) * Bp] = a[i][j];
#pragma unroll
  for (int j = 0; j < D; ++j) Lk[ivpos<D>(0, j, D) * Bp] = iv[j];
  if (bad) w.fail[b] = 1;
  if (fused_fwd) {
    double* xk = w.x + (size_t)k * D * Bp + b;
    double y[D];
#pragma unroll
    for (int q = 0; q < D; ++q) {
      double s = xk[q * Bp];
#pragma unroll
      for (int r = 0; r < q; ++r) s = fma(-a[q][r], y[r], s);
      y[q] = s * iv[q];
    }
#pragma unroll
    for (int q = 0; q < D; ++q) xk[q * Bp] = y[q];
  }
}

// L_pk = t L_kk^-T row by row, t given column-major (t[q][r] = entry (r, q)); stored into the block
template <int D>
__device__ __forceinline__ void bl_trsm_store(double* Pb, size_t Bp, double (&t)[D][D], const double (&a)[D][D],
                                              const double (&iv)[D]) {
#pragma unroll
  for (int r = 0; r < D; ++r) {
#pragma unroll
    for (int q = 0; q < D; ++q) {
      double s = t[q][r];
#pragma unroll
      for (int j = 0; j < q; ++j) s = fma(-t[j][r], a[q][j], s);
      t[q][r] = s * iv[q];
    }
#pragma unroll
    for (int q = 0; q < D; ++q) Pb[(q * D + r) * Bp] = t[q][r];
  }
}

// column task: the whole column k for element b -- the diagonal target's updates, L_kk in registers, the
// forward-substitution row and y_k = L_kk^-1 x_k, then every below target's updates solved straight from the
// accumulators (L_pk = (T_pk - acc) L_kk^-T): each block is read once and written once, T_kk is never stored.
// Same arithmetic (and rounding) as bl_update_rb + bl_factor (same contribution order per target).
// column record: r0 = (k, first block, end block, forward begin), r1 = (forward end, diagonal contributions
// begin, end, 0) -- one load instead of a chain colptr -> bcon
__device__ __forceinline__ void bl_column_record(const BLDev& g, const int4* bcon, int k, int4& r0, int4& r1) {
  const int kb0 = g.colptr[k];
  const int4 bc = bcon[kb0];
  r0 = make_int4(k, kb0, g.colptr[k + 1], g.fwdp[k]);
  r1 = make_int4(g.fwdp[k + 1], bc.x, bc.y, 0);
}

template <int D>
__device__ __forceinline__ void bl_column_task(const BLDev& g, const BLWs& w, const int4* bcon, int b, const int4 r0,
                                               const int4 r1, double tol, bool fused_fwd) {
  using C = BLC<D>;
  const size_t Bp = g.Bp;
  const int k = r0.x, kb0 = r0.y, kb1 = r0.z;
  double a[D][D], iv[D];
  int4 bcn = kb0 + 1 < kb1 ? bcon[kb0 + 1] : make_int4(0, 0, 0, 0);   // the first below block's range, early
  bl_acc_target<D>(g, w, b, r1.y, r1.z, true, a, w.L + (size_t)kb0 * C::DD * Bp + b);   // a = T_kk - sum
  bool bad = false;
  bl_chol<D>(a, iv, tol, bad);
  bl_store_diag<D>(g, w, b, k, a, iv, bad, false);
  if (fused_fwd) {   // y_k = L_kk^-1 (x_k - sum_s L_ks y_s), x_k read in the first contribution's round trip
    double* xk = w.x + (size_t)k * D * Bp + b;
    double t[D], y[D];
    bl_acc_fwd<D>(g, w, b, r0.w, r1.x, t, xk);
#pragma unroll
    for (int q = 0; q < D; ++q) {
      double s2 = t[q];
#pragma unroll
      for (int r = 0; r < q; ++r) s2 = fma(-a[q][r], y[r], s2);
      y[q] = s2 * iv[q];
    }
#pragma unroll
    for (int q = 0; q < D; ++q) xk[q * Bp] = y[q];
  }
  for (int bi = kb0 + 1; bi < kb1; ++bi) {
    const int4 bc = bcn;
    if (bi + 1 < kb1) bcn = bcon[bi + 1];   // the next block's range, with this block's loads
    double* Pb = w.L + (size_t)bi * C::DD * Bp + b;
    double acc[D][D];
    bl_acc_target<D>(g, w, b, bc.x, bc.y, false, acc, (bc.z & 2) ? nullptr : Pb);   // T_pk - sum (fill: -sum)
    double t[D][D];
#pragma unroll
    for (int q = 0; q < D; ++q)
#pragma unroll
      for (int r = 0; r < D; ++r) t[q][r] = (bc.z & 2) ? -acc[r][q] : acc[r][q];
    bl_trsm_store<D>(Pb, Bp, t, a, iv);
  }
}

// work item (target block, or forward row -2 - k; contribution range [y, z); flags | (partial slot + 1) << 8):
// a whole list is applied in place (T -= acc; a fill target stores -acc; x_k -= acc), a chunk of a split list
// stores its partial sum in the slot scratch (idle during the factorisation) for the reduction
template <int D>
__device__ __forceinline__ void bl_work_item(const BLDev& g, const BLWs& w, double* part, const int4 itm, int b,
                                             bool fused_fwd) {
  using C = BLC<D>;
  const size_t Bp = g.Bp;
  const int slot = (itm.w >> 8) - 1;
  if (itm.x >= 0) {
    const bool diag = itm.w & 1, fill = itm.w & 2;
    double* T = slot >= 0 ? part + (size_t)slot * C::DD * Bp + b : w.L + (size_t)itm.x * C::DD * Bp + b;
    double acc[D][D];
    // in place: acc = T - sum (a fill target: -sum); a chunk partial: acc = sum
    bl_acc_target<D>(g, w, b, itm.y, itm.z, diag, acc, (slot >= 0 || fill) ? nullptr : T);
    const double sg = (slot < 0 && fill) ? -1.0 : 1.0;
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int i = 0; i < D; ++i) {
        if (diag && i < j) continue;
        T[(size_t)(j * D + i) * Bp] = sg * acc[i][j];
      }
  } else if (fused_fwd) {
    const int k = -2 - itm.x;
    double* X = slot >= 0 ? part + (size_t)slot * C::DD * Bp + b : w.x + (size_t)k * D * Bp + b;
    double acc[D];
    bl_acc_fwd<D>(g, w, b, itm.y, itm.z, acc, slot >= 0 ? nullptr : X);
#pragma unroll
    for (int i = 0; i < D; ++i) X[i * Bp] = acc[i];
  }
}

// level l of the large-batch schedule: thread = (element, work item) over the level's items, where
// contribution lists longer than the plan's chunk size are split (a level's time is set by its longest
// update chain: one memory round trip per contribution); the partials are reduced by bl_factor_red
template <int D>
__global__ void __launch_bounds__(BL_TPB, DNLS_RB_MINB) bl_update_items(BLDev g, BLWs w, const int4* items, int i0,
                                                                       int nit, int fused_fwd) {
  bl_pdl();
  int b;
  long long it;
  if (!bl_item(g, nit, b, it) || b >= g.B) return;
  const int4 itm = items[i0 + it];   // loaded with the status: one round trip before the item's data
  if (w.st[b] != DNLS_ST_OK) return;
  bl_work_item<D>(g, w, w.scr, itm, b, fused_fwd != 0);
}

// bl_factor with the level's split reductions folded in: T_kk and T_pk minus their chunk partials (in chunk
// order), x_k minus the forward row's partials, then bl_factor's arithmetic.  pr = (first slot, count) per
// block (bred) and per column's forward row (cred).
template <int D>
__device__ __forceinline__ void bl_factor_item(const BLDev& g, const BLWs& w, const int4 fr, int b, bool fused_fwd,
                                               const int2* bred, const int2* cred) {
  using C = BLC<D>;
  const size_t Bp = g.Bp;
  const int k = fr.x, kb0 = fr.z;   // record: (column, block, the column's diagonal block, 0)
  const int2 fi = make_int2(fr.x, fr.y);
  const bool diag = fi.y == kb0;
  const double* Kk = w.L + (size_t)kb0 * C::DD * Bp + b;
  double* Pb = w.L + (size_t)fi.y * C::DD * Bp + b;
  const double* part = w.scr + b;
  const double tol = 1e-13 * __longlong_as_double((long long)w.maxd[b]);
  double a[D][D], iv[D], t[D][D];
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int i = j; i < D; ++i) a[i][j] = Kk[(j * D + i) * Bp];
  if (!diag) {
#pragma unroll
    for (int q = 0; q < D; ++q)
#pragma unroll
      for (int r = 0; r < D; ++r) t[q][r] = Pb[(q * D + r) * Bp];
  }
  // T_kk's chunk partials, two per memory round trip (subtracted in chunk order)
  const int2 rk = bred[kb0];
  int q = 0;
  for (; q + 1 < rk.y; q += 2) {
    const double* p0 = part + (size_t)(rk.x + q) * C::DD * Bp;
    const double* p1 = p0 + (size_t)C::DD * Bp;
    double v0[D][D], v1[D][D];
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int i = j; i < D; ++i) {
        v0[i][j] = p0[(j * D + i) * Bp];
        v1[i][j] = p1[(j * D + i) * Bp];
      }
    bl_issue_fence();
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int i = j; i < D; ++i) a[i][j] = (a[i][j] - v0[i][j]) - v1[i][j];
  }
  if (q < rk.y) {
    const double* pp = part + (size_t)(rk.x + q) * C::DD * Bp;
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int i = j; i < D; ++i) a[i][j] -= pp[(j * D + i) * Bp];
  }
  if (!diag) {
    const int2 rp = bred[fi.y];
    for (int q = 0; q < rp.y; ++q) {
      const double* pp = part + (size_t)(rp.x + q) * C::DD * Bp;
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int r = 0; r < D; ++r) t[c][r] -= pp[(c * D + r) * Bp];
    }
  }
  bool bad = false;
  bl_chol<D>(a, iv, tol, bad);
  if (diag) {
    if (fused_fwd) {
      const int2 rc = cred[k];
      if (rc.y > 0) {
        double* xk = w.x + (size_t)k * D * Bp + b;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          double v = xk[i * Bp];
          for (int q = 0; q < rc.y; ++q) v -= part[((size_t)(rc.x + q) * C::DD + i) * Bp];
          xk[i * Bp] = v;
        }
      }
    }
    bl_store_diag<D>(g, w, b, k, a, iv, bad, fused_fwd != 0);
    return;
  }
  bl_trsm_store<D>(Pb, Bp, t, a, iv);
}

template <int D>
__global__ void __launch_bounds__(BL_TPB) bl_factor_red(BLDev g, BLWs w, const int4* facr, int f0, int nfac,
                                                       int fused_fwd, const int2* bred, const int2* cred) {
  bl_pdl();
  int b;
  long long it;
  if (!bl_item(g, nfac, b, it) || b >= g.B) return;
  const int4 fr = facr[f0 + it];   // loaded with the status: one round trip before the item's data
  if (w.st[b] != DNLS_ST_OK) return;
  bl_factor_item<D>(g, w, fr, b, fused_fwd != 0, bred, cred);
}

// bottom of the elimination tree in ONE launch: every maximal subtree of columns of height <= the plan's
// sub_top is an item; thread = (element, subtree) walks the subtree's columns in increasing index (children
// before parents: parent[k] > k) as column tasks.  A subtree's factor blocks are written and re-read by the
// same thread within a few microseconds, so the left-looking source re-reads hit L1 / L2 instead of DRAM and
// the bottom levels cost no per-level launches.  Items are ordered by decreasing size (largest first).
template <int D>
#ifndef DNLS_SUB_MINB
#define DNLS_SUB_MINB 2
#endif
__global__ void __launch_bounds__(BL_TPB, DNLS_SUB_MINB) bl_subtree(BLDev g, BLWs w, const int4* bcon, const int* sub_ptr,
                                                       const int4* sub_rec, int nsub, int fused_fwd) {
  bl_pdl();
  int b;
  long long it;
  if (!bl_item(g, nsub, b, it)) return;
  if (b >= g.B || bl_frozen(w, b)) return;
  const double tol = 1e-13 * __longlong_as_double((long long)w.maxd[b]);
  const int q0 = sub_ptr[it], q1 = sub_ptr[it + 1];
  int4 r0 = sub_rec[2 * q0], r1 = sub_rec[2 * q0 + 1];
  for (int q = q0; q < q1; ++q) {
    const int4 c0 = r0, c1 = r1;
    if (q + 1 < q1) {   // the next column's record, with this column's first loads
      r0 = sub_rec[2 * q + 2];
      r1 = sub_rec[2 * q + 3];
    }
    bl_column_task<D>(g, w, bcon, b, c0, c1, tol, fused_fwd != 0);
  }
}

// next work index of a unit: dynamic scheduling through a shared counter (the result of an item does not depend
// on the unit that computes it, so the schedule does not affect the arithmetic)
template <int GW>
__device__ __forceinline__ int bl_next(int* ctr, int base) {
  const int lane = threadIdx.x & 31, lead = lane & ~(GW - 1);
  const unsigned mask = (GW == 32) ? 0xffffffffu : (((1u << GW) - 1u) << lead);
  int v = 0;
  if (lane == lead) v = atomicAdd(ctr, 1);
  return base + __shfl_sync(mask, v, lead);
}

template <int D, int GW>
__global__ void __launch_bounds__(BLP_NT, 1) bl_persist(BLDev g, BLWs w, BLPDev pd, int fused_fwd, int l_begin,
                                                        int l_end) {
  bl_pdl();
  using C = BLC<D>;
  __shared__ int ctr[4];
  const int b = blockIdx.x * GW + (threadIdx.x % GW);
  const bool act = b < g.B && !bl_frozen(w, b);
  const size_t Bp = g.Bp;
  const double tol = act ? 1e-13 * __longlong_as_double((long long)w.maxd[b]) : 0.0;
  double* part = w.scr;   // partial sums of split items: [slot][DD][Bp]
  if (threadIdx.x < 4) ctr[threadIdx.x] = 0;
  __syncthreads();
  int ph = 0;   // counters rotate over ctr[0..3]; a counter is reset two phases before its reuse
  auto next = [&](int base) { return bl_next<GW>(&ctr[ph & 3], base); };
  auto phase_end = [&]() {
    if (threadIdx.x == 0) ctr[(ph + 2) & 3] = 0;
    ++ph;
    __syncthreads();
  };
  for (int l = l_begin; l < l_end; ++l) {
    const int c0 = pd.lvl_ptr[l], c1 = pd.lvl_ptr[l + 1];
    if (c1 - c0 >= pd.coltask_min) {
      // ---- wide level: one column per unit
      // every lane of a unit takes part in the scheduling (frozen elements skip the arithmetic)
      for (int ci = next(c0); ci < c1; ci = next(c0)) {
          if (!act) continue;
          int4 r0, r1;
          bl_column_record(g, pd.bcon, pd.lvl_col[ci], r0, r1);
          bl_column_task<D>(g, w, pd.bcon, b, r0, r1, tol, fused_fwd != 0);
        }
      phase_end();
      continue;
    }
    // ---- narrow level, A: work items (targets / forward rows, long lists in chunks)
    for (int ii = next(pd.it_lvl[l]); ii < pd.it_lvl[l + 1]; ii = next(pd.it_lvl[l])) {
        if (!act) continue;
        bl_work_item<D>(g, w, part, pd.items[ii], b, fused_fwd != 0);
      }
    if (pd.rd_lvl[l + 1] > pd.rd_lvl[l]) {
      phase_end();
      // ---- R: split items, partials subtracted in chunk order
      for (int ri = next(pd.rd_lvl[l]); ri < pd.rd_lvl[l + 1]; ri = next(pd.rd_lvl[l])) {
          if (!act) continue;
          const int4 rd = pd.red[ri];
          if (rd.x >= 0) {
            const bool diag = rd.w & 1, fill = rd.w & 2;
            double* T = w.L + (size_t)rd.x * C::DD * Bp + b;
#pragma unroll
            for (int j = 0; j < D; ++j)
#pragma unroll
              for (int i = 0; i < D; ++i) {
                if (diag && i < j) continue;
                double v = fill ? 0.0 : T[(j * D + i) * Bp];
                for (int q = 0; q < rd.z; ++q) v -= part[((size_t)(rd.y + q) * C::DD + j * D + i) * Bp + b];
                T[(j * D + i) * Bp] = v;
              }
          } else if (fused_fwd) {
            double* xk = w.x + (size_t)(-2 - rd.x) * D * Bp + b;
#pragma unroll
            for (int i = 0; i < D; ++i) {
              double v = xk[i * Bp];
              for (int q = 0; q < rd.z; ++q) v -= part[((size_t)(rd.y + q) * C::DD + i) * Bp + b];
              xk[i * Bp] = v;
            }
          }
        }
    }
    phase_end();
    // ---- F: the level's blocks (bl_factor's arithmetic)
    for (int fi = next(pd.fac_lvl[l]); fi < pd.fac_lvl[l + 1]; fi = next(pd.fac_lvl[l])) {
        if (!act) continue;
        const int2 f = g.fac[fi];
        const int k = f.x;
        const int kb0 = g.colptr[k];
        const double* Kk = w.L + (size_t)kb0 * C::DD * Bp + b;
        double a[D][D], iv[D];
#pragma unroll
        for (int j = 0; j < D; ++j)
#pragma unroll
          for (int i = j; i < D; ++i) a[i][j] = Kk[(j * D + i) * Bp];
        bool bad = false;
        bl_chol<D>(a, iv, tol, bad);
        if (f.y == kb0) {
          bl_store_diag<D>(g, w, b, k, a, iv, bad, fused_fwd != 0);
        } else {
          double* Pb = w.L + (size_t)f.y * C::DD * Bp + b;
          double t[D][D];
#pragma unroll
          for (int q = 0; q < D; ++q)
#pragma unroll
            for (int r = 0; r < D; ++r) t[q][r] = Pb[(q * D + r) * Bp];
          bl_trsm_store<D>(Pb, Bp, t, a, iv);
        }
      }
    phase_end();
  }
}

// level-parallel persistent triangular solves over the levels [l_begin, L) (backward: root -> l_begin, forward:
// l_begin -> root): one CTA per group of GW elements, U = BLP_NT / GW units.  Per level, the level's items --
// (column, below block) pairs for the backward substitution, (column, forward contribution) pairs for the forward
// one, contiguous per column -- go round robin over the units, each storing its d-vector product in shared
// memory; after one barrier the units take the level's columns: x_k minus the column's item vectors in item order
// (independent of which unit computed them), then L_kk^-T (backward) / L_kk^-1 (forward).  Two barriers per level
// instead of a launch per level (or two barriers per column in bl_persist_solve).
struct BLSDev {
  const int2* bit;      // backward items (column position in lvl_col, block)
  const int* bit_lvl;   // [L+1]
  const int2* bcol;     // per column position: (first backward item, count)
  const int2* fit;      // forward items (column position, forward contribution index)
  const int* fit_lvl;   // [L+1]
  const int2* fcol;     // per column position: (first forward item, count)
};

template <int D, int GW>
__global__ void __launch_bounds__(BLP_NT, 2) bl_lsolve(BLDev g, BLWs w, BLPDev pd, BLSDev sd, const int* skip,
                                                    int forward, int l_begin, int l_end) {
  bl_pdl();
  using C = BLC<D>;
  constexpr int U = BLP_NT / GW;
  extern __shared__ double spart[];   // [level items][D][GW]
  const int u = threadIdx.x / GW, e = threadIdx.x % GW;
  const int b = blockIdx.x * GW + e;
  const bool act = b < g.B && !(skip && skip[b]);
  const size_t Bp = g.Bp;
  const int2* items = forward ? sd.fit : sd.bit;
  const int* ilvl = forward ? sd.fit_lvl : sd.bit_lvl;
  const int2* icol = forward ? sd.fcol : sd.bcol;
  const int nl = l_end - l_begin;
  // a column's x_k, strictly lower L_kk entries and inverse pivots: the unit's first column of the level is
  // loaded before the level's items (in their memory round trip), the others after the barrier
  auto load_col = [&](int ci, int& k, int2& rg, double (&xv)[D], double (&lo)[D][D], double (&iv)[D]) {
    k = pd.lvl_col[ci];
    rg = icol[ci];
    const double* xk = w.x + (size_t)k * D * Bp + b;
    const double* Lk = w.Ld + (size_t)k * C::DD * Bp + b;
#pragma unroll
    for (int q = 0; q < D; ++q) {
      xv[q] = xk[q * Bp];
      iv[q] = Lk[ivpos<D>(0, q, D) * Bp];
#pragma unroll
      for (int r = 0; r < q; ++r) lo[q][r] = Lk[(r * D + q) * Bp];   // entry (q, r), q > r
    }
  };
  for (int li = 0; li < nl; ++li) {
    const int l = forward ? l_begin + li : l_end - 1 - li;
    const int i0 = ilvl[l], i1 = ilvl[l + 1];
    const int ci0 = pd.lvl_ptr[l] + u;
    int k0 = 0;
    int2 rg0 = make_int2(0, 0);
    double xp[D], lp[D][D], ivp[D];
    if (act && ci0 < pd.lvl_ptr[l + 1]) load_col(ci0, k0, rg0, xp, lp, ivp);
    for (int ii = i0 + u; ii < i1; ii += U) {
      double acc[D];
#pragma unroll
      for (int i = 0; i < D; ++i) acc[i] = 0.0;
      if (act) {
        const int2 it = items[ii];
        if (forward) {   // acc = L_ks y_s
          const int2 f = g.fwd[it.y];
          const double* Kp = w.L + (size_t)f.x * C::DD * Bp + b;
          const double* y = w.x + (size_t)f.y * D * Bp + b;
          double kv[D][D], yv[D];
#pragma unroll
          for (int c = 0; c < D; ++c) {
            yv[c] = y[c * Bp];
#pragma unroll
            for (int i = 0; i < D; ++i) kv[c][i] = Kp[(c * D + i) * Bp];
          }
          bl_issue_fence();
#pragma unroll
          for (int c = 0; c < D; ++c)
#pragma unroll
            for (int i = 0; i < D; ++i) acc[i] = fma(kv[c][i], yv[c], acc[i]);
        } else {   // acc = L_pk^T x_p
          const double* P0 = w.L + (size_t)it.y * C::DD * Bp + b;
          const double* x0 = w.x + (size_t)g.blkrow[it.y] * D * Bp + b;
          double lv[D][D], xv[D];
#pragma unroll
          for (int q = 0; q < D; ++q) {
            xv[q] = x0[q * Bp];
#pragma unroll
            for (int c = 0; c < D; ++c) lv[c][q] = P0[(c * D + q) * Bp];
          }
          bl_issue_fence();
#pragma unroll
          for (int c = 0; c < D; ++c)
#pragma unroll
            for (int q = 0; q < D; ++q) acc[c] = fma(lv[c][q], xv[q], acc[c]);
        }
      }
#pragma unroll
      for (int i = 0; i < D; ++i) spart[((size_t)(ii - i0) * D + i) * GW + e] = acc[i];
    }
    __syncthreads();
    for (int ci = ci0; ci < pd.lvl_ptr[l + 1]; ci += U) {
      if (!act) continue;
      int k;
      int2 rg;
      double t[D], lo[D][D], iv[D], y[D];
      if (ci == ci0) {
        k = k0;
        rg = rg0;
#pragma unroll
        for (int q = 0; q < D; ++q) {
          t[q] = xp[q];
          iv[q] = ivp[q];
#pragma unroll
          for (int r = 0; r < q; ++r) lo[q][r] = lp[q][r];
        }
      } else {
        load_col(ci, k, rg, t, lo, iv);
      }
      for (int q = 0; q < rg.y; ++q)
#pragma unroll
        for (int i = 0; i < D; ++i) t[i] -= spart[((size_t)(rg.x - i0 + q) * D + i) * GW + e];
      if (forward) {
#pragma unroll
        for (int q = 0; q < D; ++q) {
          double s2 = t[q];
#pragma unroll
          for (int r = 0; r < q; ++r) s2 = fma(-lo[q][r], y[r], s2);
          y[q] = s2 * iv[q];
        }
      } else {
#pragma unroll
        for (int q = D - 1; q >= 0; --q) {
          double s2 = t[q];
#pragma unroll
          for (int p = q + 1; p < D; ++p) s2 = fma(-lo[p][q], y[p], s2);
          y[q] = s2 * iv[q];
        }
      }
      double* xk = w.x + (size_t)k * D * Bp + b;
#pragma unroll
      for (int i = 0; i < D; ++i) xk[i * Bp] = y[i];
    }
    __syncthreads();
  }
}

// persistent triangular solves over a level range (the single-column tail of the tree): one CTA per group of
// GW elements; per column the units split the column's list (backward: its below blocks, forward: its
// forward-substitution contributions), partial sums in shared memory added in unit order, unit 0 applies
// L_kk^-T / L_kk^-1.  Backward runs the levels root -> l_begin, forward l_begin -> root.
template <int D, int GW>
__global__ void __launch_bounds__(BLP_NT) bl_persist_solve(BLDev g, BLWs w, BLPDev pd, const int* skip, int forward,
                                                           int l_begin, int l_end) {
  bl_pdl();
  using C = BLC<D>;
  constexpr int U = BLP_NT / GW;
  __shared__ double part[U][D][GW];
  const int u = threadIdx.x / GW, e = threadIdx.x % GW;
  const int b = blockIdx.x * GW + e;
  const bool act = b < g.B && !(skip && skip[b]);
  const size_t Bp = g.Bp;
  const int nl = l_end - l_begin;
  for (int li = 0; li < nl; ++li) {
    const int l = forward ? l_begin + li : l_end - 1 - li;
    for (int ci = pd.lvl_ptr[l]; ci < pd.lvl_ptr[l + 1]; ++ci) {
      const int k = pd.lvl_col[ci];
      double acc[D];
#pragma unroll
      for (int i = 0; i < D; ++i) acc[i] = 0.0;
      if (act) {
        if (forward) {
          for (int q = g.fwdp[k] + u; q < g.fwdp[k + 1]; q += U) {
            const int2 f = g.fwd[q];
            const double* Kp = w.L + (size_t)f.x * C::DD * Bp + b;
            const double* y = w.x + (size_t)f.y * D * Bp + b;
            double kv[D][D], yv[D];
#pragma unroll
            for (int c = 0; c < D; ++c) {
              yv[c] = y[c * Bp];
#pragma unroll
              for (int i = 0; i < D; ++i) kv[c][i] = Kp[(c * D + i) * Bp];
            }
            bl_issue_fence();
#pragma unroll
            for (int c = 0; c < D; ++c)
#pragma unroll
              for (int i = 0; i < D; ++i) acc[i] = fma(kv[c][i], yv[c], acc[i]);
          }
        } else {
          for (int bi = g.colptr[k] + 1 + u; bi < g.colptr[k + 1]; bi += U) {
            const double* P0 = w.L + (size_t)bi * C::DD * Bp + b;
            const double* x0 = w.x + (size_t)g.blkrow[bi] * D * Bp + b;
            double lv[D][D], xv[D];
#pragma unroll
            for (int q = 0; q < D; ++q) {
              xv[q] = x0[q * Bp];
#pragma unroll
              for (int c = 0; c < D; ++c) lv[c][q] = P0[(c * D + q) * Bp];
            }
            bl_issue_fence();
#pragma unroll
            for (int c = 0; c < D; ++c)
#pragma unroll
              for (int q = 0; q < D; ++q) acc[c] = fma(lv[c][q], xv[q], acc[c]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < D; ++i) part[u][i][e] = acc[i];
      __syncthreads();
      if (u == 0 && act) {
        double* xk = w.x + (size_t)k * D * Bp + b;
        const double* Lk = w.Ld + (size_t)k * C::DD * Bp + b;
        double t[D], y[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
          double s = 0.0;
          for (int v = 0; v < U; ++v) s += part[v][i][e];
          t[i] = xk[i * Bp] - s;
        }
        if (forward) {
#pragma unroll
          for (int q = 0; q < D; ++q) {
            double s2 = t[q];
#pragma unroll
            for (int r = 0; r < q; ++r) s2 = fma(-Lk[(r * D + q) * Bp], y[r], s2);
            y[q] = s2 * Lk[ivpos<D>(0, q, D) * Bp];
          }
        } else {
#pragma unroll
          for (int q = D - 1; q >= 0; --q) {
            double s2 = t[q];
#pragma unroll
            for (int p = q + 1; p < D; ++p) s2 = fma(-Lk[(q * D + p) * Bp], y[p], s2);
            y[q] = s2 * Lk[ivpos<D>(0, q, D) * Bp];
          }
        }
#pragma unroll
        for (int i = 0; i < D; ++i) xk[i * Bp] = y[i];
      }
      __syncthreads();
    }
  }
}

// level l: item (column k, block): every thread factors L_kk in registers (redundantly; no barrier between
// the diagonal Cholesky and the TRSM rows); the diagonal item stores L_kk, the inverse pivots (in the
// block's unused upper triangle) and applies y_k = L_kk^-1 x_k; a below item solves L_pk = T_pk L_kk^-T
template <int D>
__global__ void __launch_bounds__(BL_TPB) bl_factor(BLDev g, BLWs w, int f0, int nfac, int fused_fwd) {
  bl_pdl();
  using C = BLC<D>;
  int b;
  long long it;
  if (!(g.gmajor ? bl_item_gm(g, nfac, b, it) : bl_item(g, nfac, b, it))) return;
  if (b >= g.B || bl_frozen(w, b)) return;
  const size_t Bp = g.Bp;
  const int2 fi = g.fac[f0 + it];
  const int k = fi.x;
  const bool diag = fi.y == g.colptr[k];
  const double* Kk = w.L + (size_t)g.colptr[k] * C::DD * Bp + b;
  double* Pb = w.L + (size_t)fi.y * C::DD * Bp + b;
  const double tol = 1e-13 * __longlong_as_double((long long)w.maxd[b]);
  // T_kk and (a below item) the whole T_pk in one memory round trip, before any store
  double a[D][D], iv[D], t[D][D];
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int i = j; i < D; ++i) a[i][j] = Kk[(j * D + i) * Bp];
  if (!diag) {
#pragma unroll
    for (int q = 0; q < D; ++q)
#pragma unroll
      for (int r = 0; r < D; ++r) t[q][r] = Pb[(q * D + r) * Bp];
  }
  bool bad = false;
  bl_chol<D>(a, iv, tol, bad);
  if (diag) {
    bl_store_diag<D>(g, w, b, k, a, iv, bad, fused_fwd != 0);
    return;
  }
  bl_trsm_store<D>(Pb, Bp, t, a, iv);   // row r of L_pk: x L_kk^T = t
}

// failed factorisation -> element frozen at its iterate (GN: status NOT_SPD), reading A15
__global__ void __launch_bounds__(BL_TPB) bl_check_fail(BLDev g, BLWs w) {
  bl_pdl();
  const int b = blockIdx.x * BL_TPB + threadIdx.x;
  if (b >= g.B) return;
  if (w.fail[b] && w.st[b] == DNLS_ST_OK) w.st[b] = DNLS_ST_NOT_SPD;
}

// ---------------------------------------------------------------------------- triangular solves (a4 / a7)
// standalone forward substitution of a level's columns: y_k = L_kk^-1 (x_k - sum_s L_ks y_s); warp r sums
// component r, warp 0 applies L_kk^-1 (shared memory exchange)
template <int D>
__global__ void __launch_bounds__(D * 32, 3) bl_fsolve(BLDev g, BLWs w, const int* cols, int ncol, const int* skip) {
  bl_pdl();
  using C = BLC<D>;
  __shared__ double sv[D][32];
  int b, r;
  long long it;
  if (!bl_row_item(g, ncol, b, it, r)) return;   // uniform per CTA
  const bool act = b < g.B && !(skip && skip[b]);
  const size_t Bp = g.Bp;
  const int k = cols[it];
  const int lane = threadIdx.x & 31;
  if (act) {
    double acc = w.x[((size_t)k * D + r) * Bp + b];
    for (int ci = g.fwdp[k]; ci < g.fwdp[k + 1]; ++ci) {
      const int2 f = g.fwd[ci];
      const double* Kp = w.L + ((size_t)f.x * C::DD + r) * Bp + b;
      const double* y = w.x + (size_t)f.y * D * Bp + b;
      double kv[D], yv[D];
#pragma unroll
      for (int c = 0; c < D; ++c) {
        kv[c] = Kp[(size_t)c * D * Bp];
        yv[c] = y[c * Bp];
      }
      bl_issue_fence();
#pragma unroll
      for (int c = 0; c < D; ++c) acc = fma(-kv[c], yv[c], acc);
    }
    sv[r][lane] = acc;
  }
  __syncthreads();
  if (r != 0 || !act) return;
  const double* Lk = w.Ld + (size_t)k * C::DD * Bp + b;
  double y[D];
#pragma unroll
  for (int q = 0; q < D; ++q) {
    double s2 = sv[q][lane];
#pragma unroll
    for (int p = 0; p < q; ++p) s2 = fma(-Lk[(p * D + q) * Bp], y[p], s2);
    y[q] = s2 * Lk[ivpos<D>(0, q, D) * Bp];
  }
#pragma unroll
  for (int q = 0; q < D; ++q) w.x[((size_t)k * D + q) * Bp + b] = y[q];
}

// backward substitution of a level's columns (levels root -> leaves): x_k = L_kk^-T (y_k - sum_p L_pk^T x_p);
// warp c sums component c over the column's below blocks (two blocks per round trip), warp 0 applies L_kk^-T
template <int D>
__global__ void __launch_bounds__(D * 32, 3) bl_bsolve(BLDev g, BLWs w, const int* cols, int ncol, const int* skip) {
  bl_pdl();
  using C = BLC<D>;
  __shared__ double sv[D][32];
  int b, c;
  long long it;
  if (!bl_row_item(g, ncol, b, it, c)) return;
  const bool act = b < g.B && !(skip && skip[b]);
  const size_t Bp = g.Bp;
  const int k = cols[it];
  const int lane = threadIdx.x & 31;
  if (act) {
    double acc = w.x[((size_t)k * D + c) * Bp + b], acc2 = 0.0;
    const int b0 = g.colptr[k] + 1, b1 = g.colptr[k + 1];
    int bi = b0;
    for (; bi + 1 < b1; bi += 2) {
      const double* P0 = w.L + ((size_t)bi * C::DD + c * D) * Bp + b;   // column c of L_pk: D contiguous entries
      const double* P1 = P0 + (size_t)C::DD * Bp;
      const double* x0 = w.x + (size_t)g.blkrow[bi] * D * Bp + b;
      const double* x1 = w.x + (size_t)g.blkrow[bi + 1] * D * Bp + b;
      double l0[D], l1[D], v0[D], v1[D];
#pragma unroll
      for (int q = 0; q < D; ++q) {
        l0[q] = P0[q * Bp];
        l1[q] = P1[q * Bp];
        v0[q] = x0[q * Bp];
        v1[q] = x1[q * Bp];
      }
      bl_issue_fence();
#pragma unroll
      for (int q = 0; q < D; ++q) {
        acc = fma(-l0[q], v0[q], acc);
        acc2 = fma(-l1[q], v1[q], acc2);
      }
    }
    if (bi < b1) {
      const double* P0 = w.L + ((size_t)bi * C::DD + c * D) * Bp + b;
      const double* x0 = w.x + (size_t)g.blkrow[bi] * D * Bp + b;
      double l0[D], v0[D];
#pragma unroll
      for (int q = 0; q < D; ++q) {
        l0[q] = P0[q * Bp];
        v0[q] = x0[q * Bp];
      }
#pragma unroll
      for (int q = 0; q < D; ++q) acc = fma(-l0[q], v0[q], acc);
    }
    sv[c][lane] = acc + acc2;
  }
  __syncthreads();
  if (c != 0 || !act) return;
  const double* Lk = w.Ld + (size_t)k * C::DD * Bp + b;
  double y[D];
#pragma unroll
  for (int q = D - 1; q >= 0; --q) {
    double s2 = sv[q][lane];
#pragma unroll
    for (int p = q + 1; p < D; ++p) s2 = fma(-Lk[(q * D + p) * Bp], y[p], s2);
    y[q] = s2 * Lk[ivpos<D>(0, q, D) * Bp];
  }
#pragma unroll
  for (int q = 0; q < D; ++q) w.x[((size_t)k * D + q) * Bp + b] = y[q];
}

// backward substitution, column task (large batches): thread per (element, column k of the level), one below
// block per round trip (D^2 + D loads per D^2 FMAs), the same two interleaved accumulators and order as
// bl_bsolve (identical results), L_kk^-T applied in registers
template <int D>
__global__ void __launch_bounds__(BL_TPB) bl_bsolve_ct(BLDev g, BLWs w, const int* cols, int ncol, const int* skip) {
  bl_pdl();
  using C = BLC<D>;
  int b;
  long long it;
  if (!bl_item(g, ncol, b, it)) return;
  if (b >= g.B || (skip && skip[b])) return;
  const size_t Bp = g.Bp;
  const int k = cols[it];
  double acc[2][D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    acc[0][c] = w.x[((size_t)k * D + c) * Bp + b];
    acc[1][c] = 0.0;
  }
  const int b0 = g.colptr[k] + 1, b1 = g.colptr[k + 1];
  for (int bi = b0; bi < b1; ++bi) {
    const int h = (bi - b0) & 1;
    const double* P0 = w.L + (size_t)bi * C::DD * Bp + b;
    const double* x0 = w.x + (size_t)g.blkrow[bi] * D * Bp + b;
    double l0[D][D], v0[D];
#pragma unroll
    for (int q = 0; q < D; ++q) {
      v0[q] = x0[q * Bp];
#pragma unroll
      for (int c = 0; c < D; ++c) l0[c][q] = P0[(c * D + q) * Bp];
    }
    bl_issue_fence();
    if (h == 0) {
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int q = 0; q < D; ++q) acc[0][c] = fma(-l0[c][q], v0[q], acc[0][c]);
    } else {
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int q = 0; q < D; ++q) acc[1][c] = fma(-l0[c][q], v0[q], acc[1][c]);
    }
  }
  const double* Lk = w.Ld + (size_t)k * C::DD * Bp + b;
  double y[D];
#pragma unroll
  for (int q = D - 1; q >= 0; --q) {
    double s2 = acc[0][q] + acc[1][q];
#pragma unroll
    for (int p = q + 1; p < D; ++p) s2 = fma(-Lk[(q * D + p) * Bp], y[p], s2);
    y[q] = s2 * Lk[ivpos<D>(0, q, D) * Bp];
  }
#pragma unroll
  for (int q = 0; q < D; ++q) w.x[((size_t)k * D + q) * Bp + b] = y[q];
}

// ---------------------------------------------------------------------------- retraction (a5)
template <int D>
__global__ void __launch_bounds__(BL_TPB) bl_retract(BLDev g, DevProb pr, BLWs w, double alpha) {
  bl_pdl();
  constexpr int PS = GT<D>::PS;
  int b;
  long long it;
  if (!bl_item(g, g.N, b, it)) return;
  if (b >= g.B || bl_frozen(w, b)) return;
  const int o = (int)it;
  const size_t Bp = g.Bp;
  const double* dl = w.x + (size_t)g.iperm[o] * D * Bp + b;
  double xi[D];
#pragma unroll
  for (int a = 0; a < D; ++a) xi[a] = -alpha * dl[a * Bp];
  double* T = pr.poses + ((size_t)b * g.N + o) * PS;
  if constexpr (D == 6) dev::se3_store(dev::se3_mul(dev::se3_load(T), dev::se3_exp(xi)), T);
  else dev::se2_store(dev::se2_mul(dev::se2_load(T), dev::se2_exp(xi)), T);
  if (o == 0) w.it[b] += 1;
}

__global__ void __launch_bounds__(BL_TPB) bl_init(BLDev g, BLWs w) {
  bl_pdl();
  const int b = blockIdx.x * BL_TPB + threadIdx.x;
  if (b >= g.Bp) return;
  w.st[b] = b < g.B ? DNLS_ST_OK : DNLS_ST_NOT_SPD;   // padding lanes stay frozen
  w.it[b] = 0;
  w.S[b] = 0.0;
  w.Sprev[b] = 0.0;
  w.maxd[b] = 0ull;
  w.fail[b] = 0;
}

// before the final (implicit) linearisation: keep the iteration status in ws_st, re-activate every element
__global__ void __launch_bounds__(BL_TPB) bl_pre_final(BLDev g, BLWs w) {
  bl_pdl();
  const int b = blockIdx.x * BL_TPB + threadIdx.x;
  if (b >= g.B) return;
  w.stf[b] = w.st[b];
  w.st[b] = DNLS_ST_OK;
}
// final status: a failed final (implicit) factor takes precedence; not-converged warning bit; outputs
__global__ void __launch_bounds__(BL_TPB) bl_finish(BLDev g, BLWs w, int implicit, double abs_tol, double rel_tol,
                                                    double* objective, int* status, int* iterations) {
  bl_pdl();
  const int b = blockIdx.x * BL_TPB + threadIdx.x;
  if (b >= g.B) return;
  int s = implicit ? w.stf[b] : w.st[b];
  if (implicit) {
    if (w.fail[b]) s = DNLS_ST_NOT_SPD;
    else if (w.it[b] > 0 && !(fabs(w.S[b] - w.Sprev[b]) < abs_tol + rel_tol * w.Sprev[b])) s |= DNLS_ST_WARN_NOT_CONVERGED;
  }
  if (objective) objective[b] = w.S[b];
  if (status) status[b] = s;
  if (iterations) iterations[b] = w.it[b];
  w.stf[b] = s;
  w.st[b] = s;
}

// objective at the final poses of an element without the implicit linearisation (S(theta_K)): per-slot
// costs, summed by bl_objective (final = 1)
template <int D>
__global__ void __launch_bounds__(BL_TPB) bl_cost_only(BLDev g, DevProb pr, BLWs w) {
  bl_pdl();
  int b;
  long long it;
  if (!bl_item(g, g.E + g.P, b, it)) return;
  if (b >= g.B) return;
  const int slot = (int)it;
  const DevGraph cg = bl_cost_graph(g);
  double c[D];
  eval_slot<D>(cg, pr, pr.poses + (size_t)b * g.N * GT<D>::PS, b, slot, c, nullptr, nullptr, false);
  const double wt = slot_weight<D>(cg, pr, b, slot);
  double n2 = 0.0;
#pragma unroll
  for (int q = 0; q < D; ++q) n2 += (wt * c[q]) * (wt * c[q]);
  double psi;
  w.cost[(size_t)slot * g.Bp + b] = slot_cost(cg, pr, b, slot, n2, psi);
}

// ---------------------------------------------------------------------------- implicit backward (a7 + a8)
template <int D>
__global__ void __launch_bounds__(BL_TPB) bl_bwd_rhs(BLDev g, DevProb pr, BLWs w, const double* gpose,
                                                     int grad_kind) {
  bl_pdl();
  int b;
  long long it;
  if (!bl_item(g, g.N, b, it)) return;
  if (b >= g.B) return;
  const int o = (int)it;
  double v[D];
  tangent_grad<D>(pr.poses + (size_t)b * g.N * GT<D>::PS, gpose, grad_kind, b, g.N, o, v);
  double* x = w.x + (size_t)g.iperm[o] * D * g.Bp + b;
#pragma unroll
  for (int a = 0; a < D; ++a) x[a * g.Bp] = v[a];
}
// per (element, slot): dL/dw = -2 w psi (1 - s/k^2) (C lambda).c (Prop. 1, readings A12 / W2); zero for
// elements without a valid factor
template <int D>
__global__ void __launch_bounds__(BL_TPB) bl_bwd_slots(BLDev g, DevProb pr, BLWs w, double* out) {
  bl_pdl();
  int b;
  long long it;
  if (!bl_item(g, g.E + g.P, b, it)) return;
  if (b >= g.B) return;
  const int slot = (int)it;
  const size_t Bp = g.Bp;
  if ((w.stf[b] & DNLS_ST_CODE_MASK) == DNLS_ST_NOT_SPD) {
    out[(size_t)slot * Bp + b] = 0.0;
    return;
  }
  const DevGraph cg = bl_cost_graph(g);
  const double* Tb = pr.poses + (size_t)b * g.N * GT<D>::PS;
  double c[D], Ci[D * D], Cj[D * D];
  eval_slot<D>(cg, pr, Tb, b, slot, c, Ci, Cj, true);
  const double wt = slot_weight<D>(cg, pr, b, slot);
  const bool edge = slot < g.E;
  const int vi = edge ? g.edges[2 * slot] : g.prior_vars[slot - g.E];
  const double* li = w.x + (size_t)g.iperm[vi] * D * Bp + b;
  const double* lj = edge ? w.x + (size_t)g.iperm[g.edges[2 * slot + 1]] * D * Bp + b : li;
  double lv[D], lw[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    lv[a] = li[a * Bp];
    lw[a] = lj[a * Bp];
  }
  double dot = 0.0, n2 = 0.0;
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double cl = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) {
      cl = fma(Ci[r * D + q], lv[q], cl);
      if (edge) cl = fma(Cj[r * D + q], lw[q], cl);
    }
    dot = fma(cl, c[r], dot);
    n2 = fma(c[r], c[r], n2);
  }
  double psi;
  const double sq = wt * wt * n2;
  slot_cost(cg, pr, b, slot, sq, psi);
  double fw = 1.0;
  if (pr.radius != nullptr && edge) {
    const double k = pr.radius[(size_t)b * pr.r_bstride];
    fw = psi * (1.0 - sq / (k * k));
  }
  out[(size_t)slot * Bp + b] = -2.0 * wt * fw * dot;
}
// fixed-order batch reduction (or per-element copy) of the interleaved per-slot gradients: one warp per slot,
// lane l sums elements l, l + 32, ... in order, then a fixed xor-shuffle tree (deterministic)
__global__ void bl_reduce_wgrad(int B, int Bp, int E, int P, const double* src, double* ge, double* gp, long long bstride) {
  bl_pdl();
  const int slot = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (slot >= E + P) return;
  double* dst = slot < E ? ge : gp;
  const int idx = slot < E ? slot : slot - E;
  if (!dst) return;
  const double* s = src + (size_t)slot * Bp;
  if (bstride == 0) {
    double acc = 0.0;
    for (int b = lane; b < B; b += 32) acc += s[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) dst[idx] = acc;
  } else {
    for (int b = lane; b < B; b += 32) dst[(size_t)b * bstride + idx] = s[b];
  }
}

// ============================================================================ host plan
struct BLPlan {
  int D = 0, N = 0, E = 0, P = 0, nblk = 0, L = 0;
  int* dbuf = nullptr;
  BLDev dev{};
  // host copies of the level schedule (launch sizes)
  std::vector<int> lvl_ptr, tsk_lvl_ptr, fac_lvl_ptr;
  const int* d_lvl_col = nullptr;
  const int* d_fill0 = nullptr;   // fill blocks without an update task
  int nfill0 = 0;
  int upd = -1;         // update kernel below the persistent levels: -1 automatic, 0 row-split, 1 register-blocked
  int persist = -1;     // bl_persist group width (-1 automatic, 0: per-level bl_update* + bl_factor launches)
  int persist_from = -1; // first level of the persistent launch (-1: the single-column tail of the tree)
  int solve_from = -1;    // first level of the persistent tail solves (-1: as the factorisation's split)
  std::vector<int> facf_lvl_ptr;   // per level: factor items of the columns outside the subtrees
  const int4 *d_facf = nullptr, *d_facr = nullptr;
  int lsolve = 1;         // persistent tail solves: 1 level-parallel bl_lsolve, 0 bl_persist_solve (DNLS_BL_LSOLVE)
  BLSDev sd{};
  std::vector<int> bit_lvl_h, fit_lvl_h;   // host copies: items per level of bl_lsolve
  int tail_from = 0;      // first level of the single-column tail
  int narrow_from = 0;    // first level of the narrow top (every level above has <= 6 columns)
  int bsolve_ct = 16;     // column-task backward solve on levels with >= this many columns (0: off)
  int lch = 0;            // per-level chunked update (bl_update_items + bl_factor_red): chunk size (0: off)
  std::vector<int> lit_lvl_ptr;   // per level: its chunked work items
  const int4* d_litems = nullptr;
  const int2 *d_bred = nullptr, *d_cred = nullptr;
  // filtered variant (with bl_subtree): per-level items / reductions of the columns outside the subtrees
  std::vector<int> litf_lvl_ptr;
  const int4* d_litems_f = nullptr;
  const int2 *d_bred_f = nullptr, *d_cred_f = nullptr;
  int sub_top = -1;       // bl_subtree covers the columns of height <= sub_top (-1: off)
  std::vector<int> sub_pass;   // subtrees of pass p: [sub_pass[p], sub_pass[p+1])
  int nsub = 0;           // its items: maximal subtrees of those columns, largest first
  const int* d_sub_ptr = nullptr;
  const int4* d_sub_rec = nullptr;

  BLPDev pd{};
  int64_t storage_doubles = 0;   // nblk * DD per element
  ~BLPlan() {
    if (dbuf) cudaFree(dbuf);
  }
};

// symbolic data of the pose-level block factorisation from the graph's ordering (perm, column structures)
inline std::string bl_build(const Symbolic& s, int device, BLPlan& pl) {
  const int N = s.N, D = s.D;
  pl.D = D;
  pl.N = N;
  pl.E = s.E;
  pl.P = s.P;
  std::vector<int32_t> colptr(N + 1, 0), blkrow;
  for (int k = 0; k < N; ++k) {
    colptr[k] = (int)blkrow.size();
    blkrow.push_back(k);
    for (int p : s.colstruct[k]) blkrow.push_back(p);
  }
  colptr[N] = (int)blkrow.size();
  pl.nblk = colptr[N];
  pl.storage_doubles = (int64_t)pl.nblk * D * D;
  auto blk = [&](int p, int k) -> int {   // block (p, k), p >= k
    if (p == k) return colptr[k];
    const auto& R = s.colstruct[k];
    auto it = std::lower_bound(R.begin(), R.end(), p);
    if (it == R.end() || *it != p) return -1;
    return colptr[k] + 1 + (int)(it - R.begin());
  };
  // levels: height in the pose-level elimination tree
  std::vector<int> h(N, 0);
  for (int k = 0; k < N; ++k)
    if (s.parent[k] >= 0) h[s.parent[k]] = std::max(h[s.parent[k]], h[k] + 1);
  int L = 0;
  for (int k = 0; k < N; ++k) L = std::max(L, h[k] + 1);
  pl.L = L;
  pl.lvl_ptr.assign(L + 1, 0);
  for (int k = 0; k < N; ++k) pl.lvl_ptr[h[k] + 1]++;
  for (int l = 0; l < L; ++l) pl.lvl_ptr[l + 1] += pl.lvl_ptr[l];
  std::vector<int32_t> lvl_col(N);
  {
    std::vector<int> fillp(pl.lvl_ptr.begin(), pl.lvl_ptr.end() - 1);
    for (int k = 0; k < N; ++k) lvl_col[fillp[h[k]]++] = k;
  }
  // update tasks: target (p, k) for p in {k} U cs[k]; contributions from every s with k, p in cs[s]
  // bottom subtrees: the columns of height <= sub_top (no height bound by default) whose subtree work is bounded
  // are factored by bl_subtree, below
  int sub_top = 1 << 20;
  if (const char* env = std::getenv("DNLS_BL_SUB")) sub_top = std::atoi(env);
  sub_top = std::min(sub_top, L - 1);
  std::vector<std::vector<int2>> tcon(pl.nblk);
  std::vector<std::vector<int2>> fwdl(N);
  for (int sc = 0; sc < N; ++sc) {
    const auto& R = s.colstruct[sc];
    for (size_t iq = 0; iq < R.size(); ++iq) {
      const int k = R[iq];
      fwdl[k].push_back(make_int2(blk(k, sc), sc));
      for (size_t ip = iq; ip < R.size(); ++ip) {
        const int p = R[ip];
        tcon[blk(p, k)].push_back(make_int2(blk(p, sc), blk(k, sc)));
      }
    }
  }
  std::vector<int32_t> tsk, con, fwdp(N + 1, 0), fwd, fac;
  pl.tsk_lvl_ptr.assign(L + 1, 0);
  pl.fac_lvl_ptr.assign(L + 1, 0);
  int ntask = 0, nfac = 0;
  for (int l = 0; l < L; ++l) {
    for (int i = pl.lvl_ptr[l]; i < pl.lvl_ptr[l + 1]; ++i) {
      const int k = lvl_col[i];
      for (int bi = colptr[k]; bi < colptr[k + 1]; ++bi) {
        fac.push_back(k);
        fac.push_back(bi);
        ++nfac;
        if (tcon[bi].empty()) continue;
        tsk.push_back(bi);
        tsk.push_back((int)con.size() / 2);
        for (const int2& c : tcon[bi]) {
          con.push_back(c.x);
          con.push_back(c.y);
        }
        tsk.push_back((int)con.size() / 2);
        tsk.push_back(bi == colptr[k] ? 1 : 0);
        ++ntask;
      }
    }
    pl.tsk_lvl_ptr[l + 1] = ntask;
    pl.fac_lvl_ptr[l + 1] = nfac;
  }
  for (int k = 0; k < N; ++k) {
    fwdp[k] = (int)fwd.size() / 2;
    for (const int2& f : fwdl[k]) {
      fwd.push_back(f.x);
      fwd.push_back(f.y);
    }
  }
  fwdp[N] = (int)fwd.size() / 2;
  // assembly: per slot its off-diagonal block, orientation, unique flag; shared blocks; fill blocks
  const int slots = s.E + s.P;
  std::vector<int32_t> slotd(4 * (size_t)slots, 0);
  std::map<int, std::vector<int>> shared;
  std::vector<char> written(pl.nblk, 0);
  for (int k = 0; k < N; ++k) written[colptr[k]] = 1;
  std::map<std::pair<int, int>, int> pair_count;
  for (int e = 0; e < s.E; ++e) {
    const int pi = s.iperm[s.edges[2 * e]], pj = s.iperm[s.edges[2 * e + 1]];
    pair_count[std::make_pair(std::min(pi, pj), std::max(pi, pj))]++;
  }
  for (int e = 0; e < s.E; ++e) {
    const int pi = s.iperm[s.edges[2 * e]], pj = s.iperm[s.edges[2 * e + 1]];
    const int Pp = std::max(pi, pj), Q = std::min(pi, pj);
    const int bidx = blk(Pp, Q);
    if (bidx < 0) return "bl_build: edge block missing from the factor pattern";
    const bool uniq = pair_count[std::make_pair(Q, Pp)] == 1;
    slotd[4 * e] = bidx;
    slotd[4 * e + 1] = Pp == pj ? 1 : 0;
    slotd[4 * e + 2] = uniq ? 1 : 0;
    written[bidx] = 1;
    if (!uniq) shared[bidx].push_back(e);
  }
  for (int k = 0; k < s.P; ++k) slotd[4 * (s.E + k)] = -1;
  std::vector<int32_t> dup_ptr(1, 0), dup_blk, dup_con, fill;
  for (auto& kv : shared) {
    dup_blk.push_back(kv.first);
    for (int e : kv.second) dup_con.push_back(e);
    dup_ptr.push_back((int)dup_con.size());
  }
  // fill blocks (no cost writes them): targets of an update task are flagged (tk.w bit 1) -- the
  // register-blocked update stores -acc there -- the others (none for a well-formed pattern) are zeroed
  std::vector<char> tasked(pl.nblk, 0);
  for (size_t t = 0; t < tsk.size(); t += 4) {
    tasked[tsk[t]] = 1;
    if (!written[tsk[t]]) tsk[t + 3] |= 2;
  }
  std::vector<int32_t> fill0;
  for (int bi = 0; bi < pl.nblk; ++bi)
    if (!written[bi]) {
      fill.push_back(bi);
      if (!tasked[bi]) fill0.push_back(bi);
    }
  // persistent factorisation (bl_persist): per block its contribution range and flags; per narrow level its
  // work items -- contribution lists longer than the level's chunk size split into chunks with a partial slot
  // each (level-wide numbering; the partials live in the slot scratch, so the split is disabled where it would
  // not fit) -- and the split reductions.  Chunk size: the level's contributions spread over ~2 items per unit
  // of a CTA (16 units), at least 2 contributions per chunk.
  std::vector<int32_t> bcon(4 * (size_t)pl.nblk, 0);
  for (size_t t = 0; t < tsk.size(); t += 4) {
    bcon[4 * (size_t)tsk[t]] = tsk[t + 1];
    bcon[4 * (size_t)tsk[t] + 1] = tsk[t + 2];
    bcon[4 * (size_t)tsk[t] + 2] = tsk[t + 3];
  }
  int ch_units = 16, ch_min = 2;
  if (const char* env = std::getenv("DNLS_BL_CH")) sscanf(env, "%d,%d", &ch_units, &ch_min);
  const size_t scr_doubles = (size_t)(s.E + s.P) * (D == 6 ? BLC<6>::SW : BLC<3>::SW);
  std::vector<int32_t> it_lvl(L + 1, 0), items, rd_lvl(L + 1, 0), red;
  for (int l = 0; l < L; ++l) {
    int nc = 0;
    for (int i = pl.lvl_ptr[l]; i < pl.lvl_ptr[l + 1]; ++i) {
      const int k = lvl_col[i];
      for (int bi = colptr[k]; bi < colptr[k + 1]; ++bi) nc += bcon[4 * (size_t)bi + 1] - bcon[4 * (size_t)bi];
      nc += fwdp[k + 1] - fwdp[k];
    }
    int ch = std::max(ch_min, (nc + ch_units - 1) / ch_units);
    for (int pass = 0; pass < 2; ++pass) {   // pass 1 without splitting if the partials do not fit
      int nslot = 0;
      std::vector<int32_t> it_l, rd_l;
      auto add_item = [&](int tgt, int c0, int c1, int flags) {
        const int n = c1 - c0, S = (n + ch - 1) / ch;
        if (S <= 1) {
          it_l.insert(it_l.end(), {tgt, c0, c1, flags});
          return;
        }
        rd_l.insert(rd_l.end(), {tgt, nslot, S, flags});
        for (int q = 0; q < S; ++q) {
          const int a = c0 + (int)((int64_t)n * q / S), e = c0 + (int)((int64_t)n * (q + 1) / S);
          it_l.insert(it_l.end(), {tgt, a, e, flags | ((nslot + 1) << 8)});
          ++nslot;
        }
      };
      for (int i = pl.lvl_ptr[l]; i < pl.lvl_ptr[l + 1]; ++i) {
        const int k = lvl_col[i];
        for (int bi = colptr[k]; bi < colptr[k + 1]; ++bi)
          if (bcon[4 * (size_t)bi + 1] > bcon[4 * (size_t)bi])
            add_item(bi, bcon[4 * (size_t)bi], bcon[4 * (size_t)bi + 1], bcon[4 * (size_t)bi + 2] & 3);
        if (fwdp[k + 1] > fwdp[k]) add_item(-2 - k, fwdp[k], fwdp[k + 1], 0);
      }
      if (pass == 0 && (size_t)nslot * D * D > scr_doubles) {
        ch = 1 << 30;
        continue;
      }
      items.insert(items.end(), it_l.begin(), it_l.end());
      red.insert(red.end(), rd_l.begin(), rd_l.end());
      break;
    }
    it_lvl[l + 1] = (int)items.size() / 4;
    rd_lvl[l + 1] = (int)red.size() / 4;
  }
  // bottom subtrees (bl_subtree): a column is in a subtree when its height is <= sub_top and the work of the
  // subtree rooted at it -- memory round trips of its column tasks: contributions + forward contributions + blocks --
  // is <= subw (the longest thread chain of the kernel bounds it: uncapped, C5's largest subtree is 539 round
  // trips against a mean of 91).  Eligibility is closed under descendants; a subtree is rooted at an eligible
  // column whose parent is not eligible.  Its columns in increasing index (children first), subtrees by decreasing
  // work.  The other columns (in_sub = 0) are factored by the per-level launches.
  // passes: pass p groups the columns not taken by earlier passes whose residual subtree work (their own column
  // task plus that of their untaken descendants) is <= cap p; one bl_subtree launch per pass, in pass order (a
  // pass's subtree contains every untaken descendant of its root, so earlier passes hold the rest)
  std::vector<int> subw = {400};   // measured at C5 (profiles/r3/): uncapped 2.34 ms, 80: 2.29, 160: 2.26,
                                   // 240-400: 2.22-2.23, 600: 2.25
  if (const char* env = std::getenv("DNLS_BL_SUBW")) {
    subw.clear();
    for (const char* c = env; *c;) {
      subw.push_back(std::atoi(c));
      while (*c && *c != ',') ++c;
      if (*c == ',') ++c;
    }
  }
  std::vector<int32_t> sub_ptr(1, 0), sub_col;
  pl.sub_pass.assign(1, 0);
  std::vector<char> in_sub(N, 0);
  if (sub_top >= 0) {
    std::vector<long long> wk(N, 0);
    for (int k = 0; k < N; ++k) {
      wk[k] = (colptr[k + 1] - colptr[k]) + (fwdp[k + 1] - fwdp[k]);
      for (int bi = colptr[k]; bi < colptr[k + 1]; ++bi) wk[k] += bcon[4 * (size_t)bi + 1] - bcon[4 * (size_t)bi];
    }
    for (int cap : subw) {
      std::vector<long long> W(N, 0);
      for (int k = 0; k < N; ++k) {
        if (in_sub[k]) continue;
        W[k] += wk[k];
        if (s.parent[k] >= 0) W[s.parent[k]] += W[k];
      }
      auto elig = [&](int k) { return !in_sub[k] && h[k] <= sub_top && (cap <= 0 || W[k] <= cap); };
      std::vector<int> root(N, -1);
      for (int k = N - 1; k >= 0; --k)
        if (elig(k)) root[k] = (s.parent[k] >= 0 && elig(s.parent[k])) ? root[s.parent[k]] : k;
      std::map<int, std::vector<int>> subs;
      for (int k = 0; k < N; ++k)
        if (root[k] >= 0) subs[root[k]].push_back(k);
      for (auto& kv : subs)
        for (int k : kv.second) in_sub[k] = 1;
      std::vector<std::pair<long long, int>> order;   // (-work, root)
      for (auto& kv : subs) order.push_back(std::make_pair(-W[kv.first], kv.first));
      std::sort(order.begin(), order.end());
      for (auto& o : order) {
        for (int k : subs[o.second]) sub_col.push_back(k);
        sub_ptr.push_back((int)sub_col.size());
      }
      pl.sub_pass.push_back((int)sub_ptr.size() - 1);
    }
  }
  // per-level chunked update (large-batch schedule): every level's target lists and forward rows as work items,
  // lists longer than lch contributions split into ceil(n / lch) nearly equal chunks; the first chunk is applied
  // in place, the others store partials (level-local slots in the slot scratch) that bl_factor_red subtracts in
  // chunk order.  bred / cred: per block / column (first slot, count) of its partials.
  int lch = 8;
  if (const char* env = std::getenv("DNLS_BL_LCH")) lch = std::atoi(env);
  std::vector<int32_t> litems, bred(2 * (size_t)pl.nblk, 0), cred(2 * (size_t)N, 0);
  std::vector<int32_t> litems_f, bred_f(2 * (size_t)pl.nblk, 0), cred_f(2 * (size_t)N, 0);
  pl.lit_lvl_ptr.assign(L + 1, 0);
  pl.litf_lvl_ptr.assign(L + 1, 0);
  int litems_want = 0, lch_min = 2;   // narrow levels: chunks small enough for ~litems_want items (0: off)
  if (const char* env = std::getenv("DNLS_BL_LITEMS")) sscanf(env, "%d,%d", &litems_want, &lch_min);
  // filtered variant: without the columns of the bottom subtrees (factored by bl_subtree)
  for (int var = 0; var < 2 && lch > 0; ++var) {
    const bool fv = var == 1;
    std::vector<int32_t>& litv = fv ? litems_f : litems;
    std::vector<int32_t>& bredv = fv ? bred_f : bred;
    std::vector<int32_t>& credv = fv ? cred_f : cred;
    std::vector<int>& lptr = fv ? pl.litf_lvl_ptr : pl.lit_lvl_ptr;
    const size_t cap = scr_doubles / ((size_t)D * D);
    for (int l = 0; l < L; ++l) {
      int nslot = 0, ncl = 0;
      for (int i = pl.lvl_ptr[l]; i < pl.lvl_ptr[l + 1]; ++i) {
        const int k = lvl_col[i];
        for (int bi = colptr[k]; bi < colptr[k + 1]; ++bi) ncl += bcon[4 * (size_t)bi + 1] - bcon[4 * (size_t)bi];
        ncl += fwdp[k + 1] - fwdp[k];
      }
      const int lchl = litems_want > 0 ? std::max(lch_min, std::min(lch, (ncl + litems_want - 1) / litems_want)) : lch;
      auto add = [&](int tgt, int c0, int c1, int flags, int32_t* red2) {
        const int n = c1 - c0;
        int S = (n + lchl - 1) / lchl;
        if ((size_t)(nslot + S - 1) > cap) S = 1;   // partials would not fit: whole list in place
        if (S <= 1) {
          litv.insert(litv.end(), {tgt, c0, c1, flags});
          return;
        }
        red2[0] = nslot;
        red2[1] = S - 1;
        for (int q = 0; q < S; ++q) {
          const int a = c0 + (int)((int64_t)n * q / S), e = c0 + (int)((int64_t)n * (q + 1) / S);
          litv.insert(litv.end(), {tgt, a, e, flags | (q == 0 ? 0 : ((nslot + 1) << 8))});
          if (q > 0) ++nslot;
        }
      };
      for (int i = pl.lvl_ptr[l]; i < pl.lvl_ptr[l + 1]; ++i) {
        const int k = lvl_col[i];
        if (fv && in_sub[k]) continue;   // factored by bl_subtree
        for (int bi = colptr[k]; bi < colptr[k + 1]; ++bi) {
          const int a = bcon[4 * (size_t)bi], e = bcon[4 * (size_t)bi + 1];
          if (e > a) add(bi, a, e, bcon[4 * (size_t)bi + 2] & 3, &bredv[2 * (size_t)bi]);
        }
        if (fwdp[k + 1] > fwdp[k]) add(-2 - k, fwdp[k], fwdp[k + 1], 0, &credv[2 * (size_t)k]);
      }
      lptr[l + 1] = (int)litv.size() / 4;
    }
  }
  // the per-level factor items of the columns outside the subtrees (chunked schedule)
  // (records (column, block, diagonal block of the column, 0) for bl_factor_red; facr: every column, same order
  // as fac / fac_lvl_ptr)
  std::vector<int32_t> facf, facr;
  pl.facf_lvl_ptr.assign(L + 1, 0);
  for (int l = 0; l < L; ++l) {
    for (int i = pl.lvl_ptr[l]; i < pl.lvl_ptr[l + 1]; ++i) {
      const int k = lvl_col[i];
      for (int bi = colptr[k]; bi < colptr[k + 1]; ++bi) {
        facr.insert(facr.end(), {k, bi, colptr[k], 0});
        if (!in_sub[k]) facf.insert(facf.end(), {k, bi, colptr[k], 0});
      }
    }
    pl.facf_lvl_ptr[l + 1] = (int)facf.size() / 4;
  }
  // bl_lsolve items: per level, per column (in lvl_col order) its below blocks (backward) / forward contributions
  std::vector<int32_t> bit, fit, bcolv(2 * (size_t)N, 0), fcolv(2 * (size_t)N, 0);
  pl.bit_lvl_h.assign(L + 1, 0);
  pl.fit_lvl_h.assign(L + 1, 0);
  for (int l = 0; l < L; ++l) {
    for (int i = pl.lvl_ptr[l]; i < pl.lvl_ptr[l + 1]; ++i) {
      const int k = lvl_col[i];
      bcolv[2 * (size_t)i] = (int)bit.size() / 2;
      bcolv[2 * (size_t)i + 1] = colptr[k + 1] - colptr[k] - 1;
      for (int bi = colptr[k] + 1; bi < colptr[k + 1]; ++bi) bit.insert(bit.end(), {i, bi});
      fcolv[2 * (size_t)i] = (int)fit.size() / 2;
      fcolv[2 * (size_t)i + 1] = fwdp[k + 1] - fwdp[k];
      for (int q = fwdp[k]; q < fwdp[k + 1]; ++q) fit.insert(fit.end(), {i, q});
    }
    pl.bit_lvl_h[l + 1] = (int)bit.size() / 2;
    pl.fit_lvl_h[l + 1] = (int)fit.size() / 2;
  }
  std::vector<int32_t> bit_lvl32(pl.bit_lvl_h.begin(), pl.bit_lvl_h.end()), fit_lvl32(pl.fit_lvl_h.begin(),
                                                                                       pl.fit_lvl_h.end());
  pl.lch = lch;
  std::vector<int32_t> sub_rec;   // per subtree column: (k, first block, end block, forward begin), (forward end,
                                  // diagonal contributions begin, end, 0)
  for (int k : sub_col)
    sub_rec.insert(sub_rec.end(), {k, colptr[k], colptr[k + 1], fwdp[k], fwdp[k + 1], bcon[4 * (size_t)colptr[k]],
                                   bcon[4 * (size_t)colptr[k] + 1], 0});
  pl.sub_top = sub_top;
  pl.nsub = (int)sub_ptr.size() - 1;
  std::vector<int32_t> lvl_ptr32(pl.lvl_ptr.begin(), pl.lvl_ptr.end()), fac_lvl32(pl.fac_lvl_ptr.begin(),
                                                                                   pl.fac_lvl_ptr.end());
  // upload (int32 arrays, 16-byte aligned)
  std::vector<int32_t> buf;
  std::vector<size_t> offs;
  auto add = [&](const std::vector<int32_t>& v) {
    while (buf.size() % 4) buf.push_back(0);
    offs.push_back(buf.size());
    buf.insert(buf.end(), v.begin(), v.end());
    buf.push_back(0);
  };
  add(s.perm); add(s.iperm); add(s.edges); add(s.prior_vars);
  add(colptr); add(blkrow); add(tsk); add(con); add(fwdp); add(fwd); add(fac); add(slotd);
  add(s.bc_ptr); add(s.bc); add(dup_ptr); add(dup_blk); add(dup_con); add(fill); add(lvl_col); add(fill0);
  add(bcon); add(it_lvl); add(items); add(rd_lvl); add(red); add(lvl_ptr32); add(fac_lvl32);
  add(sub_ptr); add(sub_rec);
  add(litems); add(bred); add(cred);
  add(litems_f); add(bred_f); add(cred_f);
  add(bit); add(bit_lvl32); add(bcolv); add(fit); add(fit_lvl32); add(fcolv);
  add(facf); add(facr);
  while (buf.size() % 4) buf.push_back(0);
  if (device >= 0) {
    if (cudaMalloc(&pl.dbuf, buf.size() * sizeof(int32_t)) != cudaSuccess ||
        cudaMemcpy(pl.dbuf, buf.data(), buf.size() * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaGetLastError();
      return "bl_build: device upload failed";
    }
  }
  const int* d = pl.dbuf;
  int k = 0;
  BLDev& g = pl.dev;
  g.D = D; g.N = N; g.E = s.E; g.P = s.P; g.n = N * D; g.nblk = pl.nblk;
  auto ptr = [&](size_t o) { return d ? d + o : nullptr; };
  g.perm = ptr(offs[k++]); g.iperm = ptr(offs[k++]); g.edges = ptr(offs[k++]); g.prior_vars = ptr(offs[k++]);
  g.colptr = ptr(offs[k++]); g.blkrow = ptr(offs[k++]);
  g.tsk = reinterpret_cast<const int4*>(ptr(offs[k++]));
  g.con = reinterpret_cast<const int2*>(ptr(offs[k++]));
  g.fwdp = ptr(offs[k++]);
  g.fwd = reinterpret_cast<const int2*>(ptr(offs[k++]));
  g.fac = reinterpret_cast<const int2*>(ptr(offs[k++]));
  g.slotd = reinterpret_cast<const int4*>(ptr(offs[k++]));
  g.bc_ptr = ptr(offs[k++]); g.bc = ptr(offs[k++]);
  g.dup_ptr = ptr(offs[k++]); g.dup_blk = ptr(offs[k++]); g.dup_con = ptr(offs[k++]);
  g.fill = ptr(offs[k++]);
  pl.d_lvl_col = ptr(offs[k++]);
  pl.d_fill0 = ptr(offs[k++]);
  pl.nfill0 = (int)fill0.size();
  pl.pd.bcon = reinterpret_cast<const int4*>(ptr(offs[k++]));
  pl.pd.it_lvl = ptr(offs[k++]);
  pl.pd.items = reinterpret_cast<const int4*>(ptr(offs[k++]));
  pl.pd.rd_lvl = ptr(offs[k++]);
  pl.pd.red = reinterpret_cast<const int4*>(ptr(offs[k++]));
  pl.pd.lvl_ptr = ptr(offs[k++]);
  pl.pd.fac_lvl = ptr(offs[k++]);
  pl.d_sub_ptr = ptr(offs[k++]);
  pl.d_sub_rec = reinterpret_cast<const int4*>(ptr(offs[k++]));
  pl.d_litems = reinterpret_cast<const int4*>(ptr(offs[k++]));
  pl.d_bred = reinterpret_cast<const int2*>(ptr(offs[k++]));
  pl.d_cred = reinterpret_cast<const int2*>(ptr(offs[k++]));
  pl.d_litems_f = reinterpret_cast<const int4*>(ptr(offs[k++]));
  pl.d_bred_f = reinterpret_cast<const int2*>(ptr(offs[k++]));
  pl.d_cred_f = reinterpret_cast<const int2*>(ptr(offs[k++]));
  pl.sd.bit = reinterpret_cast<const int2*>(ptr(offs[k++]));
  pl.sd.bit_lvl = ptr(offs[k++]);
  pl.sd.bcol = reinterpret_cast<const int2*>(ptr(offs[k++]));
  pl.sd.fit = reinterpret_cast<const int2*>(ptr(offs[k++]));
  pl.sd.fit_lvl = ptr(offs[k++]);
  pl.sd.fcol = reinterpret_cast<const int2*>(ptr(offs[k++]));
  if (const char* env = std::getenv("DNLS_BL_LSOLVE")) pl.lsolve = std::atoi(env);
  pl.d_facf = reinterpret_cast<const int4*>(ptr(offs[k++]));
  pl.d_facr = reinterpret_cast<const int4*>(ptr(offs[k++]));
  pl.pd.lvl_col = pl.d_lvl_col;
  pl.pd.L = L;
  pl.pd.coltask_min = 16;
  if (const char* env = std::getenv("DNLS_BL_COLTASK")) pl.pd.coltask_min = std::atoi(env);
  if (const char* env = std::getenv("DNLS_BL_PERSIST")) pl.persist = std::atoi(env);
  if (const char* env = std::getenv("DNLS_BL_GMAJOR")) g.gmajor = std::atoi(env);
  if (const char* env = std::getenv("DNLS_BL_SPLIT")) pl.persist_from = std::atoi(env);
  if (const char* env = std::getenv("DNLS_BL_SSPLIT")) pl.solve_from = std::atoi(env);

  if (const char* env = std::getenv("DNLS_BL_UPD")) pl.upd = std::atoi(env);
  if (const char* env = std::getenv("DNLS_BL_BSCT")) pl.bsolve_ct = std::atoi(env);
  pl.tail_from = L;
  while (pl.tail_from > 0 && pl.lvl_ptr[pl.tail_from] - pl.lvl_ptr[pl.tail_from - 1] == 1) --pl.tail_from;
  // level-parallel tail solves (bl_lsolve) from the first level above which every level has <= 6 columns
  pl.narrow_from = L;
  while (pl.narrow_from > 0 && pl.lvl_ptr[pl.narrow_from] - pl.lvl_ptr[pl.narrow_from - 1] <= 6) --pl.narrow_from;
  g.nfill = (int)fill.size();
  g.ndup = (int)dup_blk.size();
  return std::string();
}

inline int bl_pad(int B) { return (B + 31) / 32 * 32; }

struct BLLayout {
  size_t L, Ld, x, scr, cost, S, Sprev, maxd, fail, st, it, stf, total;
};
inline BLLayout bl_layout_sizes(int D, int N, int E, int P, int64_t nblk, int B) {
  const int Bp = bl_pad(B);
  const size_t slots = (size_t)E + P, SW = D == 6 ? BLC<6>::SW : BLC<3>::SW;
  const int64_t storage_doubles = nblk * D * D;
  BLLayout l{};
  size_t o = 0;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  l.L = o;     o = al(o + sizeof(double) * (size_t)storage_doubles * Bp);
  l.Ld = o;    o = al(o + sizeof(double) * (size_t)N * D * D * Bp);
  l.x = o;     o = al(o + sizeof(double) * (size_t)N * D * Bp);
  l.scr = o;   o = al(o + sizeof(double) * slots * SW * Bp);
  l.cost = o;  o = al(o + sizeof(double) * slots * Bp);
  l.S = o;     o = al(o + sizeof(double) * Bp);
  l.Sprev = o; o = al(o + sizeof(double) * Bp);
  l.maxd = o;  o = al(o + sizeof(double) * Bp);
  l.fail = o;  o = al(o + sizeof(int) * Bp);
  l.st = o;    o = al(o + sizeof(int) * Bp);
  l.it = o;    o = al(o + sizeof(int) * Bp);
  l.stf = o;   o = al(o + sizeof(int) * Bp);
  l.total = o;
  return l;
}
inline BLLayout bl_layout(const BLPlan& pl, int B) { return bl_layout_sizes(pl.D, pl.N, pl.E, pl.P, pl.nblk, B); }
inline BLWs bl_views(const BLLayout& l, void* base) {
  char* p = (char*)base;
  BLWs w;
  w.L = (double*)(p + l.L);
  w.Ld = (double*)(p + l.Ld);
  w.x = (double*)(p + l.x);
  w.scr = (double*)(p + l.scr);
  w.cost = (double*)(p + l.cost);
  w.S = (double*)(p + l.S);
  w.Sprev = (double*)(p + l.Sprev);
  w.maxd = (unsigned long long*)(p + l.maxd);
  w.fail = (int*)(p + l.fail);
  w.st = (int*)(p + l.st);
  w.it = (int*)(p + l.it);
  w.stf = (int*)(p + l.stf);
  return w;
}

inline unsigned bl_grid(long long items, int Bp) { return (unsigned)((items * Bp + BL_TPB - 1) / BL_TPB); }
inline unsigned bl_grid_b(int n) { return (unsigned)((n + BL_TPB - 1) / BL_TPB); }

// phase timing for the factor-kernel roofline (bench): events around each factorisation when enabled
struct BLPhaseTimer {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  void begin(cudaStream_t s) {
    if (!on) return;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    ev.push_back(std::make_pair(a, b));
  }
  void end(cudaStream_t s) {
    if (on) cudaEventRecord(ev.back().second, s);
  }
};

// linearise + assemble at the current poses (lam > 0: damping), objective into w.S
// launch schedule of a factorisation for a batch (measured, profiles/r2_factor_experiments): with >= 1024
// elements (32 warp groups) every (target, element) thread of the register-blocked update has enough company
// to cover the memory latency and the single-column tail of the tree runs in one persistent launch (group
// width: the widest of 16 / 8 / 4 elements giving >= 128 CTAs); smaller batches use the row-split update
// (6 warps per target) for every level.  Environment overrides: DNLS_BL_UPD, DNLS_BL_PERSIST, DNLS_BL_SPLIT.
struct BLSched {
  bool rb;
  int lsplit, gw;
  bool sub;     // bl_subtree for the bottom subtrees (with the chunked per-level schedule)
  int fsplit;   // first level of the factorisation's persistent launch (chunked per-level items: none)
  int sgw;      // bl_lsolve group width
};
inline BLSched bl_schedule(const BLPlan& pl, int B) {
  const bool large = bl_pad(B) / 32 >= 8;
  BLSched sc;
  sc.rb = pl.upd >= 0 ? pl.upd != 0 : large;
  const bool persist = pl.persist == 0 ? false : (pl.persist > 0 || large);
  sc.lsplit = !persist ? pl.L : (pl.persist_from >= 0 ? std::min(pl.L, pl.persist_from) : pl.tail_from);
  sc.gw = pl.persist > 0 ? pl.persist : ((B + 15) / 16 >= 128 ? 16 : (B + 7) / 8 >= 128 ? 8 : 4);
  // bl_lsolve group width: 8 elements per CTA when that still gives >= 148 CTAs (C5: 256 CTAs), else 4
  sc.sgw = pl.persist > 0 ? pl.persist : ((B + 7) / 8 >= 148 ? 8 : 4);
  if (pl.solve_from >= 0)
    sc.lsplit = std::min(pl.L, pl.solve_from);
  else if (persist && pl.lsolve && pl.persist_from < 0)
    sc.lsplit = pl.narrow_from;   // bl_lsolve: the narrow top of the tree (measured: C5 ss20 / gw 8 best)
  sc.fsplit = (sc.rb && pl.lch > 0 && pl.persist_from < 0) ? pl.L : sc.lsplit;
  sc.sub = pl.sub_top >= 0 && pl.nsub > 0 && sc.rb && pl.lch > 0;
  return sc;
}

template <int D>
void bl_linearize(const BLPlan& pl, int B, const DevProb& pr, const BLWs& w, double lam, int damping, cudaStream_t s) {
  BLDev g = pl.dev;
  g.B = B;
  g.Bp = bl_pad(B);
  bl_launch(bl_reset_iter, bl_grid_b(g.Bp), BL_TPB, s, g, w);
  // the register-blocked update stores its fill targets; the row-split one accumulates into zeroed blocks
  const BLSched sc = bl_schedule(pl, B);
  const bool zero_all = !sc.rb && sc.lsplit > 0;
  const int* fl = zero_all ? g.fill : pl.d_fill0;
  const int nf = zero_all ? g.nfill : pl.nfill0;
  if (nf) bl_launch(bl_zero_fill, bl_grid((long long)nf * D * D, g.Bp), BL_TPB, s, g, w, D * D, fl, nf);
  bl_launch(bl_lin_slots<D>, bl_grid(g.E + g.P, g.Bp), BL_TPB, s, g, pr, w);
  bl_launch(bl_lin_poses<D>, bl_grid(g.N + g.ndup, g.Bp), BL_TPB, s, g, w, lam, damping);
}

template <int D>
void bl_factor_all(const BLPlan& pl, int B, const BLWs& w, bool fused_fwd, cudaStream_t s) {
  BLDev g = pl.dev;
  g.B = B;
  g.Bp = bl_pad(B);
  const BLSched sc = bl_schedule(pl, B);
  const int lsplit = sc.fsplit;
  // chunked schedule: the bottom subtrees in one launch, then per level the items / factor items of the other
  // columns (levels whose columns are all in subtrees launch nothing)
  const bool sub = sc.sub && lsplit > pl.sub_top;
  if (sub)
    for (size_t p = 0; p + 1 < pl.sub_pass.size(); ++p) {
      const int a = pl.sub_pass[p], n = pl.sub_pass[p + 1] - a;
      if (n > 0)
        bl_launch(bl_subtree<D>, bl_grid(n, g.Bp), BL_TPB, s, g, w, pl.pd.bcon, pl.d_sub_ptr + a, pl.d_sub_rec, n,
                  fused_fwd ? 1 : 0);
    }
  for (int l = 0; l < lsplit; ++l) {
    const int t0 = pl.tsk_lvl_ptr[l], nt = pl.tsk_lvl_ptr[l + 1] - t0;
    const int c0 = pl.lvl_ptr[l], nc = pl.lvl_ptr[l + 1] - c0;
    const long long nu = (long long)nt + (fused_fwd ? nc : 0);
    if (sc.rb && pl.lch > 0) {
      // chunked work items of the level (forward rows skipped in the final factorisation: they have no
      // effect there), then the factor launch with the split reductions folded in
      const std::vector<int>& lp = sub ? pl.litf_lvl_ptr : pl.lit_lvl_ptr;
      const int i0 = lp[l], ni = lp[l + 1] - i0;
      if (ni > 0)
        bl_launch(bl_update_items<D>, bl_grid(ni, g.Bp), BL_TPB, s, g, w, sub ? pl.d_litems_f : pl.d_litems, i0, ni,
                  fused_fwd ? 1 : 0);
      const std::vector<int>& fp = sub ? pl.facf_lvl_ptr : pl.fac_lvl_ptr;
      const int f0 = fp[l], nf = fp[l + 1] - f0;
      if (nf > 0)
        bl_launch(bl_factor_red<D>, bl_grid(nf, g.Bp), BL_TPB, s, g, w, sub ? pl.d_facf : pl.d_facr, f0, nf,
                  fused_fwd ? 1 : 0, sub ? pl.d_bred_f : pl.d_bred, sub ? pl.d_cred_f : pl.d_cred);
      continue;
    }
    if (nu > 0 && sc.rb)
      bl_launch(bl_update_rb<D>, bl_grid(nu, g.Bp), BL_TPB, s, g, w, t0, nt, pl.d_lvl_col + c0, nc, fused_fwd ? 1 : 0);
    else if (nu > 0)
      bl_launch(bl_update<D>, bl_grid_rows(nu, g.Bp), D * 32, s, g, w, t0, nt, pl.d_lvl_col + c0, nc, fused_fwd ? 1 : 0);
    const int f0 = pl.fac_lvl_ptr[l], nf = pl.fac_lvl_ptr[l + 1] - f0;
    bl_launch(bl_factor<D>, bl_grid(nf, g.Bp), BL_TPB, s, g, w, f0, nf, fused_fwd ? 1 : 0);
  }
  if (lsplit < pl.L) {
    // levels [lsplit, L) in one persistent launch; group width: the widest of 16 / 8 / 4 elements that still
    // gives >= 128 CTAs (a sector is 4 doubles)
    const int gw = sc.gw;
    const int ff = fused_fwd ? 1 : 0;
    switch (gw) {
      case 32: bl_launch(bl_persist<D, 32>, (B + 31) / 32, BLP_NT, s, g, w, pl.pd, ff, lsplit, pl.L); break;
      case 16: bl_launch(bl_persist<D, 16>, (B + 15) / 16, BLP_NT, s, g, w, pl.pd, ff, lsplit, pl.L); break;
      case 8: bl_launch(bl_persist<D, 8>, (B + 7) / 8, BLP_NT, s, g, w, pl.pd, ff, lsplit, pl.L); break;
      default: bl_launch(bl_persist<D, 4>, (B + 3) / 4, BLP_NT, s, g, w, pl.pd, ff, lsplit, pl.L); break;
    }
  }
}

template <int D>
void bl_solve(const BLPlan& pl, int B, const BLWs& w, bool forward, const int* skip, cudaStream_t s) {
  BLDev g = pl.dev;
  g.B = B;
  g.Bp = bl_pad(B);
  const BLSched sc = bl_schedule(pl, B);
  // bl_lsolve: the first level from which every level's items fit the shared-memory budget
  int ls = sc.lsplit;
  size_t smem = 0;
  if (pl.lsolve && ls < pl.L) {
    constexpr size_t budget = 200 * 1024;
    auto need = [&](int l) {
      const int ni = std::max(pl.bit_lvl_h[l + 1] - pl.bit_lvl_h[l], pl.fit_lvl_h[l + 1] - pl.fit_lvl_h[l]);
      return (size_t)ni * D * sc.sgw * sizeof(double);
    };
    int lo = pl.L;
    while (lo > ls && need(lo - 1) <= budget) --lo;
    ls = lo;
    for (int l = ls; l < pl.L; ++l) smem = std::max(smem, need(l));
  }
  auto tail = [&](int fwd) {
    if (ls >= pl.L) return;
    if (pl.lsolve) {
      auto go = [&](auto kern, int gw) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        bl_launch_smem(kern, (B + gw - 1) / gw, BLP_NT, smem, s, g, w, pl.pd, pl.sd, skip, fwd, ls, pl.L);
      };
      switch (sc.sgw) {
        case 32: go(bl_lsolve<D, 32>, 32); break;
        case 16: go(bl_lsolve<D, 16>, 16); break;
        case 8: go(bl_lsolve<D, 8>, 8); break;
        default: go(bl_lsolve<D, 4>, 4); break;
      }
      return;
    }
    switch (sc.gw) {
      case 32: bl_launch(bl_persist_solve<D, 32>, (B + 31) / 32, BLP_NT, s, g, w, pl.pd, skip, fwd, ls, pl.L); break;
      case 16: bl_launch(bl_persist_solve<D, 16>, (B + 15) / 16, BLP_NT, s, g, w, pl.pd, skip, fwd, ls, pl.L); break;
      case 8: bl_launch(bl_persist_solve<D, 8>, (B + 7) / 8, BLP_NT, s, g, w, pl.pd, skip, fwd, ls, pl.L); break;
      default: bl_launch(bl_persist_solve<D, 4>, (B + 3) / 4, BLP_NT, s, g, w, pl.pd, skip, fwd, ls, pl.L); break;
    }
  };
  if (forward) {
    for (int l = 0; l < ls; ++l) {
      const int c0 = pl.lvl_ptr[l], nc = pl.lvl_ptr[l + 1] - c0;
      bl_launch(bl_fsolve<D>, bl_grid_rows(nc, g.Bp), D * 32, s, g, w, pl.d_lvl_col + c0, nc, skip);
    }
    tail(1);
  }
  tail(0);
  for (int l = ls - 1; l >= 0; --l) {
    const int c0 = pl.lvl_ptr[l], nc = pl.lvl_ptr[l + 1] - c0;
    if (sc.rb && pl.bsolve_ct && nc >= pl.bsolve_ct)
      bl_launch(bl_bsolve_ct<D>, bl_grid(nc, g.Bp), BL_TPB, s, g, w, pl.d_lvl_col + c0, nc, skip);
    else
      bl_launch(bl_bsolve<D>, bl_grid_rows(nc, g.Bp), D * 32, s, g, w, pl.d_lvl_col + c0, nc, skip);
  }
}

// K Gauss-Newton iterations (+ the undamped linearise + factor at theta_K in implicit mode)
template <int D>
void bl_forward(const BLPlan& pl, int B, const DevProb& pr, const BLWs& w, int K, double alpha, int early_stop,
                double abs_tol, double rel_tol, bool implicit, double* objective, int* status, int* iterations,
                BLPhaseTimer& tm, cudaStream_t s) {
  BLDev g = pl.dev;
  g.B = B;
  g.Bp = bl_pad(B);
  bl_launch(bl_init, bl_grid_b(g.Bp), BL_TPB, s, g, w);
  for (int k = 0; k < K; ++k) {
    bl_linearize<D>(pl, B, pr, w, -1.0, 0, s);
    bl_launch(bl_objective, g.Bp / 32, BL_SW * 32, s, g, w, early_stop, abs_tol, rel_tol, k > 0 ? 1 : 0, 1, 0);
    tm.begin(s);
    bl_factor_all<D>(pl, B, w, true, s);
    tm.end(s);
    bl_launch(bl_check_fail, bl_grid_b(B), BL_TPB, s, g, w);
    bl_solve<D>(pl, B, w, false, w.st, s);   // frozen / failed elements skip the solve and the retraction
    bl_launch(bl_retract<D>, bl_grid(g.N, g.Bp), BL_TPB, s, g, pr, w, alpha);
  }
  if (implicit) {
    bl_launch(bl_pre_final, bl_grid_b(B), BL_TPB, s, g, w);
    bl_linearize<D>(pl, B, pr, w, -1.0, 0, s);
    bl_launch(bl_objective, g.Bp / 32, BL_SW * 32, s, g, w, 0, abs_tol, rel_tol, 0, 0, 0);
    // the final factor is computed for every element that still has a defined iterate
    tm.begin(s);
    bl_factor_all<D>(pl, B, w, false, s);
    tm.end(s);
  } else {
    bl_launch(bl_cost_only<D>, bl_grid(g.E + g.P, g.Bp), BL_TPB, s, g, pr, w);
    bl_launch(bl_objective, g.Bp / 32, BL_SW * 32, s, g, w, 0, abs_tol, rel_tol, 0, 0, 1);
  }
  bl_launch(bl_finish, bl_grid_b(B), BL_TPB, s, g, w, implicit ? 1 : 0, abs_tol, rel_tol, objective, status, iterations);
}

// implicit backward on the BL factor of H(theta_K): lambda = H^-1 v, per-slot weight gradients, batch reduction
template <int D>
void bl_backward_implicit(const BLPlan& pl, int B, const DevProb& pr, const BLWs& w, const double* gpose,
                          int grad_kind, double* ge, double* gp, long long bstride, cudaStream_t s) {
  BLDev g = pl.dev;
  g.B = B;
  g.Bp = bl_pad(B);
  bl_launch(bl_bwd_rhs<D>, bl_grid(g.N, g.Bp), BL_TPB, s, g, pr, w, gpose, grad_kind);
  bl_solve<D>(pl, B, w, true, nullptr, s);
  bl_launch(bl_bwd_slots<D>, bl_grid(g.E + g.P, g.Bp), BL_TPB, s, g, pr, w, w.cost);
  const int slots = g.E + g.P;
  if (slots > 0 && (ge || gp))
    bl_launch(bl_reduce_wgrad, (slots + 3) / 4, 128, s, B, g.Bp, g.E, g.P, w.cost, ge, gp, bstride);
}
