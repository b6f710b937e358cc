/*
 * dnls.h -- C ABI of libdnls: a B200-native (sm_100a) batched pose-graph Gauss-Newton /
 * Levenberg-Marquardt solver with implicit-differentiation backward.
 *
 * It implements the hot path of "Theseus: A Library for Differentiable Nonlinear
 * Optimization" (arXiv 2207.09442; citations "PAPER.md:n" are lines of that paper's text):
 *   objective       S(theta) = 1/2 sum_i || w_i c_i(theta^i) ||^2           (Eq. 1)
 *   GN step         (sum J^T J) delta = sum J^T r ;  theta <- theta [-] delta
 *   LM              damped system, adaptive damping
 *   sparse solve    one-time symbolic analysis, batched numeric Cholesky
 *   implicit bwd    Prop. 1: differentiate one Newton step at theta*
 *                   reusing the cached factor
 * Costs: SE2/SE3 relative-pose (Between) error c = Log(Z^-1 T_i^-1 T_j) and a
 * pose prior c = Log(Z^-1 T), right-perturbation Jacobians.
 *
 * Conventions:
 *   - poses are stored as the top rows of the homogeneous matrix, row-major:
 *       SE3: [3][4] = [R | t]   (12 doubles),   SE2: [2][3] = [R | t]   (6 doubles);
 *   - tangent vectors: SE3 (rho_x, rho_y, rho_z, omega_x, omega_y, omega_z); SE2 (rho_x, rho_y, omega);
 *   - right perturbation T <- T Exp(xi); GN/LM update T <- T Exp(-alpha delta) with H delta = J^T r.
 *   - all floating point is IEEE fp64.
 *
 * Ownership: the caller owns every device buffer (poses, measurements, weights, outputs,
 * workspace), following BaSpaCho's "does not own any allocated memory".  A
 * dnls_graph owns its host symbolic analysis and small read-only device index arrays; it is
 * immutable after creation and may be shared by concurrent calls on different workspaces.
 * The workspace carries the numeric factor from dnls_forward to dnls_backward_implicit
 * ("our backward pass can cache factorizations").
 *
 * Errors: every call returns dnls_status (0 = OK).  Argument / shape / structural errors are
 * detected on the host before anything is enqueued; the message is available from
 * dnls_last_error() (thread-local).  Numerical failures are PER BATCH ELEMENT, written to the
 * device array status[B] (codes DNLS_ST_*), never a global error.
 *
 * Asynchrony: every call except dnls_graph_create / dnls_graph_* queries and
 * dnls_last_error only enqueues work on the given CUDA stream (cudaStream_t passed as void*)
 * and never synchronises the host.  Device pointers must be device-accessible fp64 / int32.
 */
#ifndef DNLS_H_
#define DNLS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DNLS_API __attribute__((visibility("default")))
#define DNLS_VERSION 1

typedef enum {
  DNLS_OK = 0,
  DNLS_E_INVALID = 1,      /* null pointer, bad enum, bad option value */
  DNLS_E_SHAPE = 2,        /* sizes inconsistent with the graph */
  DNLS_E_STRUCTURAL = 3,   /* variable without any cost (empty diagonal block), self edge */
  DNLS_E_WORKSPACE = 4,    /* workspace too small */
  DNLS_E_STATE = 5,        /* backward without a matching implicit forward on this workspace */
  DNLS_E_ALL_FAILED = 6,   /* every element failed: returned only by the host-synchronous
                              dnls_status_summary (the compute calls are asynchronous, so per-element
                              failures stay in status[B]) */
  DNLS_E_CUDA = 7,         /* a CUDA runtime call failed */
  DNLS_E_UNSUPPORTED = 8   /* e.g. graph too large for the per-element kernels */
} dnls_status;

typedef enum { DNLS_SE2 = 3, DNLS_SE3 = 6 } dnls_group;          /* value = tangent dimension d */
typedef enum { DNLS_GN = 0, DNLS_LM = 1, DNLS_DOGLEG = 2 } dnls_optimizer;
/* backward modes (§4.3 :232-271): IMPLICIT keeps the factor of H(theta_K) (Prop. 1); UNROLL /
 * TRUNCATED keep theta_k, delta_k and the factor of every (of the last backward_steps) GN iteration for
 * dnls_backward_unroll ("necessary ... for unrolling"). */
typedef enum { DNLS_BWD_NONE = 0, DNLS_BWD_IMPLICIT = 1, DNLS_BWD_UNROLL = 2, DNLS_BWD_TRUNCATED = 3 } dnls_backward;
typedef enum { DNLS_DAMP_MARQUARDT = 0, DNLS_DAMP_IDENTITY = 1 } dnls_damping;
typedef enum { DNLS_GRAD_TANGENT = 0, DNLS_GRAD_MATRIX = 1 } dnls_grad_kind;

/* per-element status codes written to dnls_problem.status[B] */
#define DNLS_ST_OK 0          /* all iterations ran */
#define DNLS_ST_CONVERGED 1   /* early stop: |S_k - S_{k-1}| < abs_tol + rel_tol S_{k-1}; frozen */
#define DNLS_ST_NOT_SPD 2     /* a pivot <= 1e-13 * max diag(H) (GN: frozen at that iterate) */
#define DNLS_ST_SATURATED 3   /* LM rejected a step with lambda already at lambda_max; frozen */
/* Warning bit OR-ed into the code (mask the code with DNLS_ST_CODE_MASK): an implicit-mode forward whose
 * last accepted iteration still changed the objective by |S_K - S_{K-1}| >= abs_tol + rel_tol S_{K-1}
 * (theta_K may not be the optimum Prop. 1 assumes; "a warning, not an error"). */
#define DNLS_ST_WARN_NOT_CONVERGED 0x100
#define DNLS_ST_CODE_MASK 0xff

typedef struct dnls_options {
  int32_t optimizer;        /* dnls_optimizer */
  int32_t max_iterations;   /* K >= 0 ("max_iterations") */
  double step_size;         /* alpha in (0, 1], default 1 */
  double lambda0;           /* LM initial damping, default 1e-3 */
  double lambda_min;        /* default 1e-8 */
  double lambda_max;        /* default 1e5 */
  double lambda_down;       /* accept: lambda <- max(lambda / down, min), default 3 */
  double lambda_up;         /* reject: lambda <- min(lambda * up, max),   default 2 */
  int32_t damping;          /* dnls_damping: H + lambda diag(H) (default) or H + lambda I */
  int32_t early_stop;       /* 0 (default): run exactly K iterations */
  double abs_tol;           /* early-stop tolerances, default 1e-10 / 1e-8 */
  double rel_tol;
  int32_t backward_mode;    /* dnls_backward: IMPLICIT keeps the undamped factor of H(theta_K) */
  int32_t cluster_ctas;     /* CTAs sharing one batch element in dnls_forward: 0 = automatic (a cluster
                               of 4 / 2 CTAs when 4B / 2B <= #SMs and N >= 1024,
                               DESIGN.md "few large problems"), else 1, 2, 4 or 8 */
  /* Dogleg trust region (reading DL1): initial, maximum and
   * minimum radius of the tangent step, defaults 1, 1e4, 1e-10.  Step: the GN point if it lies in
   * the radius, else the scaled gradient (Cauchy point outside) or the dogleg interpolation;
   * gain ratio rho: accept iff rho > 0, rho > 0.75 doubles, rho < 0.25 halves the radius; a
   * rejection below the minimum radius freezes the element (status DNLS_ST_SATURATED). */
  double trust_radius0;
  double trust_radius_max;
  double trust_radius_min;
  /* DNLS_BWD_TRUNCATED: number T >= 1 of final GN iterations the backward differentiates through
   * (TBPTT); the workspace keeps min(T, K) iterations.  Ignored by the other modes. */
  int32_t backward_steps;
  /* Path of dnls_forward / dnls_backward_implicit (DESIGN.md §6 "throughput path"): 1 = one CTA per batch
   * element (fused k_forward, any optimizer / backward mode); 32 = the batch-interleaved level-major path
   * (element-interleaved factor storage, Gauss-Newton with the implicit or no backward, quadratic costs;
   * other settings fall back to 1); 0 = automatic: 32 when supported, batch >= 256 and batch x num_vars >=
   * 262144 (measured crossover, environment DNLS_BL_MIN_BATCH for the batch bound), else 1.  Results agree to rounding (summation order), tested. */
  int32_t batch_interleave;
} dnls_options;

typedef struct dnls_problem {
  double* poses;               /* in/out [B][N][r][r+1]: theta_0 in, theta_K out */
  const double* meas;          /* [B][E][r][r+1]  measurement Z_e of edge e */
  const double* prior_meas;    /* [B][P][r][r+1]  prior targets (use stride 0 to share one [P][..]) */
  int64_t prior_meas_bstride;  /* doubles between consecutive batch elements (0 = shared) */
  const double* w_edge;        /* [E] shared (stride 0) or [B][E] per element: scalar weight w_e */
  int64_t w_edge_bstride;
  const double* w_prior;       /* [P] / [B][P] */
  int64_t w_prior_bstride;
  double* objective;           /* out [B]: S(theta_K) = 1/2 sum ||w c||^2 (with the 1/2) */
  int32_t* status;             /* out [B]: DNLS_ST_* */
  int32_t* iterations;         /* out [B]: iterations executed (LM: accepted + rejected) */
  /* Welsch robust kernel on every Between edge ("learn the radius of a Welsh robust
   * cost function"; readings W1-W3): NULL = plain quadratic costs; else the radius k > 0,
   * [1] shared (stride 0) or [B] per element.  An edge then costs rho_k(s) = k^2/2 (1 - e^{-s/k^2}),
   * s = ||w c||^2, and the GN step is the IRLS step (J, r rescaled by sqrt(psi), psi = e^{-s/k^2}). */
  const double* radius;
  int64_t radius_bstride;
} dnls_problem;

typedef struct dnls_stats {
  int32_t group;               /* 3 or 6 */
  int32_t num_vars, num_edges, num_priors;
  int32_t num_supernodes;
  int32_t num_levels;          /* supernodal elimination-tree levels (schedule depth) */
  int32_t etree_height;        /* pose-level elimination-tree height */
  int32_t max_supernode_cols;  /* scalar width of the widest supernode */
  int32_t max_panel_rows;      /* scalar rows of the tallest panel */
  int32_t reserved0;
  int64_t nnz_H_blocks;        /* lower-triangle d x d blocks of H (incl. diagonal) */
  int64_t nnz_L_blocks;        /* lower-triangle d x d blocks of L (incl. diagonal) */
  int64_t nnz_L;               /* scalar nonzeros of the lower triangle of L */
  int64_t storage_doubles;     /* per-element factor storage (supernodal panels, full diagonal blocks) */
  double factor_flops;         /* per element: sum_j (m_j + 1)^2, m_j = below-diagonal count of scalar column j */
  double solve_flops;          /* per element: 4 nnz_L */
  /* algorithmic bytes per element per GN iteration: */
  double bytes_linearize;      /* read poses+meas, write H (8 nnz_L) and b */
  double bytes_factor;         /* 16 nnz_L */
  double bytes_solve;          /* 16 nnz_L + vectors */
  double bytes_update;         /* retraction: read/write poses, read delta */
  double bytes_backward;       /* adjoint solve + weight-gradient recompute */
  int64_t index_bytes;         /* device bytes of the symbolic index arrays */
  int64_t smem_bytes;          /* dynamic shared memory per CTA of the numeric kernels */
  int64_t resident_doubles;    /* factor storage held in shared memory for the whole solve */
} dnls_stats;

typedef struct dnls_graph dnls_graph;

/* Library / build identification ("sm_100a ..."), static string. */
DNLS_API const char* dnls_version_string(void);

/* Thread-local message for the last non-OK status returned on this thread ("" if none). */
DNLS_API const char* dnls_last_error(void);

/* Default options (SPEC.md:415 values for LM): GN, K = 10, alpha = 1, lambda0 = 1e-3,
 * [1e-8, 1e5], down 3, up 2, Marquardt damping, no early stop, backward NONE. */
DNLS_API void dnls_options_default(dnls_options* opt);

/* One-time symbolic analysis ("symbolic analysis ... as a separate step ...
 * used for all subsequent factorizations", :221 elimination tree + supernodes): fill-reducing
 * minimum-degree ordering (lowest index breaks ties), elimination tree, postorder, fundamental
 * + relaxed supernodes, panel layout, assembly / update / solve index lists, level schedule.
 * edges_ij: HOST [E][2] int32 (i, j) pose indices of Between costs (measurement of T_i^-1 T_j);
 * prior_vars: HOST [P] int32.  Uploads index arrays to `device`.  Host-synchronous.
 * device < 0 creates a HOST-ONLY graph (symbolic queries work, compute calls return
 * DNLS_E_INVALID) -- used to test the symbolic analysis without a GPU.
 * Errors: DNLS_E_INVALID (bad group / counts / nulls), DNLS_E_SHAPE (index out of range),
 * DNLS_E_STRUCTURAL (self edge, or a variable with no cost), DNLS_E_CUDA. */
DNLS_API dnls_status dnls_graph_create(int32_t group, int32_t num_vars, int32_t num_edges,
                                       const int32_t* edges_ij, int32_t num_priors,
                                       const int32_t* prior_vars, int32_t device, dnls_graph** out);
DNLS_API void dnls_graph_destroy(dnls_graph* g);
DNLS_API dnls_status dnls_graph_stats(const dnls_graph* g, dnls_stats* out);

/* Symbolic queries (host arrays, caller-allocated):
 *   perm[N]: perm[k] = original variable at elimination position k (H_perm = P H P^T);
 *   etree parent[N] in permuted indices (-1 = root);
 *   L block pattern in permuted pose indices, CSC: colptr[N+1], rowidx[nnz_L_blocks]
 *     (diagonal first, then increasing rows);
 *   supernodes: first[S], ncols[S] (pose columns), level[S]. */
DNLS_API dnls_status dnls_graph_perm(const dnls_graph* g, int32_t* perm);
DNLS_API dnls_status dnls_graph_etree(const dnls_graph* g, int32_t* parent);
DNLS_API dnls_status dnls_graph_pattern(const dnls_graph* g, int32_t* colptr, int32_t* rowidx);
DNLS_API dnls_status dnls_graph_supernodes(const dnls_graph* g, int32_t* first, int32_t* ncols,
                                           int32_t* level);

/* Bytes of device workspace for `batch` elements (factor storage, vectors, per-edge Jacobian
 * scratch, per-element optimiser state; with opt->backward_mode UNROLL / TRUNCATED also the per-iteration
 * history of min(K, T) iterations: poses, steps and factors).  opt may be NULL (no history).
 * 256-byte aligned base required. */
DNLS_API dnls_status dnls_workspace_bytes(const dnls_graph* g, int32_t batch, const dnls_options* opt,
                                          size_t* bytes);

/* Forward: K iterations of GN or LM on every batch element, then -- if
 * opt->backward_mode == DNLS_BWD_IMPLICIT -- linearise and factor the UNDAMPED H(theta_K) and
 * keep that factor in the workspace for dnls_backward_implicit (reading A11).
 * poses are updated in place to theta_K; objective/status/iterations written.
 * One CUDA block owns one batch element for the whole solve. */
DNLS_API dnls_status dnls_forward(const dnls_graph* g, int32_t batch, const dnls_options* opt,
                                  const dnls_problem* prob, void* workspace, size_t ws_bytes,
                                  void* stream);

/* Implicit backward (Prop. 1 with the Gauss-Newton Hessian, readings A11/A12):
 *   lambda = H(theta_K)^-1 v  using the factor cached by the last implicit dnls_forward on this
 *            workspace (no refactorisation),
 *   dL/dw_e = -2 w_e (C_e lambda_e) . c_e,  dL/dw_p likewise (C, c unweighted, at theta_K).
 * grad_poses: [B][N][d] right-tangent gradient (DNLS_GRAD_TANGENT) or [B][N][r][r+1] Euclidean
 *   gradient on the pose matrices (DNLS_GRAD_MATRIX; projected on the device, App. D).
 * grad_w_edge / grad_w_prior: outputs, [E]/[P] summed over the batch in a fixed order when
 *   grad_bstride == 0, else per element with that stride (doubles).  Either may be NULL.
 * grad_radius: output dL/dk of the Welsch radius (prob->radius != NULL), laid out like the radius:
 *   [1] summed over the batch for a shared radius (radius_bstride == 0), else [B]; may be NULL.  With a robust kernel the weight
 *   gradient is -2 w psi (1 - s/k^2) (C lambda) . c and dL/dk = -sum_e (2 s/k^3) psi w^2 (C lambda) . c.
 * prob->poses must hold theta_K as returned by that forward; weights/measurements unchanged.
 * Errors: DNLS_E_STATE if the workspace holds no implicit factor for (graph, batch). */
DNLS_API dnls_status dnls_backward_implicit(const dnls_graph* g, int32_t batch, const dnls_problem* prob,
                                            const double* grad_poses, int32_t grad_kind,
                                            double* grad_w_edge, double* grad_w_prior, double* grad_radius,
                                            int64_t grad_bstride, void* workspace, size_t ws_bytes,
                                            void* stream);

/* DLM backward (direct loss minimisation, PAPER.md :259-271 and App. :897-934; DESIGN.md
 * readings B1-B3):
 *   theta_direct = argmin S(theta) + || eps delta - v/2 ||^2  (delta in the chart at theta*),
 *   solved by ONE Gauss-Newton step from theta* (PAPER.md:934):
 *       (J^T J + 2 eps^2 I) delta_a = J^T r - eps v,   theta_direct = theta* [+] (-delta_a)
 *   (one extra factorisation of the augmented system), then
 *       dL/dw_e ~= (1/eps) [ dS/dw_e(theta*) - dS/dw_e(theta_direct) ],  dS/dw_e = w_e ||c_e||^2
 *   (and the same for the prior weight).  Approaches the implicit gradient as eps -> 0 at a
 *   converged theta* ("lim eps->0").
 * prob->poses: theta* (e.g. as returned by dnls_forward; any mode); grad_poses / grad_kind /
 * grad_w_* / grad_radius / grad_bstride as for dnls_backward_implicit (Welsch: dS/dw_e = psi w ||c||^2,
 * dS/dk = k (1 - psi) - (s/k) psi).  epsilon > 0 (finite).
 * The call does not need a cached factor; it overwrites the factor storage of the workspace, so a
 * later dnls_backward_implicit on it returns DNLS_E_STATE.  Elements whose augmented system is not
 * SPD contribute zero gradient.  Errors: DNLS_E_INVALID (NULL grad_poses, bad kind, epsilon),
 * DNLS_E_SHAPE, DNLS_E_WORKSPACE, DNLS_E_CUDA. */
DNLS_API dnls_status dnls_backward_dlm(const dnls_graph* g, int32_t batch, const dnls_problem* prob,
                                       const double* grad_poses, int32_t grad_kind, double epsilon,
                                       double* grad_w_edge, double* grad_w_prior, double* grad_radius,
                                       int64_t grad_bstride, void* workspace, size_t ws_bytes, void* stream);

/* Unroll / Truncated backward (§4.3 :235-239 "unrolled optimization", "truncated
 * backpropagation through time"; linear-solve gradients :224; reading U1):
 * the exact reverse-mode chain rule through the GN iterations recorded by the last dnls_forward with
 * backward_mode DNLS_BWD_UNROLL (every iteration) or DNLS_BWD_TRUNCATED (the last backward_steps) on
 * this workspace: per iteration k (in reverse), with v = dL/dtheta_{k+1},
 *   u_m = -alpha Jr(-alpha delta_m)^T v_m,  lambda = H_k^-1 u  (the iteration's cached factor),
 *   dL/dw_e += 2 w_e (C lambda).(c - C delta),
 *   dL/dtheta_k = Ad(Exp(alpha delta))^T v + sum_e w_e^2 [C^T C lambda + grad_eta((C lambda).(c - C delta) - (C delta).(C lambda))]
 * (the gradient of the two contractions of the Jacobian C with fixed vectors by central differences of
 * the analytic Jacobian, step 1e-5 in the chart: ~1e-10 relative, reading U1).
 * Gauss-Newton with quadratic costs only (the forward returns DNLS_E_UNSUPPORTED for LM / Dogleg /
 * a Welsch kernel in these modes).
 * grad_poses / grad_kind / grad_w_edge / grad_w_prior / grad_bstride as for dnls_backward_implicit.
 * grad_poses0: out [B][N][d] dL/dtheta_0 in right-tangent coordinates (zero when truncated to fewer
 *   iterations than were executed), or NULL.
 * Elements whose forward stopped on a non-SPD system differentiate through the iterations they executed.
 * Errors: DNLS_E_STATE (no unroll/truncated forward on this workspace/batch), DNLS_E_INVALID, DNLS_E_SHAPE. */
DNLS_API dnls_status dnls_backward_unroll(const dnls_graph* g, int32_t batch, const dnls_problem* prob,
                                          const double* grad_poses, int32_t grad_kind, double* grad_w_edge,
                                          double* grad_w_prior, double* grad_poses0, int64_t grad_bstride,
                                          void* workspace, size_t ws_bytes, void* stream);

/* ---- stage-level entry points (standalone solvers, "as standalone ... functions";
 *      SPEC.md:400).  They share the workspace layout of dnls_forward. ---- */

/* Linearise at prob->poses: per-edge residuals/Jacobians, scatter-free assembly of
 * H_lambda = H + lambda diag(H) (or + lambda I) into the factor storage and b = J^T r;
 * objective[B] = S(theta).  lambda: device [B] or NULL (undamped). */
DNLS_API dnls_status dnls_linearize(const dnls_graph* g, int32_t batch, const dnls_problem* prob,
                                    const double* lambda, int32_t damping, void* workspace,
                                    size_t ws_bytes, void* stream);

/* In-place supernodal numeric Cholesky of the factor storage: P H P^T = L L^T per element
 * (PAPER.md:221, :584).  status[B] (device, may be NULL) receives DNLS_ST_NOT_SPD for elements
 * whose pivot <= 1e-13 * max diag(H), else DNLS_ST_OK. */
DNLS_API dnls_status dnls_factorize(const dnls_graph* g, int32_t batch, void* workspace,
                                    size_t ws_bytes, int32_t* status, void* stream);

/* x = H^-1 rhs using the factor in the workspace (forward/back substitution, permutation
 * applied internally).  rhs, x: device [B][N][d] in ORIGINAL variable order; may alias. */
DNLS_API dnls_status dnls_solve_factored(const dnls_graph* g, int32_t batch, void* workspace,
                                         size_t ws_bytes, const double* rhs, double* x, void* stream);

/* Dense views for tests and standalone use (device buffers):
 *   export_factor: [B][n][n] permuted order, lower triangle of the storage (H after
 *     dnls_linearize/import, L after dnls_factorize), zeros elsewhere;
 *   import_matrix: [B][n][n] ORIGINAL order symmetric matrix -> storage (pattern entries only);
 *   export_rhs:    [B][N][d] ORIGINAL order b = J^T r from the last dnls_linearize.
 * dnls_solve_factored and the two exports read the per-element storage: on a workspace whose last
 * dnls_forward ran the batch-interleaved path (its factor is element-interleaved) they return
 * DNLS_E_UNSUPPORTED. */
DNLS_API dnls_status dnls_export_factor(const dnls_graph* g, int32_t batch, const void* workspace,
                                        size_t ws_bytes, double* dense, void* stream);
DNLS_API dnls_status dnls_import_matrix(const dnls_graph* g, int32_t batch, const double* dense,
                                        void* workspace, size_t ws_bytes, void* stream);
DNLS_API dnls_status dnls_export_rhs(const dnls_graph* g, int32_t batch, const void* workspace,
                                     size_t ws_bytes, double* b, void* stream);

/* Assembly map of the per-element factor storage (SURVEY.md §8(b) "per-edge/prior offsets so tests can
 * scatter an oracle H"; "symbolic analysis ... used for all subsequent factorizations").
 * Each block is a d x d column-major block at `off` doubles from the element's storage base (layout
 * [B][storage_doubles] as used by the stage-level entry points), column stride `ld`:
 *   edge_desc  HOST [E][7] = (off_ii, ld_ii, off_jj, ld_jj, off_ij, ld_ij, row_is_j): the diagonal blocks
 *              of the endpoints (lower triangles significant) and the below-diagonal block between them;
 *              row_is_j = 1 if the block row is pose j (block = H_ji), else it is H_ij;
 *   prior_desc HOST [P][2] = (off, ld) of the prior's diagonal block.
 * Either pointer may be NULL.  Host-only; works on host-only graphs.  Errors: DNLS_E_INVALID. */
DNLS_API dnls_status dnls_block_offsets(const dnls_graph* g, int32_t* edge_desc, int32_t* prior_desc);

/* Host-synchronous summary of a device status[B] array written by dnls_forward (synchronises `stream`):
 * n_failed = elements whose code is DNLS_ST_NOT_SPD or DNLS_ST_SATURATED, n_warned = elements with
 * DNLS_ST_WARN_NOT_CONVERGED.  Returns DNLS_E_ALL_FAILED when batch > 0 and every element failed
 * (SPEC.md:459), else DNLS_OK.  Outputs may be NULL.  Errors: DNLS_E_INVALID, DNLS_E_CUDA. */
DNLS_API dnls_status dnls_status_summary(const int32_t* status, int32_t batch, int32_t* n_failed,
                                         int32_t* n_warned, void* stream);

/* Debug: (tag, clock64) pairs recorded by CTA 0 of the last kernels in a -DDNLS_TRACE build
 * (pairs written to out[2*i], out[2*i+1]; at most `capacity` pairs; the buffer is reset).
 * Host-synchronous.  Returns DNLS_E_UNSUPPORTED in the production build. */
DNLS_API dnls_status dnls_debug_trace(int64_t* out, int32_t capacity, int32_t* count);

/* Debug: device times (ms) of the factorisation phases of the last batch-interleaved dnls_forward on this
 * graph when the process runs with DNLS_PHASE_TIMING=1 (CUDA events around every factorisation; used for
 * the factor-kernel roofline in bench.py).  Host-synchronous; clears the record.  count = phases written. */
DNLS_API dnls_status dnls_debug_phase_times(const dnls_graph* g, double* ms, int32_t capacity, int32_t* count);

/* Debug: number of kernels the library has enqueued in this process (every entry point counts its launches;
 * bench.py reports the count of its timed region as gpu_launches).  reset != 0: the counter restarts at 0
 * after being read.  Host-only, never fails for a non-NULL count (DNLS_E_INVALID otherwise). */
DNLS_API dnls_status dnls_debug_launch_count(int64_t* count, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* DNLS_H_ */
