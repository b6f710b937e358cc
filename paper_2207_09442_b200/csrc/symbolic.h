// Host symbolic analysis of a pose graph ("symbolic analysis ... as a separate
// step", :221 "building an elimination tree and then clustering column blocks with similar
// sparsity patterns", :584 App. F).  Pure C++17, no CUDA.  All indices are pose ("block")
// indices unless named *_sc (scalar); D is the tangent dimension (3 or 6).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

// rows of a D x D target block per update item of the per-element factorisation (lane map of the level
// packets; the kernel's gather accumulates UPD_ROWS x D entries per item): 3 -> 2 items per SE3 block
constexpr int UPD_ROWS = 3;

namespace dnls {

struct SymbolicOptions {
  // relaxed supernode amalgamation (App. F: trade fragmentation against explicit zeros).
  // A child supernode is merged into its parent when the merged width (pose columns) and the
  // fraction of explicit zero blocks stay under these limits.
  int relax_always_cols = 1;      // merged width <= this: always merge
  int relax_small_cols = 1;       // ... <= this: merge if zero fraction <= relax_small_frac
  double relax_small_frac = 0.0;
  int relax_mid_cols = 1;
  double relax_mid_frac = 0.0;
  int relax_max_cols = 64;        // hard cap on supernode width (pose columns)
  double relax_big_frac = 0.0;
  // shared-memory budget (doubles) for factor panels: resident top levels + level staging
  int64_t smem_cap_doubles = 0;
  // threads per CTA of the numeric kernels (lane-group sizes are chosen against it)
  int cta_threads = 256;
  // size bound of one descriptor packet (ints); larger levels are split into chunks
  int packet_ints = 4096;
};

struct Symbolic {
  int D = 0, N = 0, E = 0, P = 0;
  std::vector<int32_t> edges;       // [E][2] original indices
  std::vector<int32_t> prior_vars;  // [P]
  std::vector<int32_t> perm, iperm; // perm[k] = original var at position k
  std::vector<int32_t> parent;      // pose-level elimination tree (permuted), -1 root
  std::vector<std::vector<int32_t>> colstruct;  // below-diagonal block rows per pose column
  int etree_height = 0;

  // supernodes (contiguous pose-column ranges in the postordered numbering)
  int S = 0;
  std::vector<int32_t> sn_first, sn_ncols, sn_level, sn_parent, sn_m, sn_ld, sn_w, col_sn;
  std::vector<int64_t> sn_off;                  // panel offset (doubles) in per-element storage
  std::vector<std::vector<int32_t>> sn_rows;    // below rows (permuted pose indices, sorted)
  int64_t storage = 0;
  int num_levels = 0;
  std::vector<int32_t> level_ptr, level_sn;     // supernodes grouped by level (height from leaves)
  std::vector<int32_t> level_off;               // [L+1] storage range of each level (level-ordered panels)
  std::vector<int32_t> level_stage_hi;          // [L] end of the staged (shared-memory) prefix of the level
  int64_t max_level_stage = 0;                  // largest staged prefix (doubles)
  int32_t res_lo = 0;                           // storage offsets >= res_lo are resident in shared memory
  int64_t res_n = 0;                            // resident doubles
  int64_t stage_cap = 0;                        // staging buffer capacity (doubles)

  // numeric factorisation: gather-form update tasks grouped by level of the target
  //   task t: target block at ut_off (storage offset of entry (0,0)), leading dim ut_ld,
  //           contributions [ut_cptr[t], ut_cptr[t+1])
  //   contribution c: source rows at uc_a (entry (row_p, k=0)), uc_b (row_q), ld uc_ld, width uc_w
  std::vector<int32_t> ut_level_ptr, ut_off, ut_ld, ut_cptr;
  std::vector<int32_t> uc_a, uc_b, uc_ld, uc_w;

  // forward substitution gather per permuted pose row p: sum over source panels holding row p
  std::vector<int32_t> fc_ptr, fc_off, fc_ld, fc_w, fc_x;
  // backward substitution: below rows of each supernode (flattened sn_rows)
  std::vector<int32_t> snr_ptr, snr;
  // update-task range [2s, 2s+1] of each target supernode
  std::vector<int32_t> ut_sn_ptr;
  // per-level descriptor packets (see symbolic.cpp 5b'), offsets in ints, largest packet
  std::vector<int32_t> pk, pk_off, pk_level;
  int pk_max = 0, npk = 0;

  // scatter-free assembly: every d x d block of the storage exactly once
  //   block k: storage offset blk_off[k], leading dim blk_ld[k], kind blk_kind[k]
  //   (0 = structural zero / upper part, 1 = diagonal, 2 = off-diagonal),
  //   contributions blk_con[blk_cptr[k] .. blk_cptr[k+1]): slot*4 + rowside*2 + colside
  //   (slot = edge e, or E + prior k; side 0 = first Jacobian J_i, 1 = J_j)
  std::vector<int32_t> blk_off, blk_ld, blk_kind, blk_cptr, blk_con;
  // b = J^T r per permuted pose: bc[bc_ptr[p] .. bc_ptr[p+1]) = slot*2 + side
  std::vector<int32_t> bc_ptr, bc;
  // off-diagonal blocks (blk_* indices) that receive contributions from more than one edge
  std::vector<int32_t> dup_blk;
  // per cost slot 3 int4: (off_ii, off_jj, off_ij, row-is-j flag), (ld_ii, ld_jj, ld_ij, 0),
  // (perm pose i, perm pose j, only-edge-between-its-poses flag, 0)
  std::vector<int32_t> slot_desc;

  // stats
  int64_t nnz_H_blocks = 0, nnz_L_blocks = 0, nnz_L = 0;
  double factor_flops = 0;
  int max_sn_cols_sc = 0, max_panel_rows = 0;
};

// Returns "" on success, else an error message; *code receives the dnls_status value.
std::string analyze(int D, int N, int E, const int32_t* edges, int P, const int32_t* priors,
                    const SymbolicOptions& opt, Symbolic& out, int* code);

}  // namespace dnls
