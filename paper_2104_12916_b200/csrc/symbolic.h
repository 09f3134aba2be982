// Host symbolic analysis for the multifrontal LDLᵀ / Cholesky factors used by
// the single-factorization IPM (arXiv 2104.12916):
//   * F = [−H Aᵀ; A 0] ordered x-block first (fill-reducing order), λ last
//     (P:L703–714 inertia; static 1×1 pivots, reading R5 in DESIGN.md);
//   * P_H = D + C·diag(H)⁻¹·Cᵀ, pattern of T = C·Cᵀ.
// Everything here is D-independent and computed once.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace qpb {

constexpr int BW = 64;          // pivot block width (columns per trsv block column)
constexpr int TILE_ELEMS = 4096; // max doubles in one trsv tile (32 KiB)
constexpr int XCH = 8;           // column blocks per X chunk of a big supernode
constexpr int FUSE_ELEMS = 2048;  // small supernodes with w·noff ≤ this are swept as one task
constexpr int TASK_SHIFT = 28;   // task = (type << TASK_SHIFT) | index
constexpr int LONG_TILE = 512;   // rows of a sweep tile of a full-width (BW) block
constexpr int LVL_MAX = 24;      // most elimination-tree levels swept level-synchronously (leaf phase)
constexpr int LVL_MIN = 1024;    // a level joins the leaf phase only with at least this many supernodes

// Lower-triangular (strict) pattern + values of a symmetric matrix already in
// factor order, by columns, plus its diagonal.
struct LowerMatrix {
  int64_t N = 0;
  std::vector<int64_t> colptr;   // N+1
  std::vector<int32_t> rowind;   // strictly lower rows, sorted per column
  std::vector<double> val;       // values (may be empty for pattern-only)
  std::vector<double> diag;      // N diagonal values (may be empty)
  std::vector<int64_t> src;      // optional source index per stored entry (P_H: index into T values)
  std::vector<int64_t> diag_src; // optional source index of diagonal (P_H)
};

struct StepDesc {
  int level, k;
  int k0;             // first pivot block of the step's group
  int kind;           // 0 DIAG+PANEL(k); UPDATE with 2: block k on the group's block columns k+1 .. e
                      // (i ≥ j); 3: blocks k0 .. e on the trailing tiles i ≥ j > e (e per front)
  int n_act;          // active fronts
  int64_t act_off;    // offset into act list
  int64_t pan_total;  // PANEL tiles
  int64_t upd_total;  // UPDATE tiles
};

struct LevelEA {        // extend-add groups of one level
  int64_t grp_off, n_grp;   // into grp arrays
  int64_t asm_off, n_asm;   // assembly entries of the level's fronts
  int64_t fr_off, n_fr;     // the level's fronts (into lev_fronts / lev_zpref)
};

struct Symbolic {
  int64_t N = 0;
  std::vector<int64_t> perm;      // new -> old (of the matrix being factored)
  std::vector<int64_t> parent, colcount, rowlev;
  int64_t nnz_L = 0, n_rowlev = 0;
  int64_t nnz_stored = 0;          // entries stored by the relaxed supernodes (≥ nnz_L)
  int64_t trailing_from = -1;       // see analyse()
  int64_t sym_true = 0;            // true nnz(L) in the columns of symmetric roots
  int64_t sym_lower = 0;           // w(w+1)/2 summed over symmetric roots (entries of S⁻¹ read per solve)
  double c_fact = 0;              // Σ cc²

  // supernodes
  int64_t ns = 0;
  std::vector<int64_t> sn_start, sn_parent, sn_level, sn_rowptr;
  std::vector<int32_t> sn_rows;   // global rows (factor order)
  int64_t n_levels = 0;

  // fronts
  std::vector<int64_t> front_off;  // doubles; fronts share memory by liveness (level schedule)
  int64_t ws_size = 0;             // doubles (peak of the liveness plan)
  int64_t ws_naive = 0;            // doubles if every front were allocated at once
  std::vector<int32_t> lev_fronts; // fronts grouped by level
  std::vector<int64_t> lev_zpref;  // per level: prefix of m² (n_fr+1 entries per level, concatenated)

  // blocks
  int64_t nb = 0;
  std::vector<int32_t> sn_blk0;    // ns+1
  std::vector<int32_t> blk_col0, blk_w, blk_sn, blk_noff;
  std::vector<int64_t> blk_rows;   // offset into sn_rows of the first off-diag row
  std::vector<int64_t> blk_inv, blk_off; // factor-storage offsets (doubles)
  int64_t fs_size = 0;
  std::vector<int32_t> col2blk;    // N

  // trsv tiles + task queues.  Task encoding: (type << 28) | index with
  // type 0 DIAG(block), 1 TILE(off-diagonal tile), 2 PREP(block of a big
  // supernode), 3 XCHUNK(chunk of the inverse diagonal block of a big
  // supernode), 4 SNF(small supernode swept in one task: diagonal + all rows),
  // 5 SCHUNK(chunk of S_J⁻¹ of a symmetric root: x_I += S_IK v_K and x_K += S_IKᵀ v_I),
  // 6 ROOTB(backward: the symmetric root's x is already final — publish it),
  // 7 SNW(up to 8 tiny single-block supernodes of one level, one warp each).
  std::vector<int32_t> tile_blk, tile_r0, tile_nr;
  std::vector<int64_t> tile_dptr;    // tile t's destination SUPERNODES: tile_dlist[tile_dptr[t] .. tile_dptr[t+1])
  std::vector<int32_t> tile_dlist;
  std::vector<int32_t> fwd_tasks, bwd_tasks, fwd_expect /*per supernode*/, bwd_expect /*per block*/;
  std::vector<int32_t> fwd_tasks_x, bwd_tasks_x;   // same queues with symmetric roots swept through X/Xᵀ (fallback)
  // partitioned inverse of multi-block ("big") supernodes
  std::vector<int64_t> sn_xinv;          // offset of X_J = L_JJ⁻¹ (w×w col-major, ld sn_ldx) or -1
  std::vector<int64_t> sn_xtr;           // offset of X_Jᵀ (same layout)
  std::vector<int64_t> sn_ldx;           // leading dimension (w rounded up to 8)
  std::vector<int32_t> xb_bK, xb_bI, xb_nI; // backward chunks: output block K, first row-block I, #blocks
  std::vector<int64_t> sn_sinv;          // symmetric root: offset of S_J⁻¹ = X_Jᵀ D_J⁻¹ X_J (lower + full diagonal tiles) or -1
  std::vector<int32_t> sexp;             // per block of a symmetric root: contributions to x_I expected
  int64_t sym_c0 = 0, sym_c1 = 0;        // chunk range [sym_c0, sym_c1) of the symmetric roots (separate GEMV kernel)
  std::vector<int32_t> xt_bI, xt_bK, xt_nK; // X chunks: row-block, first column-block, #column-blocks
  std::vector<int32_t> xexp_f, xexp_b;   // per block: X chunks covering the row-block / column-block
  std::vector<int32_t> sn_nblk;          // blocks per supernode
  std::vector<int64_t> blk_dptr;         // per block: fused destination-supernode list (nb+1)
  std::vector<int32_t> blk_dest;
  std::vector<int32_t> snw_fwd, snw_bwd; // warp-swept tiny supernodes: 8 block ids per task (type 7), -1 padded
  // leaf phase: the lowest lvl_cut levels of the supernodal elimination tree (all single-block supernodes
  // ≤ 32 columns, ≥ LVL_MIN of them per level) are swept level by level, one kernel per level and a group of
  // 16 or 32 lanes per supernode (k_lvl_fwd / k_lvl_bwd), before (forward) / after (backward) the task graph;
  // they take no part in its counters.  lvl_blk: their blocks, level by level (lvl_ptr); lvl_g: lanes per
  // supernode of each level.
  int32_t lvl_cut = 0;
  std::vector<int64_t> lvl_ptr;
  std::vector<int32_t> lvl_blk, lvl_g;
  std::vector<int32_t> blk_big;          // 1 if the block belongs to a big supernode
  int64_t x_size = 0;                    // doubles of all X_J
  int64_t xtmp_size = 0;                 // doubles of the inversion scratch
  std::vector<int64_t> sn_xtmp;          // scratch offset per big supernode

  // flattened forest (two-factor partitioned inverse, see plan_flat): with a symmetric root J0
  // (columns [rc0, N)) the forest part L11 (columns [0, rc0)) and its coupling L21 enter every
  // F-solve only through  y1 = L11⁻¹ b1,  v2 = b2 − M b1  (M = L21 L11⁻¹)  and
  // x1 = L11⁻ᵀ D1⁻¹ y1 − Mᵀ x2: dependency-free products instead of level-by-level sweeps.
  bool flat = false;
  int64_t fl_rc0 = 0;                 // first root column (= number of forest columns)
  std::vector<int64_t> fl_roff;       // per forest supernode J (ns_f + 1): offset into fl_rows
  std::vector<int32_t> fl_rows;       // R_J: root-relative rows of M[:, J] (sorted)
  std::vector<int64_t> fl_moff;       // per forest supernode: offset of M_J (|R_J| × w_J, column-major)
  int64_t fl_msize = 0;               // doubles of all M_J
  std::vector<int64_t> fl_cp;         // L11⁻¹ by columns (rc0 + 1)
  std::vector<int32_t> fl_ci;         //   rows of each column (own supernode's columns ≥ c, then ancestors')
  std::vector<int64_t> fl_rp;         // L11⁻¹ by rows (rc0 + 1)
  std::vector<int32_t> fl_rj;         //   columns of each row
  std::vector<int64_t> fl_r2c;        //   index of each row entry in the column-ordered values
  std::vector<int32_t> fl_col2sn;     // forest column → supernode
  std::vector<int32_t> fl_mt_J, fl_mt_q0, fl_mt_nq;   // M tiles (nq·w_J ≤ TILE_ELEMS) of the backward product
  std::vector<int64_t> fl_mr_ptr;     // M by root rows (w_root + 1): the forward product's row form
  std::vector<int32_t> fl_mr_col;     //   forest column of each entry
  std::vector<int32_t> fl_mr_src;     //   index of each entry in the M_J blocks (values copied once)

  // multifrontal plan
  int32_t mf_group = 4;               // pivot blocks per trailing update (see the steps in analyse)
  std::vector<int64_t> asm_dst;    // destination in workspace for each lower entry (+diag)
  std::vector<double> asm_val;     // F: values; P_H: T-values filled on device
  std::vector<int64_t> asm_src;    // P_H: index into device T values (-1 = none)
  std::vector<int64_t> diag_dst;   // P_H: workspace position of each diagonal (factor order)
  std::vector<int32_t> asm_diag;   // per assembly entry: factor column if it is a diagonal entry, else -1
  std::vector<int32_t> relind;     // per child: positions in parent of rows [w, m)
  std::vector<int64_t> relind_off; // ns
  std::vector<int32_t> grp_P, grp_pc; // extend-add groups (parent sn, parent-local col)
  std::vector<int64_t> grp_ptr;       // n_grp+1 into grp_K/grp_j
  std::vector<int32_t> grp_K, grp_j;
  std::vector<LevelEA> level_ea;      // per level
  std::vector<StepDesc> steps;
  std::vector<int32_t> act;           // concatenated active-front lists
  std::vector<int64_t> pan_pref, upd_pref; // per step: (n_act+1) prefix, concatenated at act_off + step_index
  std::vector<int64_t> pref_off;      // per step offset into pan_pref/upd_pref
  std::vector<signed char> pivsign;   // expected pivot sign per column (factor order)
};

// Build the permuted lower pattern of F = [−H Aᵀ; A 0] (x block by pinv, λ last).
LowerMatrix build_F_lower(int64_t n, int64_t m1, const int64_t* Hp, const int32_t* Hi, const double* Hx,
                          const int64_t* Ap, const int32_t* Ai, const double* Ax,
                          const std::vector<int64_t>& xperm);

// Symmetric pattern (full, both triangles, no diagonal) → approximate minimum
// degree order (new→old).
// dense_stop < 1: stop once the minimum degree reaches that fraction of the remaining nodes.
std::vector<int64_t> min_degree_order(int64_t n, const std::vector<int64_t>& ptr,
                                      const std::vector<int32_t>& idx, double dense_stop = 1.0);

// Nested dissection by BFS level structures (new→old); parts of ≤ leaf nodes keep their input order.
std::vector<int64_t> nested_dissection_order(int64_t n, const std::vector<int64_t>& ptr,
                                             const std::vector<int32_t>& idx, int64_t leaf = 64);

// Equivalent reordering by an elimination-tree postorder (same fill), composed with `order`.
std::vector<int64_t> etree_postorder(int64_t n, const std::vector<int64_t>& ptr, const std::vector<int32_t>& idx,
                                     const std::vector<int64_t>& order);

// Full symbolic analysis + multifrontal / trsv plans.  Returns "" or an error.
// trailing_from ≥ 0: after amalgamation, every supernode reaching column trailing_from or beyond is merged
// with the last supernode into one dense trailing supernode (requires that block to be closed: the
// ancestor-closed top of the tree reordered to the end).
// max_sn_width > 0: supernodes wider than that are split into a chain of pieces (P_H).
std::string analyse(const LowerMatrix& M, Symbolic& S, int64_t n_negative, bool allow_symroot = true,
                    int64_t trailing_from = -1, int64_t max_sn_width = 0);

// Decide and plan the flattened forest for a factor whose last supernode is a symmetric root
// (sets S.flat; no-op otherwise).  Limits: forest supernodes ≤ BW wide, rc0 ≤ max_cols, and
// nnz(M) ≤ max_rel_root · w_root(w_root+1)/2 (bytes bounded against the root GEMV).
void plan_flat(Symbolic& S, int64_t max_cols = 16384, double max_rel_root = 0.1);

}  // namespace qpb
