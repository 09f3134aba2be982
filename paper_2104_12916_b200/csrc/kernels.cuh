// Device-side data structures and kernel declarations (sm_100a, fp64).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace qpb {

constexpr int NT = 256;            // threads per CTA for every kernel here
constexpr int MF_BW = 64;          // pivot block (must equal symbolic BW)
constexpr int TRSV_SMEM_DBL = 4096 + 64 + 1024;  // tile R×W ≤ 4096 with R+1 padding + gathered x (≤1024); Linv 64×65 + 1024

// One factor (F or P_H): symbolic plan + numeric storage + trsv sweep state.
struct DevFactor {
  int64_t N, ns, nb, n_tiles, n_fwd_tasks, n_bwd_tasks;
  // supernodes
  const int64_t* sn_start;
  const int64_t* sn_rowptr;
  const int32_t* sn_rows;
  const int64_t* front_off;
  const int32_t* sn_blk0;
  // blocks
  const int32_t* blk_col0;
  const int32_t* blk_w;
  const int32_t* blk_noff;
  const int64_t* blk_rows;
  const int64_t* blk_inv;
  const int64_t* blk_off;
  // trsv tiles / tasks
  const int32_t* tile_blk;
  const int32_t* tile_r0;
  const int32_t* tile_nr;
  const int64_t* tile_dptr;    // destination supernodes of tile t: tile_dlist[tile_dptr[t] .. tile_dptr[t+1])
  const int32_t* tile_dlist;
  const int32_t* fwd_tasks;
  const int32_t* bwd_tasks;
  const int32_t* fwd_expect;
  const int32_t* bwd_expect;
  // numeric
  double* ws;         // multifrontal workspace (fronts)
  double* fstore;     // factor storage: per block Linv (w×w) + off-diagonal (noff×w)
  double* Dpiv;       // pivots, factor order
  const signed char* pivsign;
  // trsv sweep state
  double* acc;                    // N: forward accumulators
  double* tacc;                   // N: backward accumulators
  unsigned long long* cnt_f;      // per SUPERNODE: forward contributions received
  unsigned long long* cnt_b;      // nb
  unsigned int* ready_f;          // nb
  unsigned int* ready_b;          // nb
  unsigned int* sweep;            // [0] ticket, [1] finished CTAs, [2] fwd epoch, [3] bwd epoch
  // partitioned inverse of big supernodes
  const int32_t* blk_sn;
  const int64_t* sn_xinv;
  const int32_t* xt_bI;
  const int32_t* xt_bK;
  const int32_t* xt_nK;
  const int32_t* xb_bK;
  const int32_t* xb_bI;
  const int32_t* xb_nI;
  const int64_t* sn_xtr;
  const int64_t* sn_ldx;
  const int64_t* sn_sinv;
  const int32_t* sn_nblk;
  const int32_t* snw_fwd;         // SNW tasks: 8 block ids each (-1 padded), forward / backward grouping
  const int32_t* snw_bwd;
  const int64_t* blk_dptr;        // fused small supernodes: destination supernode lists
  const int32_t* blk_dest;
  unsigned int* ready_sb;         // ns: backward — all of supernode J final
  unsigned long long* sn_done_b;  // ns: backward — completed column blocks of a big supernode
  const int32_t* xexp_f;
  const int32_t* xexp_b;
  double* xinv;                   // X_J storage
  double* vbuf;                   // N: staged right-hand sides of big supernodes
  unsigned long long* cntx_f;     // nb
  unsigned long long* cntx_b;     // nb
  unsigned int* vready_f;         // nb
  unsigned int* vready_b;         // nb
  // multifrontal plan
  const int64_t* asm_dst;
  const double* asm_val;
  const int64_t* asm_src;
  int64_t n_asm;
  const int64_t* diag_dst;
  const int32_t* asm_diag;
  const int32_t* lev_fronts;
  const int64_t* lev_zpref;
  const int32_t* relind;
  const int64_t* relind_off;
  const int32_t* grp_P;
  const int32_t* grp_pc;
  const int64_t* grp_ptr;
  const int32_t* grp_K;
  const int32_t* grp_j;
  const int32_t* act;
  const int64_t* pan_pref;
  const int64_t* upd_pref;
  int* status;        // pivot failures (device int)
  // flattened forest (Symbolic::flat): M_J blocks, L11⁻¹ (column-ordered values + both index forms)
  int flat;                       // 1: F-solves use k_flat_fwd / root GEMV / k_flat_bwd
  int64_t fl_rc0;
  const int64_t* fl_roff;
  const int32_t* fl_rows;
  const int64_t* fl_moff;
  double* fl_mval;
  const int64_t* fl_cp;
  const int32_t* fl_ci;
  const int64_t* fl_rp;
  const int32_t* fl_rj;
  const int64_t* fl_r2c;
  double* fl_nval;                // L11⁻¹ values in column order (fl_cp / fl_ci)
  const int32_t* fl_col2sn;
  const int32_t* fl_mt_J;
  const int32_t* fl_mt_q0;
  const int32_t* fl_mt_nq;
  int64_t fl_nmt;
  const int64_t* fl_mr_ptr;       // M by root rows (forward product)
  const int32_t* fl_mr_col;
  double* fl_mr_val;
  const int4* fl_units;           // M product units (≤ 64 rows × ≤ 8 columns), 2 × int4 each (k_flat_*_t)
  int64_t fl_nunits;
  double* fl_fslot;               // per unit: 64 row partials of the forward product (deterministic reduction)
  double* fl_bslot;               // per unit: 8 column partials of the backward product
  const int64_t* fl_fr_ptr;       // per root row: its forward slots fl_fr_src[ptr[r] .. ptr[r+1]) (unit order)
  const int32_t* fl_fr_src;
  const int64_t* fl_bc_ptr;       // per forest column: its backward slots (unit order)
  const int32_t* fl_bc_src;
  int mf_group;                   // pivot blocks per trailing UPDATE (Symbolic::mf_group)
  // leaf phase (Symbolic::lvl_*): trsv_forward / trsv_backward launch one level kernel per level
  const int4* lvl_desc;           // per leaf-phase supernode (level order), 2 × int4: L offset, L_bb⁻¹ offset,
                                  // row-list offset (int64 each, lo/hi), first column, w | noff << 6
  int32_t lvl_cut;
  int64_t lvl_ptr_h[25];          // host copy: blocks of level L are lvl_blk[lvl_ptr_h[L] .. lvl_ptr_h[L+1])
  int8_t lvl_g_h[24];             // host copy: lanes per supernode (16 or 32) of each level
  unsigned long long* tprof;  // optional sweep instrumentation [2 sweeps][8 types][5] + per-task trace
  int64_t ttrace_cap;         // per-sweep trace capacity (tasks) after the 70 summary words
  int sweep_var;      // A/B switch (QPB_SWEEP_VAR, default 1): bit 0 = backward long tiles two rows per lane
  int use_sym;        // 1: symmetric roots swept through S⁻¹ (queues fwd_tasks/bwd_tasks hold SCHUNK/ROOTB)
  int l2hint;         // A/B switch (QPB_L2HINT, default 0 = measured best): bit 0 = root GEMV streams S⁻¹ with L2::evict_first,
                      // bit 1 = flattened-forest arrays loaded with L2::evict_last (kept across F-solves)
};

// Deterministic accumulation plan of a chunked symmetric GEMV (k_dense_symv, k_symroot_gemv): every chunk
// writes its row and column partials to its own slot (64 + 512 doubles); k_symv_reduce then sums each
// output block's slots in the fixed order lsrc[lptr[o] .. lptr[o+1]) and adds the sum to x — no
// floating-point atomics, so results are bit-identical run to run.
struct SymvPlan {
  double* slots;             // 64 doubles per (chunk, output block) contribution, grouped by output block
                             // (nullptr: fp64 atomics, QPB_DETERMINISTIC=0)
  int32_t nob;               // output blocks
  const int64_t* lptr;       // output block o: its contributions are slots[64·lptr[o] .. 64·lptr[o+1]), in the
                             // fixed order (row partials first, then column partials, by chunk index)
  const int64_t* woff;       // per chunk (c − c_begin), 9 entries: slot offset (doubles) of its row partial
                             // and of its column partials for output blocks cob0, cob0+1, … (−1 unused)
  const int32_t* width;      // per output block: rows (≤ 64)
  const int64_t* x0;         // per output block: first index in x
  int64_t c_begin;
  int32_t ob_lo;             // output block id of the first block (symroot: F block id − ob_lo)
};

// CSR on the device (int64 row pointers, int32 columns).
struct DevCSR {
  int64_t nrows, ncols, nnz;
  const int64_t* p;
  const int32_t* i;
  const double* v;
};

// PCG scalar state (device), written by last-block reductions.
// With `defer` set (ν rows sharded over ranks), the last block stores its LOCAL reductions in
// red[] instead; the host all-reduces red[] across ranks and k_finalize applies the same update.
struct PcgState {
  double rho, pq, rr, rz, bnorm2, tol2, alpha, beta;
  int iter, maxit, done, status;
  unsigned int arrive;
  int defer;
  double red[4];
};

// IPM scalar state (device).
struct IpmState {
  double mu, sigma_mu, sigma, tau;
  double rg_inf, re_inf, ri_inf;
  double alpha, alpha_max;
  double objective;
  unsigned int arrive;
  int defer;          // see PcgState
  double m2_total;    // global number of inequality rows (μ = sᵀν / m2_total)
  double red[4];
};

// Finalization of a deferred reduction after the cross-rank all-reduce of red[] (one thread).
enum FinKind { FIN_PCG_INIT = 0, FIN_PCG_PQ, FIN_PCG_UPD1, FIN_PCG_INIT_PH, FIN_PCG_RZ_PH, FIN_IPM_MU,
               FIN_IPM_RESID, FIN_IPM_ALPHA };
void finalize(int kind, PcgState* ps, IpmState* is, int prec, cudaStream_t s);
// u[t] = Σ_k M(t,k)·x[k] for the rows of M (plain CSR SpMV; sharded Cᵀp / Cᵀν partial products)
void spmv(const DevCSR& M, const double* x, double* y, const int* done, int grid, cudaStream_t s);

// ---- multifrontal factorization
// zero the fronts of one level, then scatter its original entries (+ D on the diagonal for P_H)
void mf_assemble_level(const DevFactor& F, int64_t fr_off, int64_t n_fr, int64_t zero_total, int64_t asm_off,
                       int64_t n_asm, const double* src_vals, const double* D, const int64_t* perm, cudaStream_t s);
void mf_extend_add(const DevFactor& F, int64_t grp_off, int64_t n_grp, cudaStream_t s);
// kind: see StepDesc (0 DIAG+PANEL, 2 band UPDATE, 3 trailing UPDATE); k0: the group's first block
void mf_step(const DevFactor& F, int k, int k0, int kind, int64_t act_off, int n_act, int64_t pref_off,
             int64_t pan_total, int64_t upd_total, cudaStream_t s);

// ---- partitioned inverse X_J = L_JJ⁻¹ of big supernodes (factor time)
struct GemmProb {
  const double* A;
  const double* B;
  double* C;
  int M, N, K, lda, ldb, ldc;
  double alpha, beta;
  int flags;  // 1: A lower-triangular (k <= row), 2: B lower-triangular (k >= col),
              // 4: A upper-triangular (k >= row), 8: only tiles with tj <= ti (lower half, diagonal tiles full)
  int pad;
};
// tile_pref: per problem prefix of ⌈M/128⌉·⌈N/128⌉ tiles
void gemm_batched(const GemmProb* probs, const int64_t* tile_pref, int nprob, int64_t total_tiles,
                  cudaStream_t s);
void build_xinv(const DevFactor& F, const int32_t* big_sns, int n_big, int64_t max_w2, cudaStream_t s);
void transpose_xinv(const DevFactor& F, const int32_t* big_sns, int n_big, int64_t max_w2, cudaStream_t s);
// Y = D_J⁻¹ X_J (rows scaled by the pivots), in place, for the listed supernodes
void scale_xinv_rows(const DevFactor& F, const int32_t* sns, int n, int64_t max_w2, bool multiply, cudaStream_t s);

// ---- level-free task-graph triangular sweeps (persistent kernels)
struct SweepRhs {
  const double* rhs;        // dense rhs (factor order) or nullptr
  const int64_t* in_perm;   // optional gather index for rhs (rhs[in_perm[c]])
  DevCSR ct;                // optional: rhs[c] = Σ ct(c,:)·p for c < ct.nrows (K_F: Cᵀp fused)
  const double* p;
  const int* done_flag;     // early-exit flag (PCG converged) or nullptr
  int rhs_ready;            // flattened forest / level products: acc / vbuf / x already prepared (fused PCG step, phase D)
};
void trsv_forward(const DevFactor& F, const SweepRhs& r, double* x, int grid, cudaStream_t s);
// q = H p (with_h) + Cᵀ(D⁻¹∘(C p)) in two streaming passes (t: m2 scratch), natural order, no factor
void op_apply(const DevCSR& Hf, const DevCSR& Cf, const DevCSR& Ctf, const double* D, const double* p, double* t,
              double* q, bool with_h, int sms, cudaStream_t s);
// halo mode: q[i] = (H p)_i for i in [h_lo, h_hi) (else 0) + (Cᵀ t)_i, rows [q_lo, q_hi) only
void op_apply_range(const DevCSR& Hf, const DevCSR& Cf, const DevCSR& Ctf, const double* D, const double* p, double* t,
                    double* q, int64_t q_lo, int64_t q_hi, int64_t h_lo, int64_t h_hi, int sms, cudaStream_t s);
// dst[0, n) += src[0, n)
void add_range(double* dst, const double* src, int64_t n, cudaStream_t s);
// v[0, N) = the right-hand side described by r, out[0, N) = 0 (dense F⁻¹ mode)
void gather_rhs(const SweepRhs& r, double* v, double* out, int64_t N, int sms, cudaStream_t s);
// v[0, n) = 0 unless *done_flag
void zero_flag(double* v, int64_t n, const int* done_flag, cudaStream_t s);
void trsv_backward(const DevFactor& F, double* x, const int* done_flag, int grid, cudaStream_t s);
int trsv_grid(int device);
// x_J += S_J⁻¹ v_J for the symmetric-root chunks [c_begin, c_end) (dedicated kernel)
// sub != nullptr: the root's right-hand side is vbuf − sub (flattened forest: sub = acc = M b1)
void symroot_gemv(const DevFactor& F, double* x, int64_t c_begin, int64_t c_end, const SymvPlan* plan,
                  const int* done_flag, int grid,
                  cudaStream_t s, const double* sub = nullptr);
// flattened forest F-solve halves (see Symbolic::flat) and the per-column extraction of M and L11⁻¹
void flat_forward(const DevFactor& F, const SweepRhs& r, double* x, int sms, cudaStream_t s);
void flat_backward(const DevFactor& F, double* x, const int* done_flag, int sms, cudaStream_t s);
void flat_extract(const DevFactor& F, int64_t col, const double* x, double* unit, int64_t prev, cudaStream_t s);
void flat_set_unit(double* unit, int64_t col, cudaStream_t s);
// after the extraction: row-form values of M gathered from the M_J blocks
void flat_fill_rows(const DevFactor& F, const int32_t* src, int64_t nnz, cudaStream_t s);

// ---- level products (partitioned inverse by elimination-tree levels, F only; DESIGN §5 "level products")
// Every supernode J above the leaf phase and below the symmetric root stores the panel
//   Z_J = [X_J; Y_J],  X_J = L_JJ⁻¹ (w×w, lower),  Y_J = L_ext,J · X_J (noff×w),
// column-major with an even leading dimension.  With v_J = b_J − acc_J the forward step of J is the one
// product [y_J; u] = Z_J v_J (u added to acc[rows]); backward x_J = X_Jᵀ D_J⁻¹ y_J − Y_Jᵀ x_rows = Z_Jᵀ s.
// Neither has a dependency inside the supernode, so one level of the tree is one dependency-free kernel
// over tiles of ≤ 512 rows × ≤ 64 columns (the classical no-fill partitioned inverse with the
// elimination-tree levels as partitions).
struct PiTile {          // 32 bytes, read as two int4
  int64_t zoff;          // first entry of the tile in Z (even)
  int64_t roff;          // first row of the tile in sn_rows
  int32_t ld;            // leading dimension of Z_J (even)
  int32_t col0;          // factor column of the tile's first column
  int16_t nr, nc;        // rows (≤ 512), columns (≤ 64)
  int16_t wx;            // rows of the tile that lie in X_J (the supernode's own columns): 0 … nr
  int16_t pad;
};
constexpr int PI_MAXLEV = 64;
// Subtrees (below the level products): a maximal subtree of small supernodes whose factor entries fit a byte
// budget is swept by ONE WARP, bottom-up (forward) / top-down (backward) with the subtree's part of the
// vector in shared memory — __syncwarp between its local levels replaces kernel boundaries, updates
// inside the subtree never touch global memory, and its rows above the subtree (all contained in the root's
// row list) are flushed / gathered once.  The subtree's factor entries are one contiguous range of fstore
// (postorder), prefetched into L2 when the CTA starts.
constexpr int ST_FRAME = 512;
constexpr int ST_MAXSN = 48;    // most supernodes of a subtree (its descriptors are staged in shared memory); local levels ≤ 31   // most doubles of a subtree's frame (its columns + the root's external rows)
struct StHdr {           // 48 bytes
  int32_t d0;            // first descriptor (st_desc, 2 × int4 each, local-level order)
  int32_t nlev;          // local levels
  int32_t c_lo, ncols;   // the subtree's columns [c_lo, c_lo + ncols)
  int32_t next;          // external rows of the subtree's root
  int32_t lptr;          // st_lptr[lptr .. lptr + nlev]: descriptor ranges of the local levels (relative to d0)
  int64_t rootrows;      // offset into sn_rows of the root's external rows
  int64_t fslo;          // the subtree's entries: fstore[fslo, fslo + fslen)
  int32_t fslen, pad;
};
struct PiSweep {
  int enabled = 0;
  int nlev = 0;                        // levels lvl_cut … top−1 (the symmetric root excluded)
  const PiTile* tiles = nullptr;       // forward tiles, level-major
  const int32_t* tile_J = nullptr;     // supernode of each forward tile (build only)
  const PiTile* btiles = nullptr;      // backward tiles (same Z, strips for taller supernodes than forward)
  int64_t blev_ptr[PI_MAXLEV + 1] = {0};
  int64_t blev_sptr[PI_MAXLEV] = {0};
  int prefetch = 1;                    // CTA tiles prefetch their part of Z into L2 before the dependent loads
  double* Z = nullptr;
  int64_t z_size = 0;
  int64_t root0 = 0;                   // first column of the symmetric root
  int64_t lev_ptr[PI_MAXLEV + 1] = {0};
  int64_t lev_sptr[PI_MAXLEV] = {0};   // level L: CTA tiles [lev_ptr[L], lev_sptr[L]), then strips (≤ 64 rows, a warp
                                       // each, 8 per CTA) [lev_sptr[L], lev_ptr[L + 1])
  // subtrees (st_n = 0: the leaf phase's level kernels run instead)
  int64_t st_n = 0;
  int st_g = 16;                       // lanes per supernode (16: every subtree supernode has ≤ 16 columns)
  const StHdr* st_hdr = nullptr;
  const int4* st_desc = nullptr;       // as DevFactor::lvl_desc, the row-list offset pointing into st_loc
  const int32_t* st_lptr = nullptr;
  const int32_t* st_loc = nullptr;     // per off-diagonal row of a subtree supernode: its index in the frame
};
// Z from the factor storage (after the numeric factorization and the X_J inverses); zoffJ: per supernode offset of Z_J (device)
void pi_build(const DevFactor& F, const PiSweep& P, const int64_t* zoffJ, cudaStream_t s);
// pi_forward starts with pi_init unless r.rhs_ready (the fused PCG step's phase D, next_rhs = 4, did the same)
void pi_init(const DevFactor& F, const PiSweep& P, const SweepRhs& r, double* x, int sms, cudaStream_t s);
void pi_forward(const DevFactor& F, const PiSweep& P, const SweepRhs& r, double* x, int sms, cudaStream_t s);
void pi_backward(const DevFactor& F, const PiSweep& P, double* x, const int* done_flag, cudaStream_t s);

// ---- vector / SpMV kernels
void kf_q(const DevCSR& Cf, const int32_t* longr, int64_t nlong, const double* D, const double* p, const double* z,
          double* q, double* partial, PcgState* st, int grid, cudaStream_t s, bool pcg_mode);
void pcg_init(int prec, int64_t m2, const double* b, const double* D, double* x, double* r, double* z,
              double* p, double* partial, PcgState* st, double tol, int maxit, int grid, cudaStream_t s);
void pcg_init_ph(int64_t m2, const double* r, const double* z, double* p, double* partial, PcgState* st,
                 int grid, cudaStream_t s);
void pcg_update1(int prec, int64_t m2, const double* D, const double* p, const double* q, double* x,
                 double* r, double* z, double* partial, PcgState* st, int grid, cudaStream_t s);
void pcg_rz_ph(int64_t m2, const double* r, const double* z, double* partial, PcgState* st, int grid,
               cudaStream_t s);
void pcg_update2(int64_t m2, const double* z, double* p, PcgState* st, int grid, cudaStream_t s);
// Launch timeline instrumentation (debug): kernels 0 flat_rhs, 1 flat_fwd, 2 root GEMV, 3 flat_bwd,
// 4 pcg_step, 5 trsv_fwd, 6 trsv_bwd, 7 spmv; buf = nullptr disables.
constexpr int TL_K = 10, TL_RING = 256;
void timeline_enable(unsigned long long* buf);
// Fused a5 + a6 (P_L / none, unsharded): cooperative launch; false if it could not be launched.
// Rows of C with more than KF_LONG_ROW entries (listed in `longr`) are done warp per row, the rest thread per row.
constexpr int KF_LONG_ROW = 32;
// next_rhs (phase D, after p = z + βp and one more grid sync) prepares the next F-solve's right-hand side
// u = Cᵀp, thread per row of Ct: 0 = none, 1 = flattened forest (acc / vbuf, xout = 0, as k_flat_rhs),
// 2 = dense into ubuf (as the pregather SpMV), 3 = into ubuf with xout[0, n) = 0 (dense W GEMV next),
// 4 = level products: into ubuf, acc = tacc = xout = 0 on [0, N), vbuf = u on the root's columns (as k_pi_init).
bool pcg_step(const DevCSR& Cf, const int32_t* longr, int64_t nlong, int prec, const double* D, double* p,
              const double* w, double* q, double* x, double* r, double* z, double* partial, PcgState* st, int grid,
              cudaStream_t s, int next_rhs = 0, const DevFactor* F = nullptr, const DevCSR* Ct = nullptr,
              double* xout = nullptr, double* ubuf = nullptr);
// building W: the symmetric root's x-part from S⁻¹'s lower storage; diagonal 64-blocks completed
void w_copy_root(const double* Sinv, int64_t ldx, double* W, int64_t ld, int64_t r0, int64_t n, cudaStream_t s);
void w_symmetrize_diag(double* W, int64_t ld, int64_t n, cudaStream_t s);
// x += W v, W the explicit x-block of F⁻¹ (k_dense_symv; chunks = (row block, first column block) pairs)
void dense_symv(const double* W, int64_t ld, int64_t n, const int2* chunks, int64_t nch, const SymvPlan* plan,
                const double* v, double* x,
                const int* done_flag, int sms, cudaStream_t s, bool reduce = true);
// x += the fixed-order sums of a SymvPlan's slots (the second half of dense_symv with reduce = false)
void symv_reduce(const SymvPlan* P, double* x, const int* done_flag, int sms, cudaStream_t s);
// the flattened forest's right-hand side kernel alone (k_flat_rhs), for the first PCG iteration
void flat_rhs(const DevFactor& F, const SweepRhs& r, double* x, int sms, cudaStream_t s);

void gather(double* out, const double* in, const int64_t* idx, int64_t n, const int* done, cudaStream_t s);
void scatter(double* out, const double* in, const int64_t* idx, int64_t n, const int* done, cudaStream_t s);

// ---- x-space twin (augmented system K_C, projected CG with the F factor as constraint
//      preconditioner).  Vectors of length n in factor order; W = D⁻¹.
void g_apply(const DevCSR& Hf, const DevCSR& Cf, const DevCSR& Ctf, const double* W, const double* p, double* q,
             double* partial, PcgState* st, bool pcg_mode, int grid, cudaStream_t s);
void xp_update1(int64_t n, const double* p, const double* q, double* x, double* r, double* rhs, const PcgState* st,
                int grid, cudaStream_t s);
void xp_update2(const DevCSR& Atf, int64_t m1, const double* sol, double* r, double* lam, double* p, double* partial,
                PcgState* st, bool init, int grid, cudaStream_t s);
void xp_update3(int64_t n, const double* g, double* p, const PcgState* st, int grid, cudaStream_t s);
void xp_init_r(int64_t n, const double* q, const double* f, double* r, double* rhs, int grid, cudaStream_t s);
void x_rhs(const DevCSR& Ctf, int64_t m1, const double* rg_re, const double* ra, const double* D, double* fe,
           int grid, cudaStream_t s);
void x_dnu(const DevCSR& Cf, const double* ra, const double* D, const double* dx, double* dnu, int grid,
           cudaStream_t s);
void recip(int64_t m, const double* D, double* W, int grid, cudaStream_t s);

// ---- IPM kernels (a9–a11)
void ipm_mu(int64_t m2, const double* s_, const double* nu, double* partial, IpmState* st, int grid,
            cudaStream_t s);
// ctnu: optional precomputed Cᵀν (factor order, all ranks' rows summed); NULL = from Ctf
void ipm_residuals(const DevCSR& Hf, const DevCSR& Atf, const DevCSR& Ctf, const DevCSR& Af, const DevCSR& Cf,
                   const double* gf, const double* b, const double* d, const double* x, const double* lam,
                   const double* nu, const double* s_, double* rhs_f, double* rc, double* ra, double* D,
                   double* partial, IpmState* st, int grid, cudaStream_t s, const double* ctnu = nullptr);
void ipm_rnu(const DevCSR& Cf, const double* ra, const double* y, double* rnu, int grid, cudaStream_t s);
// ctdnu: optional precomputed CᵀΔν (summed over ranks); NULL = from Ctf
void ipm_recovery_rhs(const DevCSR& Ctf, int64_t n, int64_t m1, const double* rg_re, const double* dnu,
                      double* rhs_f, int grid, cudaStream_t s, const double* ctdnu = nullptr);
void ipm_ds_alpha(int64_t m2, const double* rc, const double* nu, const double* D, const double* dnu,
                  const double* s_, double* ds, double* partial, IpmState* st, int grid, cudaStream_t s);
void ipm_update(int64_t N, int64_t m2, const double* dxl, const double* dnu, const double* ds, double* xl,
                double* nu, double* s_, const IpmState* st, int grid, cudaStream_t s);
void ipm_objective(const DevCSR& Hf, const double* gf, const double* x, double* partial, IpmState* st, int grid,
                   cudaStream_t s);

// ---- P_H setup: numeric T = C diag(H)^-1 C^T on a given pattern
void t_values(const DevCSR& Cnu /*m2×n, original cols*/, const double* hdiag, const int64_t* t_row,
              const int32_t* t_col, int64_t nnz_t, double* t_val, cudaStream_t s);

}  // namespace qpb
