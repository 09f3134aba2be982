/*
 * qp_b200.h — C ABI of the B200-native single-factorization inexact IPM
 * (arXiv 2104.12916, "PAPER.md" in the citations below).
 *
 * The library solves convex QPs
 *
 *     min ½xᵀHx + gᵀx   s.t.  Ax = b,  Cx ≥ d
 *
 * with a primal-dual IPM whose Newton system is reduced to the SPD
 * inequality-constraint-reduced system (eq. ineq-const-reduced)
 *
 *     K_F Δν = r_ν,   K_F = D − [C 0] F⁻¹ [Cᵀ; 0],   F = [−H Aᵀ; A 0],
 *     r_ν = −r_a + [C 0] F⁻¹ (r_g; r_e),
 *
 * solved by PCG with P_L = D or
 * P_H = D + C·diag(H)⁻¹·Cᵀ.  F is LDLᵀ-factored ONCE
 * and every K_F product is Cᵀ-SpMV → F-solve → C-SpMV
 * (P:L144).  (Δx, Δλ) are recovered from F(Δx;Δλ) = −(r_g + CᵀΔν; r_e)
 * and Δs = −V⁻¹r_c − DΔν.
 *
 * All arithmetic is fp64 and runs in hand-written sm_100a CUDA kernels; there
 * is no CPU fallback: every compute entry point returns QP_ECUDA when no
 * usable GPU is present.
 *
 * Conventions (all entry points):
 *  - Return value: a qp_status; on error a message is kept per context
 *    (qp_last_error).  QP_MAXIT is a non-fatal status.
 *  - Ownership: every pointer argument is BORROWED for the duration of the
 *    call and never retained.  qp_setup deep-copies the problem to the GPU.
 *    Output buffers are caller-owned.
 *  - Vectors: by default host pointers (the library copies in/out).  With
 *    qp_setup_opts.vectors_on_device = 1, the vector arguments of pcg_solve,
 *    ipm_factor_once, qp_f_solve, qp_kf_apply and the x/lam/nu/s buffers of
 *    qp_ipm_result are DEVICE pointers on opts.device.
 *  - Call order: qp_setup → ipm_factor_once → any number of pcg_solve /
 *    ipm_solve / qp_ipm_* calls.  Anything else returns QP_ESTATE.
 *  - Streams: all work is issued on opts.stream (a cudaStream_t; NULL = the
 *    library's own stream).  Calls are synchronous with respect to the host.
 */
#ifndef QP_B200_H
#define QP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qp_ctx qp_ctx; /* opaque; one per process / GPU */

/* Compressed sparse row matrix, host pointers, canonical: column indices
 * sorted and unique within each row, 0-based.  nrows+1 indptr entries. */
typedef struct {
  int64_t nrows, ncols;
  const int64_t* indptr;
  const int32_t* indices;
  const double* values;
} qp_csr;

typedef enum {
  QP_OK = 0,
  QP_MAXIT = 1,        /* non-fatal: PCG stopped at maxit (the IPM continues) */
  QP_EINVAL = -1,      /* bad CSR / dimensions / non-finite input */
  QP_ENOTSPD = -2,     /* F inertia != (n negative, m1 positive): H not SPD or A
                          rank-deficient; or a P_H pivot <= 0 */
  QP_EBREAKDOWN = -3,  /* PCG breakdown: pᵀq <= 0 or non-finite */
  QP_ENOMEM = -4,
  QP_ECUDA = -5,       /* CUDA error or no usable sm_100 device */
  QP_ENCCL = -6,
  QP_ESTATE = -7       /* call order violated */
} qp_status;

typedef enum {
  QP_PREC_NONE = 0, /* U-KF: unpreconditioned CG */
  QP_PREC_LOW = 1,  /* PL-KF: P_L = D */
  QP_PREC_HIGH = 2  /* PH-KF: P_H = D + C diag(H)^-1 C^T, Cholesky per IPM iteration */
} qp_precond;

/* Cross-rank collective used by the sharded mode instead of NCCL (optional).
 * In-place all-reduce of `count` doubles at DEVICE pointer buf, ordered on the
 * cudaStream_t `stream` (the call may synchronise it); op: 0 sum, 1 max, 2 min.
 * Every rank must produce bit-identical results.  The reduced values must be visible to work enqueued on
 * `stream` after the call returns: write them with cudaMemcpyAsync on `stream` (and synchronise it), not
 * with a plain cudaMemcpy from pageable memory — that may return before its DMA lands and is not ordered
 * with a non-blocking stream.  Return 0 on success. */
typedef int (*qp_allreduce_fn)(void* user, double* buf, int64_t count, int32_t op, void* stream);

/* Neighbour exchange used by the halo mode of the sharded operator instead of NCCL send/recv (optional;
 * needed for that mode when `allreduce` is set).  Sends n_to_prev doubles at DEVICE pointer to_prev to
 * rank − 1 and n_to_next doubles at to_next to rank + 1; receives n_from_prev doubles from rank − 1 into
 * from_prev and n_from_next from rank + 1 into from_next (a count of 0: no transfer; the first rank has
 * no previous, the last no next).  Ordered on `stream` (the call may synchronise it).  0 on success. */
typedef int (*qp_halo_fn)(void* user, const double* to_prev, int64_t n_to_prev, const double* to_next,
                          int64_t n_to_next, double* from_prev, int64_t n_from_prev, double* from_next,
                          int64_t n_from_next, void* stream);

typedef struct {
  int device;              /* CUDA device ordinal */
  void* stream;            /* cudaStream_t or NULL */
  int rank, world;         /* SPMD rank / size; world = 1 for single GPU */
  const void* nccl_uid;    /* 128-byte ncclUniqueId from qp_nccl_unique_id on rank 0,
                              broadcast by the caller (sharded mode), or NULL */
  const int64_t* x_perm;   /* optional fill-reducing order of the x block (new→old,
                              length n); NULL = the library's minimum-degree order */
  int vectors_on_device;   /* see Conventions */
  int64_t workspace_limit_bytes; /* multifrontal workspace cap; 0 = 120 GiB */
  qp_allreduce_fn allreduce;     /* optional collective provider (sharded mode), else NULL */
  void* allreduce_user;          /* passed to allreduce */
  qp_halo_fn halo;               /* optional neighbour exchange (halo mode of the sharded operator), else NULL */
  void* halo_user;               /* passed to halo */
} qp_setup_opts;

/* Sharded mode (enabled when world > 1, nccl_uid != NULL or
 * allreduce != NULL).  Every rank calls every entry point collectively with the
 * same GLOBAL H, A, C, g, b, d.  The m2 inequality rows are split into
 * contiguous nnz-balanced slices (qp_partition_rows); rank r owns rows
 * [row0, row1) (qp_get_partition): its slices of C, d, D, ν, s and of every
 * PCG vector.  Per PCG iteration the partial products C_rᵀp_r are all-reduced
 * (n doubles) before the replicated F-solve, and the three PCG reductions are
 * all-reduced (the north_star's "dot products NCCL-allreduced"); the IPM
 * all-reduces Cᵀν, CᵀΔν, μ, ‖r_i‖∞ and α_max.  The x-space (x, λ, F-solves)
 * is replicated.  Then the m2-length arguments of pcg_solve, qp_kf_apply and
 * the nu / s buffers of qp_ipm_result are the rank's (row1 − row0)-row slice;
 * ipm_factor_once(QP_PREC_HIGH) returns QP_EINVAL (P_H couples all rows). */

/* Copy the QP to the GPU and validate it.  H: full symmetric n×n (both
 * triangles stored); A: m1×n, m1 >= 0 (m1 = 0 ⇒ F = −H); C: m2×n, m2 >= 1.
 * g (n), b (m1), d (m2): host arrays.  Errors: QP_EINVAL on shape/CSR/NaN
 * problems, QP_ECUDA without a GPU, QP_ENOMEM. */
int qp_setup(qp_ctx** ctx, const qp_csr* H, const qp_csr* A, const qp_csr* C,
             const double* g, const double* b, const double* d, const qp_setup_opts* opts);

/* Setup phase: ordering (x block by x_perm or minimum
 * degree, λ block last), symbolic analysis, multifrontal numeric LDLᵀ of F
 * on the GPU with static 1×1 pivots and an inertia check (x pivots < 0,
 * λ pivots > 0) → QP_ENOTSPD on failure.  For QP_PREC_HIGH also
 * T = C·diag(H)⁻¹·Cᵀ and the symbolic analysis of D + T; D0 (m2
 * values, may be NULL = ones) gives the first numeric P_H factor.  When it
 * reads fewer bytes than one F-solve (and fits), the explicit x-block
 * W = (F⁻¹)₁₁ is also formed here and guarded against an
 * F-solve (≤ 1e-10); PCG's K_F products then use it (qp_stats.dense_w_*). */
int ipm_factor_once(qp_ctx* ctx, const double* D0, qp_precond p);

/* Solve K_F(D_k) Δν = rhs from Δν = 0 by PCG with the preconditioner chosen
 * at ipm_factor_once (P_H is refactored when D_k changed).  Stop when
 * ‖r‖₂ <= tol·‖rhs‖₂ or after maxit iterations (→ QP_MAXIT).
 * D_k, rhs, dnu_out: m2 values.  iters / relres may be NULL. */
int pcg_solve(qp_ctx* ctx, const double* D_k, const double* rhs, double tol, int32_t maxit,
              double* dnu_out, int32_t* iters, double* relres);

/* x-space twin of PL-KF: solve the augmented system K_C
 *
 *     G Δx − Aᵀ Δλ = f,   A Δx = e,   G = H + Cᵀ D_k⁻¹ C,
 *
 * by projected CG (Gould–Hribar–Nocedal, the paper's ref. gould2001solution, with the residual
 * update) with the constraint preconditioner [H Aᵀ; A 0] applied through the F factor
 * of ipm_factor_once — one F-solve per iteration — and the operator G p = H p + Cᵀ(D_k⁻¹∘(C p))
 * applied matrix-free in one fused kernel.  Stops when √(rᵀg) ≤ tol·√(r₀ᵀg₀) (g the projected
 * residual) or after maxit products (QP_MAXIT).  D_k: m2 values (> 0); f, dx_out: n values in the
 * caller's x order; e, dlam_out: m1 values.  Host or device pointers per vectors_on_device.
 * QP_EINVAL in sharded mode.  iters / relres may be NULL. */
int pcg_solve_x(qp_ctx* ctx, const double* D_k, const double* f, const double* e, double tol, int32_t maxit,
                double* dx_out, double* dlam_out, int32_t* iters, double* relres);

typedef struct {
  double ipm_tol;      /* 1e-8 */
  double pcg_tol;      /* ε = 1e-3 */
  double sigma;        /* 0.1 */
  double tau;          /* 0.995 */
  int32_t max_ipm;     /* 100 */
  int32_t pcg_maxit;   /* 2000 */
  int32_t pcg_forcing; /* 1: ε_k = min(ε, μ_k) (reading R4); 0: fixed ε */
  int32_t space;       /* 0: ν-space K_F with the chosen preconditioner (default); 1: the x-space
                          twin — projected CG on the augmented system K_C (pcg_solve_x); not with
                          sharded rows */
} qp_ipm_opts;

typedef struct {
  double *x, *lam, *nu, *s; /* caller buffers (n, m1, m2, m2) or NULL */
  double objective;         /* ½xᵀHx + gᵀx */
  int32_t n_ipm;            /* IPM iterations taken (N_I) */
  int32_t* pcg_iters;       /* caller buffer of length max_ipm or NULL (n_kr per iteration) */
  int32_t status;           /* QP_OK if converged, QP_MAXIT if max_ipm reached */
  int32_t pcg_total;        /* Σ n_kr */
  double t_setup_s, t_solve_s;
  double mu, rg_inf, re_inf, ri_inf; /* final μ and residual ∞-norms */
  double alpha;             /* step length of the last IPM iteration */
} qp_ipm_result;

/* The inexact IPM (readings R1–R4): start x=0, λ=0, ν=1,
 * s=|d|+1; per iteration residuals → r_ν → PCG → recovery → Δs → common
 * fraction-to-boundary step; stop on the KKT test of DESIGN.md. */
int ipm_solve(qp_ctx* ctx, const qp_ipm_opts* o, qp_ipm_result* r);

/* Step-wise IPM control (bench / tests): qp_ipm_init resets the iterate to
 * the starting point; qp_ipm_iterate runs up to nsteps IPM iterations
 * (stopping early at convergence) and fills r (vectors only when non-NULL);
 * *done = 1 once converged. */
int qp_ipm_init(qp_ctx* ctx, const qp_ipm_opts* o);
int qp_ipm_iterate(qp_ctx* ctx, int32_t nsteps, qp_ipm_result* r, int32_t* done);

/* The reduced system of the last IPM iteration run by qp_ipm_iterate:
 * D_k (m2), r_ν (m2) and the PCG tolerance ε_k it was solved to (bench e2e
 * replay; vector conventions as above, eps a host pointer). */
int qp_ipm_last_system(qp_ctx* ctx, double* D, double* rnu, double* eps);

/* Number of CUDA kernel launches this context has issued so far. */
int64_t qp_launch_count(const qp_ctx* ctx);

/* Component entry points (parity tests; same conventions):
 * qp_f_solve:  (y; z) = F⁻¹ (r1; r2), vectors in the ORIGINAL order,
 *              rhs/out of length n + m1 (a2–a4 of SURVEY §8(a)).
 * qp_kf_apply: q = K_F(D) p (a1–a5). */
int qp_f_solve(qp_ctx* ctx, const double* rhs, double* out);

/* q = G p = H p + Cᵀ(D⁻¹∘(C p)): the x-space operator of the augmented system K_C (the
 * north_star's "H·p + Cᵀ(D·(C·p))" with D = V⁻¹S, so its D·(C·p) is D⁻¹∘(C p) here), applied without
 * any factorization — callable right after qp_setup, at sizes whose F cannot be factored (full C3/C4).
 * Two streaming kernels over C, then H and Cᵀ, in natural order.  D: m2 (this rank's rows, > 0),
 * p: n, q: n (replicated; sharded mode all-reduces the ranks' partial products).  Host or device
 * pointers per vectors_on_device.  Errors: QP_ESTATE before qp_setup, QP_ENOMEM. */
int qp_operator_apply(qp_ctx* ctx, const double* D, const double* p, double* q);

/* Halo mode of the sharded operator (BJ configs[4]: "rows are partitioned across 2/4/8 GPUs with a halo
 * exchange"; north_star: "boundary entries of p are exchanged with NCCL").  When every rank's rows of C and
 * of H reach only into the two neighbouring ranks' parts of x (band-local C, grid H), x is split into
 * contiguous OWNED ranges [own_lo, own_hi), one per rank, and one product exchanges two halos with the
 * neighbours instead of all-reducing n doubles:
 *   1. p on the rank's window [p_lo, p_hi) ⊇ owned range: the entries outside it are received from the
 *      neighbours that own them (ncclSend/ncclRecv in one group, or opts.halo);
 *   2. t = D⁻¹∘(C_g p) on the rank's rows, q = (H p on the owned rows) + C_gᵀ t on [q_lo, q_hi);
 *   3. the parts of q outside the owned range are sent to their owners and added there.
 * qp_operator_halo_plan (collective, after qp_setup) derives the plan from the rank's rows with the rule
 * "owned boundary b_g = midpoint between the last column rank g − 1 touches and the first column rank g
 * touches" and writes info[0..8) = {enabled (0/1, agreed by all ranks), own_lo, own_hi, p_lo, p_hi, q_lo,
 * q_hi, doubles this rank sends per product}.  qp_operator_apply_halo: D = the rank's m2 rows (> 0); p and
 * q full-length (n) buffers; on entry p must hold the rank's OWNED entries, on return p also holds its
 * window and q holds G p on the OWNED range (other entries unspecified).  Errors: QP_ESTATE if the plan
 * is absent or not enabled, QP_ENCCL from the exchange. */
int qp_operator_halo_plan(qp_ctx* ctx, int64_t* info);
int qp_operator_apply_halo(qp_ctx* ctx, const double* D, double* p, double* q);
int qp_kf_apply(qp_ctx* ctx, const double* D, const double* p, double* q);

/* Host-only symbolic analysis (no GPU needed): ordering of the x block
 * (x_perm or minimum degree), λ last, elimination tree, column counts,
 * supernodes, levels of the LDLᵀ factor of F.  The returned context
 * supports qp_get_structure / qp_get_stats / qp_free only. */
int qp_analyse(qp_ctx** ctx, const qp_csr* H, const qp_csr* A, const int64_t* x_perm);

/* Structure export for bit-exact parity.  which:
 *  0 perm (new→old, N = n+m1)  1 etree parent  2 column counts
 *  3 supernode starts (ns+1)   4 supernode parent  5 supernode level
 *  6 supernode row pointer (ns+1)  7 supernode rows  8 row levels
 *  9 trailing_from: first column of the forced dense trailing supernode (−1 if none)
 *  10.. the same for the P_H factor (m2 unknowns).
 * Call with out = NULL to get *len; then with a buffer of *len int64. */
int qp_get_structure(qp_ctx* ctx, int32_t which, int64_t* out, int64_t* len);

typedef struct {
  int64_t n, m1, m2, nnz_H, nnz_A, nnz_C;
  int64_t nnz_LF, n_supernodes_F, n_blocks_F, n_levels_F, row_levels_F;
  int64_t nnz_LPH, n_supernodes_PH;
  int64_t workspace_bytes, factor_bytes;
  int64_t nnz_LF_stored;             /* entries stored by the relaxed supernodes (explicit zeros incl.) */
  double c_fact_F, c_fact_PH;        /* paper model flops Σ nz(L[:,j])² */
  double t_symbolic_s, t_factor_s, t_factor_ph_s;
  double pcg_bytes_per_iter;         /* algorithmic bytes B_it */
  double pcg_flops_per_iter;         /* 2c_trsv(L_F) + 2c_spmv(C) (+2c_trsv(L_PH)) */
  double sweep_bytes_F;              /* algorithmic bytes of one L_F sweep: 8·nnz(L_F) */
  double fsolve_bytes_F;             /* bytes one F-solve must read in this implementation: 8·(2·nnz of L_F
                                        outside symmetric roots + w(w+1)/2 of each root's S⁻¹); with the
                                        flattened forest 8·(w(w+1)/2 + 2·nnz(M) + 2·nnz(L11⁻¹)) */
  double sym_discrepancy;            /* ‖y_S⁻¹ − y_X‖/‖y_X‖ of the factor-time accuracy guard */
  double sym_enabled;                /* 1 if the symmetric-root S⁻¹ shortcut is in use (guard ≤ 1e-10) */
  double flat_discrepancy;           /* ‖y_flat − y_sweeps‖/‖y_sweeps‖ of the flattened-forest guard (−1: n/a) */
  double flat_enabled;               /* 1 if F-solves use the flattened forest (M = L21·L11⁻¹) */
  double flat_nnz_M;                 /* stored entries of M */
  double dense_w_enabled;            /* 1 if PCG's K_F products use the explicit x-block W = (F⁻¹)₁₁ */
  double dense_w_discrepancy;        /* ‖W·u − (F⁻¹[u; 0])ₓ‖/‖·‖ of its factor-time guard (−1: not built) */
  double kf_bytes_W;                 /* bytes of W this rank reads per K_F product: 8·n(n+1)/2, times the
                                        rank's share of W's chunks in sharded mode (0 when not in use) */
  double dense_finv_enabled;         /* 1 if F-solves use the explicit F⁻¹ (small N, DESIGN §5 "dense F⁻¹") */
  double dense_finv_discrepancy;     /* its factor-time guard against the sweeps (−1: not built) */
  double lvl_levels_F, lvl_levels_PH;  /* leaf phase: bottom levels of L_F / L_PH swept level-synchronously
                                          (one launch per level, DESIGN §5 "leaf phase"); 0 = none */
  double lvl_supernodes_F, lvl_supernodes_PH;  /* supernodes in those levels */
  double pi_enabled;                 /* 1 if F-solves sweep the levels above the leaf phase as level products
                                        (Z_J = [L_JJ⁻¹; L_ext,J L_JJ⁻¹], one kernel per level) */
  double pi_discrepancy;             /* their factor-time guard against the task-graph sweeps (−1: not built) */
  double pi_levels;                  /* levels swept that way */
  double pi_subtrees;                /* subtrees below them swept by one warp each (0: the leaf phase instead) */
  double pi_fsolve_ms, sweep_fsolve_ms; /* factor-time medians of one F-solve through the level products / the
                                        task-graph sweeps: the faster path is kept (0: not timed) */
} qp_stats;
int qp_get_stats(qp_ctx* ctx, qp_stats* s);

/* Kernel-time accounting with CUDA events on the library stream.
 * qp_profile(ctx, 1) enables, 0 disables and clears.  qp_profile_read
 * returns, per class, accumulated ms and launch count:
 *  0 F forward sweep (or flattened forward product), 1 F backward sweep (or
 *  flattened backward product), 2 K_F q-SpMV (a5), 3 PCG vector updates (a6),
 *  4 P_H sweeps (a7), 5 P_H refactor (a8), 6 IPM rhs (a9), 7 other,
 *  8 symmetric-root GEMV of the F-solve, 9 dense W GEMV of a PCG K_F product (10 entries each). */
int qp_profile(qp_ctx* ctx, int32_t enable);
int qp_profile_read(qp_ctx* ctx, double* ms /*10*/, int64_t* count /*10*/);

/* Debug instrumentation of the L_F sweeps: enable = 1 resets and enables;
 * enable = 0 disables and copies 80 int64 = [fwd, bwd] × [DIAG, TILE, PREP,
 * XCHUNK, SNF, SCHUNK, ROOTB, SNW] × [count, wait ns, busy ns, first start ns, last end ns]. */
int qp_debug_sweep_profile(qp_ctx* ctx, int32_t enable, int64_t* out);

/* Debug: per-task trace of the sweeps profiled by the last enable/disable pair of
 * qp_debug_sweep_profile.  sweep 0 = forward, 1 = backward.  Writes min(cap, #tasks)
 * records of 6 int64 to out (host, caller-owned), indexed by dispatch ticket:
 * [task word | SM id << 32, start, dependency met, marker a, marker b, end] in
 * globaltimer ns; markers are task-type specific (0 = unused).
 * Returns the number of records, or a negative qp_status. */
int64_t qp_debug_sweep_trace(qp_ctx* ctx, int32_t sweep, int64_t* out, int64_t cap);

/* Debug: launch timeline of the instrumented kernels (0 flat rhs, 1 flat forward, 2 root GEMV,
 * 3 flat backward, 4 fused PCG step, 5 forward sweep, 6 backward sweep, 7 SpMV, 8 / 9 leaf-phase
 * level kernels forward / backward).  enable = 1
 * resets the device buffer and turns recording on (kernels read the switch at run time, so
 * captured CUDA graphs are recorded too); enable = 0 turns it off and copies
 * min(cap, W) uint64 words to out (host, caller-owned), W = 2*10 + 2*10*256:
 * [10 launch counters][10 scratch][10][256] earliest block start, [10][256] latest block end
 * (globaltimer ns; slot = launch number, the first 256 launches per kernel after enable).
 * Returns W or a negative qp_status. */
int64_t qp_debug_timeline(qp_ctx* ctx, int32_t enable, int64_t* out, int64_t cap);

/* Host-only: the contiguous split of m2 rows (CSR indptr, m2+1 entries) over
 * `world` ranks balancing nnz+1 per row; bounds (caller-owned, world+1 entries)
 * receives row offsets, bounds[0] = 0, bounds[world] = m2.  Deterministic. */
int qp_partition_rows(const int64_t* indptr, int64_t m2, int32_t world, int64_t* bounds);

/* This context's inequality-row slice [row0, row1) of m2_global rows (row0 = 0,
 * row1 = m2_global when not sharded).  Any pointer may be NULL. */
int qp_get_partition(qp_ctx* ctx, int64_t* row0, int64_t* row1, int64_t* m2_global);

/* Host-only: a fresh ncclUniqueId (128 bytes into out) for qp_setup_opts.nccl_uid.
 * NCCL is loaded on demand (dlopen libnccl.so.2); QP_ENCCL when unavailable. */
int qp_nccl_unique_id(void* out);

const char* qp_last_error(const qp_ctx* ctx);
void qp_free(qp_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* QP_B200_H */
