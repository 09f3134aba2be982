"""The paper's flop-cost model (TEST INFRASTRUCTURE ONLY).

Kernel costs:
    c_fact(X)            = Σ_j nz(L_X[:,j])²
    c_trsv(L_X)          = 2 nz(L_X)
    c_spmv(B)            = 2 nz(B)
    c_spmm(Bᵀ, D1 B)     = Σ_i nz(B[i,:])²
    c_spmm(B, D2 Bᵀ)     = Σ_j nz(B[:,j])²
    c_norm(X)            = nz(X)
c_rhs = N_I [c_spmv(H) + 2 c_spmv(A) + 2 c_spmv(C)]

Per-variant totals (Table tab:costs P:L173–203) for the two
methods of the paper, with per-IPM-iteration n_kr summed (not averaged).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def c_fact(colcounts):
    cc = np.asarray(colcounts, dtype=np.int64)
    return int(np.sum(cc * cc))


def c_trsv(nnz_L):
    return 2 * int(nnz_L)


def c_spmv(B):
    return 2 * int(sp.csr_matrix(B).nnz)


def c_spmm_BtDB(B):
    B = sp.csr_matrix(B)
    return int(np.sum(np.diff(B.indptr).astype(np.int64) ** 2))


def c_spmm_BDBt(B):
    B = sp.csc_matrix(B)
    return int(np.sum(np.diff(B.indptr).astype(np.int64) ** 2))


def c_rhs(qp, N_I):
    return N_I * (c_spmv(qp.H) + 2 * c_spmv(qp.A) + 2 * c_spmv(qp.C))


def pl_kf(qp, cf_F, nnz_LF, n_kr):
    """PL-KF (and U-KF) total: c_fact(F) + Σ_k [4c_trsv + 2c_spmv(C) + 2n_kr c_trsv + 2n_kr c_spmv(C)] + c_rhs."""
    n_kr = list(n_kr)
    N_I = len(n_kr)
    t, s = c_trsv(nnz_LF), c_spmv(qp.C)
    return cf_F + sum(4 * t + 2 * s + 2 * k * t + 2 * k * s for k in n_kr) + c_rhs(qp, N_I)


def ph_kf(qp, cf_F, nnz_LF, cf_PH, nnz_LPH, n_kr):
    """PH-KF total + c_rhs."""
    n_kr = list(n_kr)
    N_I = len(n_kr)
    t, s, tp = c_trsv(nnz_LF), c_spmv(qp.C), c_trsv(nnz_LPH)
    return (cf_F + c_spmm_BDBt(qp.C)
            + sum(4 * t + 2 * s + 2 * k * t + 2 * k * s + cf_PH + 2 * k * tp for k in n_kr)
            + c_rhs(qp, N_I))


def pcg_iteration_flops(nnz_LF, nnz_C, nnz_LPH=0):
    """Model flops of one PCG step: 2c_trsv(L_F) + 2c_spmv(C) (+ 2c_trsv(L_PH))."""
    return 2 * c_trsv(nnz_LF) + 2 * 2 * int(nnz_C) + 2 * c_trsv(nnz_LPH)


def pcg_iteration_bytes(nnz_LF, nnz_C, n, m1, m2, nnz_LPH=0):
    """Algorithmic HBM bytes of one PCG step:
    B_it = 16·nnz(L_F) + 24·nnz(C) + 8·(15·m2 + 6·(n+m1)) (+ 16·nnz(L_PH))."""
    return 16 * int(nnz_LF) + 24 * int(nnz_C) + 8 * (15 * m2 + 6 * (n + m1)) + 16 * int(nnz_LPH)
