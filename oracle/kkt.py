"""Oracle KKT pieces of one IPM iteration (TEST INFRASTRUCTURE ONLY).

Notation of PAPER.md §2/§4: slacks s, multipliers ν (inequalities) and λ
(equalities); S = diag(s), V = diag(ν).

* residuals            r_g, r_e, r_i, r_c (the rhs of eq. augmented,
                       P:L486–505), with the sign reading r_g = −(Hx+g−Aᵀλ−Cᵀν)
                       (reading R1) and r_a = r_i + V⁻¹r_c (R2)
* diag_D               D = V⁻¹S
* r_nu                 r_ν = −r_a + [C 0]F⁻¹(r_g; r_e)
* KF_apply             K_F p = D p − [C 0]F⁻¹[Cᵀp; 0]
* recover              F(Δx;Δλ) = −(r_g + CᵀΔν; r_e)
* delta_s              Δs = −V⁻¹r_c − DΔν
* P_L / P_H            P_L = D; P_H = D + C·diag(H)⁻¹·Cᵀ
                       and the exact form D + CH⁻¹Cᵀ (Theorem 2)
* step_length          fraction-to-boundary α = min(1, τ·α_max) (reading R3)
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def residuals(qp, x, lam, nu, s, sigma):
    """Return dict with r_g, r_e, r_i, r_c, r_a, mu and the KKT gradient."""
    m2 = qp.C.shape[0]
    mu = float(s @ nu) / m2                                   # μ = sᵀν/m2
    grad = qp.H @ x + qp.g - qp.A.T @ lam - qp.C.T @ nu       # ∇ₓ Lagrangian
    r_g = -grad                                              # reading R1 (§0.3 of SURVEY)
    r_e = qp.A @ x - qp.b
    r_i = qp.C @ x - s - qp.d
    r_c = s * nu - sigma * mu
    r_a = r_i + r_c / nu
    return dict(r_g=r_g, r_e=r_e, r_i=r_i, r_c=r_c, r_a=r_a, mu=mu, grad=grad)


def diag_D(s, nu):
    """D = V⁻¹S."""
    return s / nu


def r_nu(qp, fs, res):
    """r_ν = −r_a + [C 0] F⁻¹ (r_g; r_e)."""
    y, _ = fs.solve(res["r_g"], res["r_e"])
    return -res["r_a"] + qp.C @ y


def KF_apply(qp, fs, D, p):
    """K_F p = D∘p − [C 0] F⁻¹ [Cᵀp; 0], never forming K_F."""
    u = qp.C.T @ p
    w = fs.solve_x(u) if hasattr(fs, "solve_x") else fs.solve(u, None)[0]
    return D * p - qp.C @ w


def recover(qp, fs, res, dnu):
    """(Δx, Δλ) from F(Δx;Δλ) = −(r_g + CᵀΔν; r_e)."""
    return fs.solve(-(res["r_g"] + qp.C.T @ dnu), -res["r_e"])


def delta_s(res, D, nu, dnu):
    """Δs = −V⁻¹r_c − DΔν."""
    return -res["r_c"] / nu - D * dnu


def step_length(s, ds, nu, dnu, tau):
    """Common step α = min(1, τ·α_max), α_max = sup{α : s+αΔs ≥ 0, ν+αΔν ≥ 0} (reading R3)."""
    amax = np.inf
    neg = ds < 0
    if neg.any():
        amax = min(amax, float(np.min(-s[neg] / ds[neg])))
    neg = dnu < 0
    if neg.any():
        amax = min(amax, float(np.min(-nu[neg] / dnu[neg])))
    return min(1.0, tau * amax), amax


class PrecondL:
    """P_L = D (eq. prec-mat-1): z = r / D."""

    def __init__(self, D):
        self.D = D

    def __call__(self, r):
        return r / self.D


class PrecondNone:
    """U-KF: no preconditioner."""

    def __call__(self, r):
        return r.copy()


def chol_blocked(P, nb=2048):
    """Right-looking blocked Cholesky P = L Lᵀ, in place in the lower triangle (textbook; Golub–Van Loan
    Alg. 4.2.x): for each diagonal block k, L_kk = chol(P_kk); L_ik = P_ik L_kk⁻ᵀ; P_ij −= L_ik L_jkᵀ.
    Used for the large dense P_H (c1: 40 000²), where this image's LAPACK potrf fails beyond ~3·10⁴
    unknowns; each step calls LAPACK/BLAS only on ≤ nb-wide blocks.  Returns L (= P, lower part)."""
    n = P.shape[0]
    for k0 in range(0, n, nb):
        k1 = min(n, k0 + nb)
        P[k0:k1, k0:k1] = np.linalg.cholesky(P[k0:k1, k0:k1])
        if k1 < n:
            P[k1:, k0:k1] = sla.solve_triangular(P[k0:k1, k0:k1], P[k1:, k0:k1].T, lower=True).T
            for j0 in range(k1, n, nb):
                j1 = min(n, j0 + nb)
                P[j0:, j0:j1] -= P[j0:, k0:k1] @ P[j0:j1, k0:k1].T
    return P


def chol_blocked_solve(L, r, nb=2048):
    """x = L⁻ᵀL⁻¹r with the lower triangle of L from chol_blocked (block forward, then block backward)."""
    n = L.shape[0]
    y = np.array(r, dtype=float, copy=True)
    for k0 in range(0, n, nb):
        k1 = min(n, k0 + nb)
        y[k0:k1] = sla.solve_triangular(L[k0:k1, k0:k1], y[k0:k1], lower=True)
        if k1 < n:
            y[k1:] -= L[k1:, k0:k1] @ y[k0:k1]
    for k1 in range(n, 0, -nb):
        k0 = max(0, k1 - nb)
        if k1 < n:
            y[k0:k1] -= L[k1:, k0:k1].T @ y[k1:]
        y[k0:k1] = sla.solve_triangular(L[k0:k1, k0:k1], y[k0:k1], lower=True, trans="T")
    return y


def T_matrix(qp):
    """T = C·diag(H)⁻¹·Cᵀ, formed once in the setup phase."""
    dH = qp.H.diagonal()
    return (qp.C @ sp.diags(1.0 / dH) @ qp.C.T).tocsr()


class PrecondH:
    """P_H = D + T with T = C diag(H)⁻¹ Cᵀ, Cholesky-factored per IPM iteration.

    ``exact=True`` uses the theoretical form P_H = D + C H⁻¹ Cᵀ of Theorem 2
     — dense, tiny problems only.  ``sparse=True`` factors the sparse
    D + T with SuperLU instead of dense LAPACK Cholesky (an SPD matrix: no
    pivoting, diag_pivot_thresh = 0) in SuperLU's own minimum-degree order, or
    in the given row order with ``order="natural"`` (banded T, e.g. c4s) — the
    full-size configs.  ``keep=False`` factors the dense matrix in place (c1:
    a 40 000² matrix) and drops ``self.P``.
    """

    def __init__(self, qp, D, T=None, exact=False, sparse=False, order="mmd", keep=True):
        self.sparse = sparse and not exact
        if exact:
            Hd = qp.H.toarray()
            Cd = qp.C.toarray()
            P = Cd @ np.linalg.solve(Hd, Cd.T) + np.diag(D)
        elif self.sparse:
            Tm = T if T is not None else T_matrix(qp)
            P = (Tm + sp.diags(np.asarray(D, dtype=float))).tocsc()
            spec = "NATURAL" if order == "natural" else "MMD_AT_PLUS_A"
            self.lu = spla.splu(P, permc_spec=spec, diag_pivot_thresh=0.0, options=dict(SymmetricMode=True))
            self.P = P
            return
        else:
            P = (T if T is not None else T_matrix(qp)).toarray()
            P[np.diag_indices_from(P)] += D                  # P_H = D + T
        self.big = P.shape[0] > 8192
        if self.big:                                         # blocked: see chol_blocked
            self.L = chol_blocked(P if not keep else P.copy())
            self.P = P if keep else None
            return
        self.c = sla.cho_factor(P, lower=True, overwrite_a=not keep)
        self.P = P if keep else None

    def __call__(self, r):
        if self.sparse:
            return self.lu.solve(np.asarray(r, dtype=float))
        if self.big:
            return chol_blocked_solve(self.L, r)
        return sla.cho_solve(self.c, r)
