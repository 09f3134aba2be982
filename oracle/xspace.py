"""Oracle for the x-space twin of PL-KF — TEST INFRASTRUCTURE ONLY.

Eliminating Δν = −D⁻¹(r_a + CΔx) (eq. delnu) from the double saddle point system gives the
augmented system K_C (eq. augmented-2):

    [ −(H + CᵀWC)  Aᵀ ] [Δx]      [r_u]        W = D⁻¹ = V S⁻¹,
    [      A        0 ] [Δλ] = −  [r_e],       r_u = r_g − CᵀW r_a,

i.e. G Δx − Aᵀ Δλ = r_u, A Δx = −r_e with G = H + CᵀWC symmetric positive definite.  The matrix-free
operator is G p = H p + Cᵀ(W∘(C p)) — the north_star's "H·p + Cᵀ(D·(C·p))".

It is solved by projected preconditioned CG with the constraint preconditioner P_CP = [E Aᵀ; A 0]
(eq. const-prec) for E = H.  Then P_CP is, up to the sign of its (1,1) block, the matrix
F = [−H Aᵀ; A 0] that is factored once, so every projection is one F-solve.
The method is the projected CG of Gould, Hribar and Nocedal, the paper's ref. gould2001solution.  It
keeps A x = e at every iterate, so the iteration runs in the nullspace Z of A.  Its preconditioned
spectrum is {1} ∪ eig((ZᵀHZ)⁻¹ ZᵀGZ).  The second set equals 1 + the nonzero
eigenvalues of W C Z (ZᵀHZ)⁻¹ ZᵀCᵀ, and so matches P_L⁻¹K_F's spectrum except for the multiplicity
of 1.  Hence "twin": the same Krylov convergence at the same F-solve cost, plus one
H-SpMV per iteration.

* x_rhs(qp, res, D)            (f = r_u, e = −r_e, W)
* G_apply(qp, W, p)            H p + Cᵀ(W∘(C p))
* project(fs, r)               (z, w) with H z + Aᵀ w = r, A z = 0  — one F-solve of [−r; 0]
* ppcg(qp, fs, W, f, e, …)     projected CG with residual update; stop when √(rᵀg) ≤ ε·√(r₀ᵀg₀);
                               Δλ = Σ of the projections' multipliers
* newton_from_x(res, D, nu, dx) Δν = −W(r_a + CΔx), Δs = −V⁻¹r_c − DΔν
"""
from __future__ import annotations

import numpy as np


def x_rhs(qp, res, D):
    """(f, e, W): f = r_u = r_g − CᵀW r_a, e = −r_e, W = D⁻¹."""
    W = 1.0 / D
    f = res["r_g"] - qp.C.T @ (W * res["r_a"])
    return f, -res["r_e"], W


def G_apply(qp, W, p):
    """G p = (H + CᵀWC) p, matrix-free (two SpMVs with C, one with H)."""
    return qp.H @ p + qp.C.T @ (W * (qp.C @ p))


def project(fs, r):
    """Constraint-preconditioner solve [H Aᵀ; A 0][z; w] = [r; 0] through F = [−H Aᵀ; A 0]:
    F [z; −w] = [−r; 0]."""
    z, v = fs.solve(-r, None)
    return z, -v


def particular(fs, e):
    """x₀ with A x₀ = e (and H x₀ ∈ range Aᵀ): F [x₀; v] = [0; e]."""
    n = fs.n
    x0, _ = fs.solve(np.zeros(n), e)
    return x0


def ppcg(qp, fs, W, f, e, tol, maxit):
    """Projected PCG for min ½xᵀGx − fᵀx s.t. Ax = e (Gould–Hribar–Nocedal, Alg. II.2 with the
    residual update of their Alg. II.3: after each projection H g + Aᵀw = r the range(Aᵀ) part Aᵀw is
    removed from r and accumulated into Δλ, so r → 0 instead of → AᵀΔλ and the projections do not
    lose accuracy to a large residual).

    Returns (Δx, Δλ, iters, relres, converged, history of √(rᵀg)/√(r₀ᵀg₀)), with G Δx − Aᵀ Δλ ≈ f.
    The iteration count is the number of G products, as in oracle.pcg."""
    x = particular(fs, e) if e is not None and len(e) else np.zeros(qp.n)
    lam = np.zeros(qp.m1)
    r = G_apply(qp, W, x) - f
    g, w = project(fs, r)
    r = r - qp.A.T @ w
    lam = lam + w
    rg = float(r @ g)
    rg0 = rg
    hist = []
    if rg0 <= 0.0:
        return x, lam, 0, 0.0, True, hist
    p = -g
    rel = 1.0
    for j in range(1, maxit + 1):
        q = G_apply(qp, W, p)
        alpha = rg / float(p @ q)
        x = x + alpha * p
        r = r + alpha * q
        g, w = project(fs, r)
        r = r - qp.A.T @ w
        lam = lam + w
        rg_new = float(r @ g)
        rel = np.sqrt(abs(rg_new) / rg0)
        hist.append(rel)
        if rel <= tol:
            return x, lam, j, rel, True, hist
        p = -g + (rg_new / rg) * p
        rg = rg_new
    return x, lam, maxit, rel, False, hist


def newton_from_x(qp, res, D, nu, dx):
    """Δν = −D⁻¹(r_a + CΔx) and Δs = −V⁻¹r_c − DΔν."""
    dnu = -(res["r_a"] + qp.C @ dx) / D
    ds = -res["r_c"] / nu - D * dnu
    return dnu, ds
