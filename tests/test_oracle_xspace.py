"""Pins of the x-space twin oracle (oracle/xspace.py) — no GPU.

* the augmented system K_C solved by projected CG equals a dense solve of
  [G −Aᵀ; A 0] (numpy), and Δν = −D⁻¹(r_a + CΔx) completes the brute-force Newton step;
* every PPCG iterate satisfies A x = e (the projection invariant);
* the preconditioned spectrum is {1} ∪ eig((ZᵀHZ)⁻¹ZᵀGZ) and its non-unit part equals
  P_L⁻¹K_F's (Theorem 1 setting) — computed independently from dense matrices;
* iteration counts track PL-KF's (same Krylov spectrum) and respect Corollary 1's (n − m1) + 1 bound;
* the x-space IPM reaches the ν-space IPM's optimum.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import qpgen
from oracle import kkt, xspace
from oracle.fsolve import DenseF
from oracle.ipm import ipm_solve
from oracle.pcg import pcg
from test_oracle_fsolve_kkt import newton_brute_force, tiny


def _state(qp, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(qp.n)
    lam = rng.standard_normal(qp.m1)
    nu = rng.uniform(0.2, 2, qp.m2)
    s = rng.uniform(0.2, 2, qp.m2)
    return x, lam, nu, s


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_ppcg_solves_augmented_system_and_gives_newton_step(seed):
    qp = tiny(10, 4, 14, seed=seed)
    x, lam, nu, s = _state(qp, seed + 20)
    res = kkt.residuals(qp, x, lam, nu, s, 0.1)
    D = kkt.diag_D(s, nu)
    fs = DenseF(qp.H, qp.A)
    f, e, W = xspace.x_rhs(qp, res, D)
    dx, dlam, it, rel, conv, _ = xspace.ppcg(qp, fs, W, f, e, 1e-14, 500)
    assert conv
    # dense augmented system, written out from P:L507–522
    Hd, Ad, Cd = qp.H.toarray(), qp.A.toarray(), qp.C.toarray()
    G = Hd + Cd.T @ np.diag(W) @ Cd
    KC = np.block([[-G, Ad.T], [Ad, np.zeros((qp.m1, qp.m1))]])
    sol = np.linalg.solve(KC, -np.concatenate([f, res["r_e"]]))
    assert np.linalg.norm(dx - sol[:qp.n]) <= 1e-10 * max(1, np.linalg.norm(sol[:qp.n]))
    assert np.linalg.norm(dlam - sol[qp.n:]) <= 1e-9 * max(1, np.linalg.norm(sol[qp.n:]))
    dnu, ds = xspace.newton_from_x(qp, res, D, nu, dx)
    bx, bl, bn, bs = newton_brute_force(qp, x, lam, nu, s, 0.1)
    for a, b in ((dx, bx), (dlam, bl), (dnu, bn), (ds, bs)):
        assert np.linalg.norm(a - b) <= 1e-9 * max(1.0, np.linalg.norm(b))


def test_ppcg_iterates_stay_feasible():
    qp = tiny(12, 5, 16, seed=3)
    x, lam, nu, s = _state(qp, 7)
    res = kkt.residuals(qp, x, lam, nu, s, 0.1)
    D = kkt.diag_D(s, nu)
    fs = DenseF(qp.H, qp.A)
    f, e, W = xspace.x_rhs(qp, res, D)
    for k in (1, 2, 5):
        dx, *_ = xspace.ppcg(qp, fs, W, f, e, 0.0, k)
        assert np.linalg.norm(qp.A @ dx - e) <= 1e-12 * (1 + np.linalg.norm(e))


@pytest.mark.parametrize("m1", [2, 5, 9])
def test_spectrum_matches_pl_kf(m1):
    """Non-unit eigenvalues of (ZᵀHZ)⁻¹ZᵀGZ == non-unit eigenvalues of D⁻¹K_F (both dense)."""
    n, m2 = 12, 9
    qp = tiny(n, m1, m2, seed=m1)
    rng = np.random.default_rng(m1)
    D = rng.uniform(0.1, 5.0, m2)
    Hd, Ad, Cd = qp.H.toarray(), qp.A.toarray(), qp.C.toarray()
    Z = sla.null_space(Ad)
    G = Hd + Cd.T @ np.diag(1 / D) @ Cd
    ex = np.sort(sla.eigh(Z.T @ G @ Z, Z.T @ Hd @ Z, eigvals_only=True))
    fs = DenseF(qp.H, qp.A)
    KF = np.column_stack([kkt.KF_apply(qp, fs, D, e) for e in np.eye(m2)])
    ek = np.sort(np.linalg.eigvals(np.diag(1 / D) @ KF).real)
    nx = ex[np.abs(ex - 1) > 1e-8]
    nk = ek[np.abs(ek - 1) > 1e-8]
    assert len(nx) == len(nk) and np.allclose(nx, nk, rtol=1e-8)
    assert np.all(ex >= 1 - 1e-10)                          # G ⪰ H on the nullspace


@pytest.mark.parametrize("m1", [3, 6])
def test_iteration_counts_track_pl_kf(m1):
    n, m2 = 14, 18
    qp = tiny(n, m1, m2, seed=10 + m1)
    x, lam, nu, s = _state(qp, m1)
    res = kkt.residuals(qp, x, lam, nu, s, 0.1)
    D = kkt.diag_D(s, nu)
    fs = DenseF(qp.H, qp.A)
    f, e, W = xspace.x_rhs(qp, res, D)
    _, _, itx, _, convx, _ = xspace.ppcg(qp, fs, W, f, e, 1e-10, 200)
    rnu = kkt.r_nu(qp, fs, res)
    _, itn, _, convn, _ = pcg(lambda p: kkt.KF_apply(qp, fs, D, p), rnu, kkt.PrecondL(D), 1e-10, 200)
    assert convx and convn
    assert itx <= (n - m1) + 1 + 2 and itn <= (n - m1) + 1 + 2   # Corollary 1
    assert abs(itx - itn) <= 3


def test_xspace_ipm_reaches_nu_space_optimum():
    qp = qpgen.make("c0")
    rn = ipm_solve(qp, precond="low", ipm_tol=1e-10)
    rx = ipm_solve(qp, space="x", ipm_tol=1e-10)
    assert rn.converged and rx.converged
    assert abs(rx.objective - rn.objective) <= 1e-8 * max(1, abs(rn.objective))
