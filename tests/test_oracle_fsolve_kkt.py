"""Pins for oracle/fsolve.py and oracle/kkt.py (CPU only).

Each test checks the oracle against something other than itself: numpy's
dense inverse, the eigen-decomposition, the Newton system written from the
KKT conditions, SPEC.md's hand examples (tests/golden/spec_examples.json).
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

import qpgen
from oracle import kkt, spectral
from oracle.fsolve import DenseF, SparseF, assemble_F
from oracle.pcg import pcg

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def tiny(n=7, m1=3, m2=9, seed=1):
    return qpgen.scaled_random_qp(n, m1, m2, seed=seed, g_nnz=3, a_nnz=3, c_nnz=3)


@pytest.mark.parametrize("shape", [(7, 3, 9), (12, 0, 15), (10, 10, 6), (30, 8, 40)])
def test_denseF_matches_numpy_inverse(shape):
    qp = tiny(*shape)
    F = assemble_F(qp.H, qp.A).toarray()
    fs = DenseF(qp.H, qp.A)
    rng = np.random.default_rng(0)
    r1, r2 = rng.standard_normal(qp.n), rng.standard_normal(qp.m1)
    y, z = fs.solve(r1, r2)
    ref = np.linalg.solve(F, np.concatenate([r1, r2]))
    sol = np.concatenate([y, z])
    assert np.linalg.norm(sol - ref) <= 1e-13 * np.linalg.cond(F) * np.linalg.norm(ref)
    res = F @ np.concatenate([y, z]) - np.concatenate([r1, r2])
    assert np.linalg.norm(res) <= 1e-12 * np.linalg.norm(F, 2) * np.linalg.norm(np.concatenate([y, z]))


def test_F_inertia_haynsworth():
    """inertia(F) = (n negative, m1 positive)."""
    qp = tiny(20, 6, 25)
    w = np.linalg.eigvalsh(assemble_F(qp.H, qp.A).toarray())
    assert (w < 0).sum() == qp.n and (w > 0).sum() == qp.m1


def test_sparseF_matches_denseF_with_perm():
    qp = qpgen.make("c0")
    perm = np.random.default_rng(3).permutation(qp.n)
    d = DenseF(qp.H, qp.A)
    s = SparseF(qp.H, qp.A, perm)
    rng = np.random.default_rng(1)
    r1, r2 = rng.standard_normal(qp.n), rng.standard_normal(qp.m1)
    y1, z1 = d.solve(r1, r2)
    y2, z2 = s.solve(r1, r2)
    assert np.linalg.norm(y1 - y2) <= 1e-10 * np.linalg.norm(y1)
    assert np.linalg.norm(z1 - z2) <= 1e-10 * np.linalg.norm(z1)


def test_KF_two_ways_and_operator():
    """K_F = D − C(F⁻¹)₁₁Cᵀ = D + CH⁻¹(H−H̄_A)H⁻¹Cᵀ."""
    qp = tiny(9, 4, 12, seed=5)
    D = np.random.default_rng(2).uniform(0.1, 3.0, qp.m2)
    K1 = spectral.KF_via_Finv(qp, D)
    K2 = spectral.KF_via_schur(qp, D)
    fs = DenseF(qp.H, qp.A)
    K3 = np.column_stack([kkt.KF_apply(qp, fs, D, e) for e in np.eye(qp.m2)])
    scale = np.abs(K1).max()
    assert np.abs(K1 - K2).max() <= 1e-12 * scale
    assert np.abs(K1 - K3).max() <= 1e-12 * scale
    assert np.linalg.eigvalsh(0.5 * (K1 + K1.T)).min() > 0          # SPD
    assert np.abs(K1 - K1.T).max() <= 1e-12 * scale


def newton_brute_force(qp, x, lam, nu, s, sigma):
    """Newton step on the perturbed KKT conditions, written from the math:
    Hx+g−Aᵀλ−Cᵀν = 0, Ax=b, Cx−s=d, s∘ν=σμ."""
    H, A, C = qp.H.toarray(), qp.A.toarray(), qp.C.toarray()
    n, m1, m2 = qp.n, qp.m1, qp.m2
    mu = s @ nu / m2
    J = np.zeros((n + m1 + 2 * m2,) * 2)
    J[:n, :n] = H
    J[:n, n:n + m1] = -A.T
    J[:n, n + m1:n + m1 + m2] = -C.T
    J[n:n + m1, :n] = A
    J[n + m1:n + m1 + m2, :n] = C
    J[n + m1:n + m1 + m2, n + m1 + m2:] = -np.eye(m2)
    J[n + m1 + m2:, n + m1:n + m1 + m2] = np.diag(s)
    J[n + m1 + m2:, n + m1 + m2:] = np.diag(nu)
    F = np.concatenate([H @ x + qp.g - A.T @ lam - C.T @ nu, A @ x - qp.b, C @ x - s - qp.d,
                        s * nu - sigma * mu])
    d = np.linalg.solve(J, -F)
    return d[:n], d[n:n + m1], d[n + m1:n + m1 + m2], d[n + m1 + m2:]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_reduced_route_gives_newton_direction(seed):
    """r_ν → CG(1e-13) → recovery → Δs equals the brute-force Newton step (pins
    the residual signs R1/R2 and eqs. delz, ineq-const-reduced, schur-delta-x)."""
    qp = tiny(8, 3, 10, seed=seed)
    rng = np.random.default_rng(seed + 10)
    x = rng.standard_normal(qp.n)
    lam = rng.standard_normal(qp.m1)
    nu = rng.uniform(0.2, 2, qp.m2)
    s = rng.uniform(0.2, 2, qp.m2)
    res = kkt.residuals(qp, x, lam, nu, s, 0.1)
    fs = DenseF(qp.H, qp.A)
    D = kkt.diag_D(s, nu)
    rnu = kkt.r_nu(qp, fs, res)
    dnu, it, _, _, _ = pcg(lambda p: kkt.KF_apply(qp, fs, D, p), rnu, kkt.PrecondL(D), 1e-14, 500)
    dx, dlam = kkt.recover(qp, fs, res, dnu)
    ds = kkt.delta_s(res, D, nu, dnu)
    bx, bl, bn, bs = newton_brute_force(qp, x, lam, nu, s, 0.1)
    for a, b in ((dx, bx), (dlam, bl), (dnu, bn), (ds, bs)):
        assert np.linalg.norm(a - b) <= 1e-9 * max(1.0, np.linalg.norm(b))


def test_spec_residual_example():
    e = GOLD["residuals"][0]
    m2 = e["m2"]
    qp = qpgen.QP(H=sp.identity(3, format="csr"), A=sp.csr_matrix((1, 3)), C=sp.csr_matrix(np.ones((m2, 3))),
                  g=np.zeros(3), b=np.zeros(1), d=np.zeros(m2))
    res = kkt.residuals(qp, np.zeros(3), np.zeros(1), np.ones(m2), np.ones(m2), sigma=1.0)
    assert res["mu"] == 1.0 and np.all(res["r_c"] == 0.0)


def test_spec_step_length():
    e = GOLD["step_lengths"][0]
    a, _ = kkt.step_length(np.array(e["s"]), np.array(e["ds"]), np.ones(1), np.zeros(1), e["tau"])
    assert a == pytest.approx(e["alpha"], rel=1e-15)
    a0, _ = kkt.step_length(np.ones(3), np.zeros(3), np.ones(3), np.zeros(3), 0.995)
    assert a0 == 1.0
    a1, _ = kkt.step_length(np.ones(3), np.ones(3), np.ones(3), np.ones(3), 0.995)
    assert a1 == 1.0


def test_step_length_nu_branch():
    """The ν side of the fraction-to-boundary rule (reading R3), by hand: s + αΔs ≥ 0 never binds
    (Δs ≥ 0); ν = (1, 4), Δν = (−2, −1) hits zero first at α = 1/2 (row 0) ⇒ α_max = 1/2,
    α = 0.995/2.  Mixed: the s side binds at 1/4 (s = 1, Δs = −4) before ν's 1/2."""
    a, amax = kkt.step_length(np.array([1.0, 2.0]), np.array([0.5, 1.0]), np.array([1.0, 4.0]),
                              np.array([-2.0, -1.0]), 0.995)
    assert amax == 0.5 and a == pytest.approx(0.4975, rel=1e-15)
    a, amax = kkt.step_length(np.array([1.0]), np.array([-4.0]), np.array([1.0]), np.array([-2.0]), 0.995)
    assert amax == 0.25 and a == pytest.approx(0.995 * 0.25, rel=1e-15)
    a, amax = kkt.step_length(np.array([1.0]), np.array([-1.0]), np.array([3.0]), np.array([-12.0]), 0.5)
    assert amax == 0.25 and a == 0.125


def test_spec_build_ph():
    e = GOLD["build_ph"][0]
    n = e["n"]
    qp = qpgen.QP(H=sp.csr_matrix(e["h"] * np.eye(n)), A=sp.csr_matrix((0, n)), C=sp.identity(n, format="csr"),
                  g=np.zeros(n), b=np.zeros(0), d=np.zeros(n))
    P = kkt.PrecondH(qp, np.full(n, e["D"]))
    assert np.allclose(P.P, e["PH_diag"] * np.eye(n), atol=1e-15)
    assert np.allclose(P(np.full(n, e["apply_in"])), e["apply_out"], rtol=1e-14)


def test_spec_kf_operator_n1():
    e = GOLD["kf_operator"][0]
    qp = qpgen.QP(H=sp.csr_matrix([[e["H"]]]), A=sp.csr_matrix([[e["A"]]]), C=sp.csr_matrix([[e["C"]]]),
                  g=np.zeros(1), b=np.zeros(1), d=np.zeros(1))
    fs = DenseF(qp.H, qp.A)
    q = kkt.KF_apply(qp, fs, np.array([e["D"]]), np.array([1.0]))
    assert q[0] == pytest.approx(e["KF"], abs=1e-15)


def test_T_matrix_closed_form():
    """T = C diag(H)⁻¹ Cᵀ against the dense triple product."""
    qp = tiny(10, 2, 14, seed=4)
    T = kkt.T_matrix(qp).toarray()
    Cd = qp.C.toarray()
    ref = Cd @ np.diag(1.0 / qp.H.diagonal()) @ Cd.T
    assert np.allclose(T, ref, rtol=1e-14, atol=1e-14)


def test_chol_blocked_matches_lapack():
    """The blocked Cholesky used for large dense P_H (c1) against LAPACK on a small SPD matrix with
    ragged blocks: L Lᵀ = P, L equals numpy's factor, and the blocked solve inverts P."""
    rng = np.random.default_rng(8)
    n = 301
    G = rng.standard_normal((n, n))
    P = G @ G.T + n * np.eye(n)
    L = kkt.chol_blocked(P.copy(), nb=64)
    Lo = np.tril(L)
    assert np.allclose(Lo @ Lo.T, P, rtol=1e-13, atol=1e-10)
    assert np.allclose(Lo, np.linalg.cholesky(P), rtol=1e-12, atol=1e-12)
    r = rng.standard_normal(n)
    x = kkt.chol_blocked_solve(L, r, nb=64)
    assert np.linalg.norm(P @ x - r) <= 1e-12 * np.linalg.norm(r) * np.linalg.cond(P)


def test_blockf_matches_dense_block_inverse():
    """BlockF (SuperLU of H + dense F_H) against numpy.linalg.inv(F) on small QPs, with and without x_perm."""
    from oracle.fsolve import BlockF
    for qp in (tiny(40, 9, 50, seed=31), qpgen.make_grid_qp(10, 12, 20, seed=5, name="g10")):
        F = assemble_F(qp.H, qp.A).toarray()
        rng = np.random.default_rng(2)
        r = rng.standard_normal(qp.n + qp.m1)
        ref = np.linalg.inv(F) @ r
        for xp in (None, qp.x_perm):
            if xp is None and qp.x_perm is not None:
                continue
            y, z = BlockF(qp.H, qp.A, xp).solve(r[:qp.n], r[qp.n:])
            assert np.linalg.norm(np.concatenate([y, z]) - ref) <= 1e-11 * np.linalg.norm(ref)


def test_dense_explicit_w_matches_solve():
    """DenseF's written-out (F⁻¹)₁₁ (used for c1's K_F products) equals the x-part of F⁻¹[u; 0]
    computed by numpy.linalg.inv(F)."""
    qp = tiny(30, 7, 40, seed=41)
    fs = DenseF(qp.H, qp.A, explicit_w=True)
    Finv = np.linalg.inv(assemble_F(qp.H, qp.A).toarray())
    assert np.allclose(fs.W, Finv[:qp.n, :qp.n], rtol=1e-10, atol=1e-12)
    u = np.random.default_rng(3).standard_normal(qp.n)
    assert np.allclose(fs.solve_x(u), fs.solve(u, None)[0], rtol=1e-11, atol=1e-12)


def test_direct_ipm_dense_kf_route_matches_column_route():
    """The oracle's direct IPM with K_F = D − C W Cᵀ (explicit W) follows the same iterates as the
    column-by-column K_F route on a small QP (the c1 objective golden is made this way)."""
    from oracle.ipm import ipm_solve
    qp = tiny(40, 10, 60, seed=42)
    a = ipm_solve(qp, precond="low", ipm_tol=1e-10, fs=DenseF(qp.H, qp.A), direct=True)
    b = ipm_solve(qp, precond="low", ipm_tol=1e-10, fs=DenseF(qp.H, qp.A, explicit_w=True), direct=True)
    assert a.converged and b.converged and a.n_ipm == b.n_ipm
    assert abs(a.objective - b.objective) <= 1e-11 * abs(a.objective)
