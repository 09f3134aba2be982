"""Pins for oracle/pcg.py and the spectral theorems (CPU only)."""
import numpy as np
import pytest
import scipy.sparse as sp

import qpgen
from oracle import kkt, spectral
from oracle.fsolve import DenseF
from oracle.pcg import pcg


def spd_with_spectrum(eigs, seed=0):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((len(eigs), len(eigs))))
    return Q @ np.diag(eigs) @ Q.T


def test_pcg_matches_dense_solve():
    A = spd_with_spectrum(np.linspace(1, 50, 40))
    b = np.random.default_rng(1).standard_normal(40)
    x, it, rr, ok, _ = pcg(lambda v: A @ v, b, lambda r: r.copy(), 1e-13, 500)
    ref = np.linalg.solve(A, b)
    assert ok and np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)


def test_pcg_trivial_cases():
    b = np.arange(1.0, 6.0)
    x, it, *_ = pcg(lambda v: v, b, lambda r: r.copy(), 1e-12, 10)
    assert it == 1 and np.allclose(x, b)
    d = np.array([1.0, 2.0, 3.0])
    x, it, *_ = pcg(lambda v: d * v, d, lambda r: r / d, 1e-12, 10)
    assert it == 1 and np.allclose(x, 1.0)
    x, it, rr, ok, _ = pcg(lambda v: v, np.zeros(4), lambda r: r, 1e-3, 10)
    assert it == 0 and ok and np.all(x == 0)


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_pcg_terminates_within_distinct_eigenvalues(k):
    """CG needs at most #distinct eigenvalues iterations, +2 rounding slack."""
    eigs = np.repeat(np.linspace(1.0, 4.0, k), 30 // k + 1)[:30]
    A = spd_with_spectrum(eigs, seed=k)
    b = np.random.default_rng(k).standard_normal(30)
    _, it, _, ok, _ = pcg(lambda v: A @ v, b, lambda r: r.copy(), 1e-10, 100)
    assert ok and it <= k + 2


def _state(qp, seed=0):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.3, 3.0, qp.m2)


@pytest.mark.parametrize("m1", [2, 6, 10])
def test_theorem1_PL_spectrum(m1):
    """Theorem 1: eigenvalue 1 with multiplicity ≥ max(0, m2−(n−m1)),
    all eigenvalues ≥ 1 (X is PSD)."""
    qp = qpgen.scaled_random_qp(12, m1, 20, seed=m1, g_nnz=3, a_nnz=3, c_nnz=3)
    D = _state(qp)
    K = spectral.KF_via_Finv(qp, D)
    w = spectral.precond_spectrum(K, np.diag(D))
    mult = int(np.sum(np.abs(w - 1.0) < 1e-8))
    assert mult >= max(0, qp.m2 - (qp.n - qp.m1))
    assert w.min() >= 1 - 1e-10


@pytest.mark.parametrize("m1", [1, 4, 9])
def test_theorem2_PH_exact_spectrum(m1):
    """Theorem 2: exact P_H = D + CH⁻¹Cᵀ gives eigenvalue 1 with
    multiplicity ≥ max(0, m2−m1) and all eigenvalues ≤ 1 (Y is PSD)."""
    qp = qpgen.scaled_random_qp(12, m1, 20, seed=m1, g_nnz=3, a_nnz=3, c_nnz=3)
    D = _state(qp)
    K = spectral.KF_via_Finv(qp, D)
    P = kkt.PrecondH(qp, D, exact=True).P
    w = spectral.precond_spectrum(K, P)
    mult = int(np.sum(np.abs(w - 1.0) < 1e-8))
    assert mult >= max(0, qp.m2 - qp.m1)
    assert w.max() <= 1 + 1e-10 and w.min() > 0


def test_lemma_ranks():
    """Lemma 1: rank(H̄_A) ≤ m1; Lemma 2: rank(H − H̄_A) ≤ n − m1."""
    qp = qpgen.scaled_random_qp(10, 4, 5, seed=3, g_nnz=3, a_nnz=3, c_nnz=3)
    Hb = spectral.HbarA(qp)
    H = qp.H.toarray()
    assert np.linalg.matrix_rank(Hb, tol=1e-9 * np.abs(H).max()) <= qp.m1
    assert np.linalg.matrix_rank(H - Hb, tol=1e-9 * np.abs(H).max()) <= qp.n - qp.m1


def _cg_count(qp, D, M, tol=1e-10):
    fs = DenseF(qp.H, qp.A)
    b = np.random.default_rng(7).standard_normal(qp.m2)
    _, it, _, ok, _ = pcg(lambda p: kkt.KF_apply(qp, fs, D, p), b, M, tol, 10 * qp.m2)
    return it, ok


@pytest.mark.parametrize("m1", [8, 12, 15, 16])
def test_corollary1_PL_iteration_bound(m1):
    """Corollary 1: PL-CG ≤ (n−m1)+1 iterations (+2 rounding slack);
    m1 = n gives exactly 1 iteration."""
    qp = qpgen.make_syqp(16, m1)
    D = np.random.default_rng(m1).uniform(0.5, 2.0, qp.m2)
    it, ok = _cg_count(qp, D, kkt.PrecondL(D))
    assert ok and it <= (qp.n - m1) + 1 + 2
    if m1 == qp.n:
        assert it == 1


@pytest.mark.parametrize("m1", [1, 2, 4])
def test_corollary2_PH_iteration_bound(m1):
    """Corollary 2: exact-P_H CG ≤ m1+1 iterations (+2 slack)."""
    qp = qpgen.make_syqp(16, m1)
    D = np.random.default_rng(m1).uniform(0.5, 2.0, qp.m2)
    it, ok = _cg_count(qp, D, kkt.PrecondH(qp, D, exact=True))
    assert ok and it <= m1 + 1 + 2


def test_PH_one_iteration_m1_zero_diagonal_H():
    """m1 = 0 and diagonal H: practical P_H = D + C diag(H)⁻¹ Cᵀ = K_F exactly → 1 iteration
    (Theorem 2 with m1 = 0)."""
    n, m2 = 10, 14
    rng = np.random.default_rng(0)
    H = sp.diags(rng.uniform(0.5, 2.0, n)).tocsr()
    C = qpgen.canonical_csr(sp.random(m2, n, density=0.3, random_state=1) + sp.identity(n).tocsr()[[i % n for i in range(m2)]])
    qp = qpgen.QP(H=qpgen.canonical_csr(H), A=qpgen.canonical_csr(sp.csr_matrix((0, n))), C=C,
                  g=np.zeros(n), b=np.zeros(0), d=np.zeros(m2))
    D = rng.uniform(0.5, 2.0, m2)
    it, ok = _cg_count(qp, D, kkt.PrecondH(qp, D))
    assert ok and it == 1
