"""GPU: the failure paths of the C ABI (include/qp_b200.h qp_status).

QP_ENOTSPD is the inertia check of the LDLᵀ of F (F is nonsingular with inertia
(n negative, m1 positive) exactly when H is SPD and A has full row rank; the static 1×1 pivots of
the x block must be negative and those of the λ block positive, DESIGN reading R5) and the
positivity of the P_H Cholesky pivots (P_H = D + T is SPD for D > 0).
"""
import numpy as np
import pytest
import scipy.sparse as sp

import qpgen

pytestmark = pytest.mark.gpu


def _solver(qp):
    from paper_2104_12916_b200.binding import from_qp
    return from_qp(qp)


def _code(exc):
    return getattr(exc.value, "code", None)


def test_enotspd_indefinite_H():
    """H negative definite: every x pivot of −H is positive, the wrong sign → QP_ENOTSPD."""
    from paper_2104_12916_b200.binding import QPError
    qp = qpgen.scaled_random_qp(60, 10, 80, seed=21)
    qp.H = qpgen.canonical_csr(-qp.H)
    s = _solver(qp)
    with pytest.raises(QPError) as e:
        s.ipm_factor_once("low")
    assert _code(e) == -2


def test_enotspd_rank_deficient_A():
    """A with an empty row (structurally rank-deficient): its λ pivot is exactly 0 → QP_ENOTSPD
    (or the input is rejected up front with QP_EINVAL)."""
    from paper_2104_12916_b200.binding import QPError
    qp = qpgen.scaled_random_qp(60, 10, 80, seed=22)
    A = qp.A.tolil()
    A[3, :] = 0
    qp.A = qpgen.canonical_csr(A.tocsr())
    assert np.diff(qp.A.indptr)[3] == 0
    s = _solver(qp)
    with pytest.raises(QPError) as e:
        s.ipm_factor_once("low")
    assert _code(e) in (-2, -1)


def test_enotspd_ph_nonpositive_D():
    """P_H = D + T with D ≤ 0 on a row with no C entries is not SPD → QP_ENOTSPD from the P_H factor."""
    from paper_2104_12916_b200.binding import QPError
    qp = qpgen.scaled_random_qp(40, 8, 50, seed=23)
    s = _solver(qp)
    D0 = np.full(qp.m2, -1.0)
    with pytest.raises(QPError) as e:
        s.ipm_factor_once("high", D0=D0)
    assert _code(e) in (-2, -1)


def test_recovers_after_failed_ph_refactor():
    """A failed P_H refactor inside pcg_solve reports QP_ENOTSPD; the context stays usable with a valid D."""
    from paper_2104_12916_b200.binding import QPError
    qp = qpgen.scaled_random_qp(40, 8, 50, seed=24)
    s = _solver(qp)
    D = np.ones(qp.m2)
    s.ipm_factor_once("high", D0=D)
    b = np.random.default_rng(0).standard_normal(qp.m2)
    with pytest.raises(QPError) as e:
        s.pcg_solve(-D, b, tol=1e-10, maxit=100)
    assert _code(e) in (-2, -1)
    x, it, rr, rc = s.pcg_solve(D, b, tol=1e-10, maxit=100)
    assert rc == 0 and rr <= 1e-10
