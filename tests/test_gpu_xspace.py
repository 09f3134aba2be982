"""GPU parity of the x-space twin (pcg_solve_x, qp_ipm_opts.space = 1) against oracle/xspace.py.

Tolerances as for the ν-space path (BASELINE north_star): solutions 1e-8 relative at fixed iteration
counts and at a tight tolerance, counts ±2, IPM objective 1e-8 relative + KKT at the GPU solution."""
import numpy as np
import pytest

import qpgen
from oracle import kkt, xspace
from oracle.fsolve import DenseF, SparseF
from oracle.ipm import ipm_solve as oracle_ipm

pytestmark = pytest.mark.gpu

CASES = {
    "tiny": lambda: qpgen.scaled_random_qp(9, 4, 12, seed=1, g_nnz=3, a_nnz=3, c_nnz=3),
    "m1_zero": lambda: qpgen.scaled_random_qp(30, 0, 40, seed=2, g_nnz=3, a_nnz=3, c_nnz=3),
    "c0": lambda: qpgen.make("c0"),
    "ragged": lambda: qpgen.scaled_random_qp(700, 130, 900, seed=3),
}


@pytest.fixture(scope="module", params=list(CASES))
def case(request):
    from paper_2104_12916_b200.binding import from_qp
    qp = CASES[request.param]()
    s = from_qp(qp)
    s.ipm_factor_once("low")
    return request.param, qp, s


def _system(qp, seed):
    rng = np.random.default_rng(seed)
    D = rng.uniform(0.2, 5.0, qp.m2)
    f = rng.standard_normal(qp.n)
    e = rng.standard_normal(qp.m1)
    return D, f, e


def test_pcg_x_matches_oracle(case):
    name, qp, s = case
    fs = DenseF(qp.H, qp.A) if qp.n + qp.m1 <= 3000 else SparseF(qp.H, qp.A)
    D, f, e = _system(qp, 5)
    W = 1.0 / D
    for tol, maxit in ((0.0, 1), (0.0, 3), (1e-12, 3000)):
        dx, dl, it, rr, rc = s.pcg_solve_x(D, f, e, tol=tol, maxit=maxit)
        ox, ol, oit, orr, oconv, _ = xspace.ppcg(qp, fs, W, f, e, tol, maxit)
        if tol == 0.0:
            assert it == oit == maxit
        else:   # late CG steps at 1e-12 are rounding-decided (DESIGN R12): ±max(2, 5 %)
            assert abs(it - oit) <= max(2, 0.05 * oit)
        assert np.linalg.norm(dx - ox) <= 1e-8 * max(1.0, np.linalg.norm(ox)), (name, tol, maxit)
        if qp.m1:
            assert np.linalg.norm(dl - ol) <= 1e-8 * max(1.0, np.linalg.norm(ol)), (name, tol, maxit)
    # the converged solution solves the augmented system
    dx, dl, it, rr, rc = s.pcg_solve_x(D, f, e, tol=1e-12, maxit=3000)
    G = lambda v: xspace.G_apply(qp, W, v)
    assert np.linalg.norm(G(dx) - qp.A.T @ dl - f) <= 1e-8 * (np.linalg.norm(f) + 1)
    if qp.m1:
        assert np.linalg.norm(qp.A @ dx - e) <= 1e-10 * (np.linalg.norm(e) + 1)


def test_xspace_ipm_matches_oracle(case):
    name, qp, s = case
    if name == "ragged":
        pytest.skip("oracle PPCG-IPM at this size takes minutes on the host")
    ref = oracle_ipm(qp, space="x", ipm_tol=1e-10)
    got = s.ipm_solve(ipm_tol=1e-10, space="x")
    assert got["converged"] and ref.converged
    assert abs(got["objective"] - ref.objective) <= 1e-8 * max(1.0, abs(ref.objective))
    x, lam, nu, sl = got["x"], got["lam"], got["nu"], got["s"]
    assert np.abs(qp.H @ x + qp.g - qp.A.T @ lam - qp.C.T @ nu).max() <= 1e-9 * (1 + np.abs(qp.g).max())
    assert np.abs(qp.C @ x - sl - qp.d).max() <= 1e-9 * (1 + np.abs(qp.d).max())
    n_cmp = min(len(ref.pcg_iters), len(got["pcg_iters"]), 3)
    for a, b in zip(ref.pcg_iters[:n_cmp], got["pcg_iters"][:n_cmp]):
        assert abs(a - b) <= 2
    # same optimum as the ν-space IPM
    nu_space = s.ipm_solve(ipm_tol=1e-10)
    assert abs(nu_space["objective"] - got["objective"]) <= 1e-8 * max(1.0, abs(got["objective"]))
