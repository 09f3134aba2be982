"""Bit-reproducibility of the deterministic paths (SURVEY §5 "deterministic reductions").

Every floating-point reduction on these paths has a fixed order: the PCG dot products (per-block
partials summed in block order by every block), the symmetric GEMVs of W / F⁻¹ / S⁻¹ / P_H⁻¹ (per-chunk
slots summed per output block in a fixed list order by the last arriver), the flattened forest's M and
L11⁻¹ products (per-unit slots reduced per row / column in unit order).  So two runs of the same
computation give the same bits:
* c0 (N = 250: explicit F⁻¹): pcg_solve, K_F products, a full PL-KF IPM solve, and PH-KF with the
  opt-in explicit P_H⁻¹ (QPB_DENSE_PHINV);
* c1 (explicit W = (F⁻¹)₁₁ for every PCG K_F product, flattened forest for the full F-solves): pcg_solve,
  F-solves and K_F products, 3 IPM iterations.
(The task-graph sweeps of the large sparse factors still accumulate their fan-out with fp64 atomics —
c2/c3s/c4s — and are checked against the oracle with tolerances instead; DESIGN R12.)
"""
import numpy as np
import pytest

import qpgen

pytestmark = pytest.mark.gpu


def _solver(qp, prec="low"):
    from paper_2104_12916_b200.binding import from_qp
    s = from_qp(qp)
    s.ipm_factor_once(prec)
    return s


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("cfg", ["c0", "c1"])
def test_pcg_and_products_bit_identical(cfg):
    qp = qpgen.make(cfg)
    pr = qpgen.probe_inputs(qp)
    s = _solver(qp)
    st = s.stats()
    if cfg == "c0":
        assert st["dense_finv_enabled"] == 1.0
    else:
        assert st["dense_w_enabled"] == 1.0 and st["flat_enabled"] == 1.0
    runs = [s.pcg_solve(pr.D, pr.b, tol=1e-6, maxit=500) for _ in range(3)]
    assert all(r[1] == runs[0][1] for r in runs) and runs[0][1] > 5
    assert all(_same(r[0], runs[0][0]) for r in runs)
    fa = [np.concatenate(s.f_solve(pr.f)) for _ in range(3)]
    assert all(_same(f, fa[0]) for f in fa)
    qa = [s.kf_apply(pr.D, pr.p) for _ in range(3)]
    assert all(_same(q, qa[0]) for q in qa)


def test_ipm_iterations_bit_identical_c1():
    qp = qpgen.make("c1")
    s = _solver(qp)
    out = []
    for _ in range(2):
        s.ipm_init(ipm_tol=1e-8, max_ipm=100, pcg_maxit=2000)
        r = s.ipm_iterate(3, with_vectors=True)
        out.append(r)
    assert out[0]["pcg_iters"] == out[1]["pcg_iters"]
    for k in ("x", "lam", "nu", "s"):
        assert _same(out[0][k], out[1][k]), k


@pytest.mark.parametrize("prec", ["low", "high"])
def test_ipm_solve_bit_identical_c0(prec, monkeypatch):
    monkeypatch.setenv("QPB_DENSE_PHINV", "4096")
    qp = qpgen.make("c0")
    res = []
    for _ in range(2):
        s = _solver(qp, prec)
        res.append(s.ipm_solve(ipm_tol=1e-10))
        s.close()
    a, b = res
    assert a["converged"] and b["converged"] and a["pcg_iters"] == b["pcg_iters"]
    assert a["objective"] == b["objective"] and _same(a["x"], b["x"]) and _same(a["nu"], b["nu"])
