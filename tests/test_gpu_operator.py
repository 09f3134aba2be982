"""qp_operator_apply: the x-space operator G p = H p + Cᵀ(D⁻¹∘(C p)) (the north_star's fused
"H·p + Cᵀ(D·(C·p))" chain) without any factorization, against the oracle's G_apply (oracle/xspace.py),
on small cases (several quads and a ragged tail, long Zipf rows) and at the c3s / c4s stand-in sizes
(the oracle is two SciPy SpMVs there), plus the sharded mode through the two-process worker's pattern:
every rank applies its rows of C, rank 0 adds H p, the caller-visible q is the all-reduced sum."""
import numpy as np
import pytest

import qpgen
from oracle.xspace import G_apply

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c0", "ragged", "c3s", "c4s"])
def test_operator_apply_matches_oracle(name):
    from paper_2104_12916_b200.binding import from_qp
    qp = qpgen.scaled_random_qp(700, 130, 900, seed=3) if name == "ragged" else qpgen.make(name)
    s = from_qp(qp)                      # no ipm_factor_once: the operator needs no factor
    rng = np.random.default_rng(21)
    D = np.exp(rng.uniform(-4, 4, qp.m2))
    p = rng.standard_normal(qp.n)
    q = s.operator_apply(D, p)
    ref = G_apply(qp, 1.0 / D, p)
    assert np.linalg.norm(q - ref) <= 1e-13 * np.linalg.norm(ref)
    q2 = s.operator_apply(D, p)          # fixed-order sums: bit-identical reruns
    assert np.array_equal(q, q2)
