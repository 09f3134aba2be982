"""Small end-to-end run of every kernel family (compute-sanitizer is unavailable on the GPU pool): c0 and a 700/130/900 QP through PL-KF, PH-KF, the x-space
twin, f_solve and kf_apply (every kernel family of the library at sizes that run in seconds)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import qpgen
from paper_2104_12916_b200.binding import from_qp
for qp in (qpgen.make("c0"), qpgen.scaled_random_qp(700, 130, 900, seed=3),
           qpgen.make_grid_qp(24, 40, 60, seed=4, name="grid24")):
    for prec in ("low", "high"):
        s = from_qp(qp)
        s.ipm_factor_once(prec)
        rng = np.random.default_rng(0)
        D = rng.uniform(0.5, 2, qp.m2)
        s.kf_apply(D, rng.standard_normal(qp.m2))
        s.f_solve(rng.standard_normal(qp.n + qp.m1))
        s.pcg_solve(D, rng.standard_normal(qp.m2), tol=1e-8, maxit=50)
        r = s.ipm_solve(ipm_tol=1e-6, max_ipm=6)
        if prec == "low":
            s.pcg_solve_x(D, rng.standard_normal(qp.n), rng.standard_normal(qp.m1), tol=1e-8, maxit=50)
            s.ipm_solve(ipm_tol=1e-6, max_ipm=4, space="x")
        s.close()
print("sanitize run ok")
