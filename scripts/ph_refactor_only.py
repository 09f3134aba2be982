"""c1 P_H: factor once, then one more P_H refactor (new D) — a short command for ncu launch lists."""
import sys
sys.path.insert(0, '.')
import numpy as np
import qpgen
from paper_2104_12916_b200.binding import from_qp
qp = qpgen.make(sys.argv[1] if len(sys.argv) > 1 else 'c1')
s = from_qp(qp)
s.ipm_factor_once('high')
rng = np.random.default_rng(1)
D = rng.uniform(0.5, 2.0, qp.m2)
s.pcg_solve(D, rng.standard_normal(qp.m2), tol=1e-3, maxit=3)   # forces a P_H refactor at D
print('ok')
