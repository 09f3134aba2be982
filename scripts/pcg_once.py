"""Factor c1 (or another config) and run one fixed-count PCG solve — a short command for ncu."""
import sys
import numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
name = sys.argv[1] if len(sys.argv) > 1 else 'c1'
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
qp = qpgen.make(name)
s = from_qp(qp)
s.ipm_factor_once('low')
rng = np.random.default_rng(0)
D = rng.uniform(0.5, 2.0, qp.m2)
b = rng.standard_normal(qp.m2)
x, it, rr, rc = s.pcg_solve(D, b, tol=0.0, maxit=iters)
print('ok', it, rr)
