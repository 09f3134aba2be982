"""Factor c1 (or another config) and run one fixed-count PCG solve — a short command for ncu.
python scripts/pcg_once.py CFG ITERS [low|high] [ipm]   (ipm: also 2 IPM iterations, for k_ipm_* kernels)"""
import sys
import numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
name = sys.argv[1] if len(sys.argv) > 1 else 'c1'
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
qp = qpgen.make(name)
s = from_qp(qp)
prec = sys.argv[3] if len(sys.argv) > 3 else 'low'
s.ipm_factor_once(prec)
rng = np.random.default_rng(0)
D = rng.uniform(0.5, 2.0, qp.m2)
b = rng.standard_normal(qp.m2)
x, it, rr, rc = s.pcg_solve(D, b, tol=0.0, maxit=iters)
if len(sys.argv) > 4 and sys.argv[4] == 'ipm':
    s.ipm_init(ipm_tol=1e-8, max_ipm=100, pcg_maxit=200)
    s.ipm_iterate(2)
print('ok', it, rr)
