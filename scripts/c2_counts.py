"""PCG counts of the first IPM iterations of c2 PL-KF, repeated (run-to-run spread of the atomics-based sweeps)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
cfg = sys.argv[1] if len(sys.argv) > 1 else 'c2'
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
nit = int(sys.argv[3]) if len(sys.argv) > 3 else 8
qp = qpgen.make(cfg)
s = from_qp(qp)
s.ipm_factor_once('low')
print('pi', s.stats()['pi_enabled'])
for rep in range(reps):
    s.ipm_init(ipm_tol=1e-8, max_ipm=100, pcg_maxit=2000)
    cnt = []
    for k in range(nit):
        r = s.ipm_iterate(1)
        cnt.append(int(r['pcg_iters'][-1]))
    print(rep, cnt, flush=True)
