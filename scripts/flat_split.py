"""Per-section CUDA-event times of c1 PCG iterations (profile mode, no graphs): forward (rhs + forward
product), root GEMV, backward product, K_F q / PCG vectors.  Used with QPB_* switches to see what each
part of the flattened F-solve costs."""
import json
import sys
import numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
name = sys.argv[1] if len(sys.argv) > 1 else 'c1'
qp = qpgen.make(name)
s = from_qp(qp)
s.ipm_factor_once('low')
rng = np.random.default_rng(0)
D = rng.uniform(0.5, 2.0, qp.m2)
b = rng.standard_normal(qp.m2)
import os, time
s.pcg_solve(D, b, tol=0.0, maxit=20)
for _ in range(int(os.environ.get('WARM_REPS', '0'))):   # heat the GPU first (power / clocks)
    s.pcg_solve(D, b, tol=0.0, maxit=1000)
t = time.perf_counter(); x, it, rr, rc = s.pcg_solve(D, b, tol=0.0, maxit=300); t = time.perf_counter() - t
print('graph pcg %.4f ms/it' % (1e3 * t / it))
s.profile(True)
try:
    s.pcg_solve(D, b, tol=0.0, maxit=100)
except Exception as e:   # timing-only switches can break the operator
    print('pcg:', e)
print(json.dumps({k: (round(1e3 * m / c, 2), c) for k, (m, c) in s.profile_read().items() if c}))
