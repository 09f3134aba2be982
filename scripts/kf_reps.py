"""Run R K_F products (qp_kf_apply) on a config after warm-up — a fixed workload for ncu launch lists.
python scripts/kf_reps.py [config] [reps]"""
import sys
import numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
qp = qpgen.make(name)
s = from_qp(qp)
s.ipm_factor_once('low')
rng = np.random.default_rng(0)
D = rng.uniform(0.5, 2.0, qp.m2)
p = rng.standard_normal(qp.m2)
for _ in range(3):
    s.kf_apply(D, p)
import time
t = time.time()
for _ in range(reps):
    s.kf_apply(D, p)
print('ms per kf_apply (wall, eager)', (time.time() - t) / reps * 1e3)
