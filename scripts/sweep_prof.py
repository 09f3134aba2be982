import sys, numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
qp = qpgen.make(sys.argv[1] if len(sys.argv) > 1 else 'c1')
s = from_qp(qp); s.ipm_factor_once('low')
rng = np.random.default_rng(0); D = rng.uniform(0.5, 2, qp.m2); p = rng.standard_normal(qp.m2)
s.kf_apply(D, p)
s.debug_sweep_profile(True); s.kf_apply(D, p); pr = s.debug_sweep_profile(False)
names = ['DIAG', 'TILE', 'PREP', 'XCHUNK', 'SNF', 'SCHUNK', 'ROOTB', 'SNW']
for sw in range(2):
    t0 = min(pr[sw, t, 3] for t in range(8) if pr[sw, t, 0] > 0)
    for t in range(8):
        c, w, b, f, l = pr[sw, t]
        if c == 0: continue
        print(['fwd', 'bwd'][sw], names[t], 'count', c, 'avg wait us %.2f' % (w / c / 1e3), 'avg busy us %.2f' % (b / c / 1e3),
              'first %.1f us' % ((f - t0) / 1e3), 'last %.1f us' % ((l - t0) / 1e3))
