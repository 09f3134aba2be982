"""A/B: sweep timing for c1 with the library's order vs a given order (postorder on/off)."""
import sys, time, numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp, Analysis
qp = qpgen.make('c1')
mode = sys.argv[1] if len(sys.argv) > 1 else 'lib'
perm = None
if mode == 'nopost':
    # min-degree order without postorder: take it from a dedicated env switch in the library
    import os
    os.environ['QPB_NO_POSTORDER'] = '1'
s = from_qp(qp, x_perm=perm)
s.ipm_factor_once('low')
st = s.stats()
print(mode, 'ns', st['n_supernodes_F'], 'levels', st['n_levels_F'])
rng = np.random.default_rng(0); D = rng.uniform(0.5, 2, qp.m2); b = rng.standard_normal(qp.m2)
s.profile(True)
s.pcg_solve(D, b, tol=0.0, maxit=5)
s.profile(False); s.profile(True)
t = time.time(); x, it, rr, rc = s.pcg_solve(D, b, tol=0.0, maxit=60); dt = time.time() - t
pr = s.profile_read()
print(mode, 'wall ms/it %.3f' % (1e3 * dt / it), 'fwd ms %.3f' % (pr['f_fwd'][0] / pr['f_fwd'][1]), 'root ms %.3f' % (pr['f_root'][0] / max(1, pr['f_root'][1])), 'bwd ms %.3f' % (pr['f_bwd'][0] / pr['f_bwd'][1]))
s.profile(False)
for _ in range(2):
    t = time.time(); x, it, rr, rc = s.pcg_solve(D, b, tol=0.0, maxit=200); dt = time.time() - t
print(mode, 'noprof wall ms/it %.4f' % (1e3 * dt / it))
