import sys, time, json
import numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
name = sys.argv[1] if len(sys.argv) > 1 else 'c1'
prec = sys.argv[2] if len(sys.argv) > 2 else 'low'
t = time.time(); qp = qpgen.make(name); print('gen', time.time() - t, flush=True)
t = time.time(); s = from_qp(qp); print('setup', time.time() - t, flush=True)
t = time.time(); s.ipm_factor_once(prec); print('factor_once', time.time() - t, flush=True)
st = s.stats(); print(json.dumps({k: st[k] for k in st}), flush=True)
rng = np.random.default_rng(0)
D = rng.uniform(0.5, 2.0, qp.m2); b = rng.standard_normal(qp.m2)
s.profile(True)
for maxit in (10, 50):
    t = time.time(); x, it, rr, rc = s.pcg_solve(D, b, tol=0.0, maxit=maxit); dt = time.time() - t
    print('pcg', maxit, it, rr, 'wall ms/it', 1e3 * dt / it, flush=True)
print(json.dumps(s.profile_read()), flush=True)
s.profile(False); s.profile(True)
t = time.time(); r = s.ipm_solve(with_vectors=False, max_ipm=int(sys.argv[3]) if len(sys.argv) > 3 else 100); dt = time.time() - t
print('ipm', dt, {k: r[k] for k in ('objective', 'n_ipm', 'status', 'pcg_total', 'mu', 'rg_inf', 're_inf', 'ri_inf', 'pcg_iters')}, flush=True)
print(json.dumps(s.profile_read()), flush=True)
