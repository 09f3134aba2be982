import sys, time, json
import numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
name, prec = sys.argv[1], sys.argv[2]
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
qp = qpgen.make(name)
s = from_qp(qp)
t = time.time(); s.ipm_factor_once(prec); tf = time.time() - t
st = s.stats()
t = time.time(); r = s.ipm_solve(ipm_tol=1e-8, max_ipm=100, pcg_maxit=maxit); dt = time.time() - t
x, lam, nu, sl = r["x"], r["lam"], r["nu"], r["s"]
grad = qp.H @ x + qp.g - qp.A.T @ lam - qp.C.T @ nu
print(json.dumps(dict(name=name, prec=prec, factor_s=tf, solve_s=dt, n_ipm=r['n_ipm'], conv=r['converged'], obj=r['objective'],
      mu=r['mu'], rg=r['rg_inf'], re=r['re_inf'], ri=r['ri_inf'], pcg_total=r['pcg_total'], pcg=r['pcg_iters'],
      nnz_LPH=st['nnz_LPH'], t_factor_ph=st['t_factor_ph_s'])), flush=True)
