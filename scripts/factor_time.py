import sys, time, json
import numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
qp = qpgen.make(sys.argv[1] if len(sys.argv) > 1 else 'c1')
prec = sys.argv[2] if len(sys.argv) > 2 else 'high'
s = from_qp(qp)
t = time.time(); s.ipm_factor_once(prec); tf = time.time() - t
st = s.stats()
D = np.random.default_rng(0).uniform(0.5, 2.0, qp.m2); b = np.random.default_rng(1).standard_normal(qp.m2)
t = time.time(); x, it, rr, rc = s.pcg_solve(D, b, tol=1e-8, maxit=500); tp = time.time() - t   # includes a P_H refactor
print(json.dumps(dict(factor_once=tf, t_symbolic=st['t_symbolic_s'], t_factor=st['t_factor_s'], t_factor_ph=st['t_factor_ph_s'],
                      c_fact_F=st['c_fact_F'], c_fact_PH=st['c_fact_PH'], pcg_s=tp, pcg_it=it, rr=rr)))
