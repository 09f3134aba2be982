import sys; sys.path.insert(0,'.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
for name in ['c0']:
    qp=qpgen.make(name); s=from_qp(qp); s.ipm_factor_once('low'); st=s.stats()
    print(name, {k: st[k] for k in ('fsolve_bytes_F','kf_bytes_W','dense_w_enabled','dense_w_discrepancy','flat_enabled','sym_enabled','n')})
qp=qpgen.scaled_random_qp(700, 130, 900, seed=3); s=from_qp(qp); s.ipm_factor_once('low'); st=s.stats()
print('ragged', {k: st[k] for k in ('fsolve_bytes_F','kf_bytes_W','dense_w_enabled','dense_w_discrepancy','flat_enabled','sym_enabled','n')})
