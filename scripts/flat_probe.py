import sys, time
sys.path.insert(0, '.')
import numpy as np
import qpgen
from paper_2104_12916_b200.binding import from_qp
for name in sys.argv[1:]:
    qp = qpgen.make(name)
    s = from_qp(qp)
    t = time.perf_counter(); s.ipm_factor_once('low'); t = time.perf_counter() - t
    st = s.stats()
    print(name, 'factor_once %.2f s' % t, 'flat', st['flat_enabled'], 'disc %.2e' % st['flat_discrepancy'],
          'nnzM %.3g' % st['flat_nnz_M'], 'sym', st['sym_enabled'], 'fsolve bytes %.4g' % st['fsolve_bytes_F'], flush=True)
