import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
import qpgen
from test_gpu_sharded import run_ranks
from paper_2104_12916_b200.binding import from_qp
qp = qpgen.make('c0')
s1 = from_qp(qp); s1.ipm_factor_once('low'); s1.ipm_init(ipm_tol=1e-10, pcg_maxit=qp.m2)
def body(rank, comm):
    s = from_qp(qp, rank=rank, world=2, allreduce=comm.fn(rank)); s.ipm_factor_once('low')
    s.ipm_init(ipm_tol=1e-10, pcg_maxit=qp.m2)
    out = []
    for k in range(12):
        r = s.ipm_iterate(1, with_vectors=True)
        out.append((r['mu'], r['rg_inf'], r['re_inf'], r['ri_inf'], r['alpha'], r['pcg_iters'][-1:] , r['x'][:3]))
    return out
res = run_ranks(2, body)
for k in range(12):
    r = s1.ipm_iterate(1, with_vectors=True)
    print(k, 'single mu %.3e rg %.2e ri %.2e a %.4f it %s' % (r['mu'], r['rg_inf'], r['ri_inf'], r['alpha'], r['pcg_iters'][-1:]))
    for rk in range(2):
        m = res[rk][k]
        print('   rank', rk, 'mu %.3e rg %.2e ri %.2e a %.4f it %s' % (m[0], m[1], m[3], m[4], m[5]))
