"""Per-task timeline of the F-solve sweeps (debug): which level / task type is on the critical path."""
import sys
import numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp

import os
qp = qpgen.make(sys.argv[1] if len(sys.argv) > 1 else 'c1')
PH = len(sys.argv) > 2 and sys.argv[2] == 'ph'      # trace the P_H factor's sweeps (QPB_TRACE_PH=1)
if PH:
    os.environ['QPB_TRACE_PH'] = '1'
s = from_qp(qp)
s.ipm_factor_once('high' if PH else 'low')
ss = s.structure('sn_start', ph=PH); lev = s.structure('sn_level', ph=PH)
w = np.diff(ss)
nblk = (w + 63) // 64
blk_sn = np.repeat(np.arange(len(w)), nblk)
rng = np.random.default_rng(0)
D = rng.uniform(0.5, 2, qp.m2); p = rng.standard_normal(qp.m2)
def run():
    if PH:   # one P_H apply per PCG iteration; the trace keeps the last sweep pair
        s.pcg_solve(D, p, tol=1e-30, maxit=2)
    else:
        s.kf_apply(D, p)
for rep in range(3):
    run()
s.debug_sweep_profile(True); run(); s.debug_sweep_profile(False)
names = ['DIAG', 'TILE', 'PREP', 'XCHUNK', 'SNF', 'SCHUNK', 'ROOTB', 'SNW']
for sw in range(2):
    tr = s.debug_sweep_trace(sw)
    task = tr[:, 0] & 0xffffffff
    sm = tr[:, 0] >> 32
    typ, idx = task >> 28, task & ((1 << 28) - 1)
    t0 = tr[:, 1].min()
    a, b, c = (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3, (tr[:, 5] - t0) / 1e3
    ma, mb = (tr[:, 3] - t0) / 1e3, (tr[:, 4] - t0) / 1e3
    L = np.where(np.isin(typ, [0, 2, 4]), lev[blk_sn[np.minimum(idx, len(blk_sn) - 1)]], -1)
    print(['fwd', 'bwd'][sw], 'tasks', len(tr), 'span %.1f us' % c.max(), 'SMs used', len(np.unique(sm)))
    for ty in np.unique(typ):
        for lv in np.unique(L[typ == ty]):
            k = (typ == ty) & (L == lv)
            print('  %-6s lev %2d n %4d  start[min %.1f max %.1f]  dep-met[med %.1f max %.1f]  end[med %.1f max %.1f]  busy %.2f'
                  % (names[ty], lv, k.sum(), a[k].min(), a[k].max(), np.median(b[k]), b[k].max(),
                     np.median(c[k]), c[k].max(), np.mean(c[k] - b[k])))
    order = np.argsort(b)
    print('  tickets: first 5 types', [names[t] for t in typ[:5]], 'last 5', [names[t] for t in typ[-5:]])
    st = a
    print('  start time by ticket decile:', ['%.1f' % np.median(st[i:i + len(st) // 10]) for i in range(0, len(st), len(st) // 10)])
    print('  setup (dep-met - start) by type:', {names[t]: '%.2f' % np.median((b - a)[typ == t]) for t in np.unique(typ)})
    print('  tasks per SM: min %d max %d' % (np.bincount(sm).min(), np.bincount(sm).max()))
    for ty in np.unique(typ):
        k = typ == ty
        print('  %-6s total busy %.1f us (%.1f%% of span x CTAs)  median busy %.2f us  median wait %.2f us' % (
            names[ty], (c[k] - b[k]).sum(), 100 * (c[k] - b[k]).sum() / (c.max() * len(np.unique(sm)) * 4),
            np.median(c[k] - b[k]), np.median(b[k] - a[k])))
    k = typ == 4
    if k.any() and (tr[k, 3] > 0).any():
        print('  SNF phases (us, median): dep->solved %.2f  solved->atomics done %.2f  atomics->end %.2f' % (
            np.median(ma[k] - b[k]), np.median(mb[k] - ma[k]), np.median(c[k] - mb[k])))
    k7 = typ == 7
    if k7.any() and (tr[k7, 3] > 0).any():
        print('  SNW warp-0 phases (us, median): start->solved %.2f  solved->fan-out issued %.2f  ->end (fences) %.2f' % (
            np.median(ma[k7] - a[k7]), np.median(mb[k7] - ma[k7]), np.median(c[k7] - mb[k7])))
    print('  SNF start quantiles', np.percentile(a[k], [10, 50, 90]).round(1), 'dep-start quantiles', np.percentile((b - a)[k], [10, 50, 90]).round(1))
