"""Device launch timeline of PCG iterations (qp_debug_timeline): per kernel its average duration and the
average idle gap before it (from the previous launch's end), over fixed-count PCG solves run through the
production path (CUDA graphs included).  python scripts/timeline.py [config] [iters]"""
import json
import sys
from collections import defaultdict
import numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
NAMES = ["flat_rhs", "flat_fwd", "root_gemv", "flat_bwd", "pcg_step", "trsv_fwd", "trsv_bwd", "spmv", "lvl_fwd", "lvl_bwd"]
name = sys.argv[1] if len(sys.argv) > 1 else 'c1'
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
qp = qpgen.make(name)
s = from_qp(qp)
import os
s.ipm_factor_once(os.environ.get('TL_PREC', 'low'))
_st = s.stats()
print('flat', _st['flat_enabled'], 'discrepancy %.2e' % _st['flat_discrepancy'])
rng = np.random.default_rng(0)
D = rng.uniform(0.5, 2.0, qp.m2)
b = rng.standard_normal(qp.m2)
s.pcg_solve(D, b, tol=0.0, maxit=50)        # graphs captured, warm
import os
if os.environ.get('TL_PROFILE'):
    s.profile(True)                          # CUDA events around every section, no graphs
s.debug_timeline(True)
if os.environ.get('TL_KF'):                  # K_F products only (works with timing-only switches)
    for _ in range(iters):
        s.kf_apply(D, b)
else:
    s.pcg_solve(D, b, tol=0.0, maxit=iters)
ev = s.debug_timeline(False)
ev = ev[len(ev) // 4:]                       # steady state (skip the first eager iterations)
dur, gap, cnt = defaultdict(float), defaultdict(float), defaultdict(int)
for (k0, s0, e0), (k1, s1, e1) in zip(ev, ev[1:]):
    gap[k1] += (s1 - e0) / 1e3
    dur[k1] += (e1 - s1) / 1e3
    cnt[k1] += 1
span = (ev[-1][2] - ev[0][1]) / 1e3
per_it = span / max(1, cnt[2] or cnt[5])
out = {NAMES[k]: {"n": cnt[k], "dur_us": round(dur[k] / cnt[k], 2), "gap_before_us": round(gap[k] / cnt[k], 2)}
       for k in sorted(cnt)}
print(json.dumps({"config": name, "us_per_iteration": round(per_it, 2), "kernels": out}))
if os.environ.get('TL_SERIES'):
    print('gemv series', [round((e - s0) / 1e3, 1) for k, s0, e in ev if k == 2])
if _st.get('pi_enabled'):
    # level products: per-level durations (launch order within a sweep), averaged over the recorded sweeps
    for kk, nm in ((5, 'level fwd'), (6, 'level bwd'), (8, 'leaf fwd'), (9, 'leaf bwd')):
        e = [(s0, e0) for k, s0, e0 in ev if k == kk]
        nl = max(1, round(len(e) / max(1, cnt[2])))
        e = e[:len(e) // nl * nl]
        d = np.array([(b - a) / 1e3 for a, b in e]).reshape(-1, nl)
        print(nm, 'levels per sweep', nl, 'us per level', d.mean(0).round(1).tolist(), 'sum', round(float(d.mean(0).sum()), 1))
