"""Device timeline of ONE K_F product (qp_kf_apply) on a config, launch by launch: kernel, start and end
relative to the first launch (µs) — shows the leaf-phase level kernels and the task-graph sweeps in order.
python scripts/fsolve_timeline.py [config] [reps]"""
import json
import sys
import numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
NAMES = ["flat_rhs", "flat_fwd", "root_gemv", "flat_bwd", "pcg_step", "trsv_fwd", "trsv_bwd", "spmv", "lvl_fwd",
         "lvl_bwd"]
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
qp = qpgen.make(name)
s = from_qp(qp)
s.ipm_factor_once('low')
st = s.stats()
rng = np.random.default_rng(0)
D = rng.uniform(0.5, 2.0, qp.m2)
p = rng.standard_normal(qp.m2)
for _ in range(3):
    s.kf_apply(D, p)
res = []
for r in range(reps):
    s.debug_timeline(True)
    s.kf_apply(D, p)
    ev = s.debug_timeline(False)
    t0 = ev[0][1]
    res.append([(NAMES[k], round((a - t0) / 1e3, 1), round((b - t0) / 1e3, 1)) for k, a, b in ev])
best = min(res, key=lambda e: e[-1][2])
print(json.dumps({"config": name, "lvl_levels_F": st["lvl_levels_F"], "lvl_supernodes_F": st["lvl_supernodes_F"],
                  "span_us": [e[-1][2] for e in res], "launches": best}))
