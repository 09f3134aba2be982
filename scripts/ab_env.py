"""A/B timing of the c1 PCG iteration under environment variants, interleaved A B A B … in fresh
processes (same box): python scripts/ab_env.py 'QPB_ROOT_SPLIT=0' 'QPB_ROOT_SPLIT=1' [--reps 3] [--config c1]"""
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, time, json, numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
qp = qpgen.make(sys.argv[1])
s = from_qp(qp); s.ipm_factor_once(sys.argv[2])
rng = np.random.default_rng(0); D = rng.uniform(0.5, 2, qp.m2); b = rng.standard_normal(qp.m2)
s.pcg_solve(D, b, tol=0.0, maxit=20)
best = 1e9
for _ in range(3):
    t = time.perf_counter(); x, it, rr, rc = s.pcg_solve(D, b, tol=0.0, maxit=300); dt = time.perf_counter() - t
    best = min(best, 1e3 * dt / it)
print(json.dumps({"ms_per_it": best}))
'''

CHILD_REFACTOR = r'''
import sys, time, json, numpy as np
sys.path.insert(0, '.')
import qpgen
from paper_2104_12916_b200.binding import from_qp
qp = qpgen.make(sys.argv[1])
s = from_qp(qp); s.ipm_factor_once('high')
rng = np.random.default_rng(0); b = rng.standard_normal(qp.m2)
best = 1e9
for _ in range(4):   # each new D forces one P_H numeric refactor inside pcg_solve
    s.pcg_solve(rng.uniform(0.5, 2, qp.m2), b, tol=0.0, maxit=1)
    best = min(best, 1e3 * s.stats()['t_factor_ph_s'])
print(json.dumps({"ms_per_it": best}))
'''


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = 3
    cfg = "c1"
    pre = "low"
    for i, a in enumerate(sys.argv):
        if a == "--reps":
            reps = int(sys.argv[i + 1])
        if a == "--config":
            cfg = sys.argv[i + 1]
        if a == "--precond":
            pre = sys.argv[i + 1]
    variants = [a for a in args if a not in (str(reps), cfg, pre)]
    res = {v: [] for v in variants}
    for _ in range(reps):
        for v in variants:
            env = dict(os.environ)
            for kv in v.split(","):
                if "=" in kv:
                    k, val = kv.split("=", 1)
                    env[k] = val
            child = CHILD_REFACTOR if "--refactor" in sys.argv else CHILD
            out = subprocess.run([sys.executable, "-c", child, cfg, pre], env=env, capture_output=True, text=True)
            line = [l for l in out.stdout.splitlines() if l.startswith("{")]
            res[v].append(json.loads(line[-1])["ms_per_it"] if line else float("nan"))
            if not line:
                print(out.stderr[-2000:])
    for v, xs in res.items():
        xs_s = sorted(xs)
        print(f"{v:40s} median {xs_s[len(xs_s) // 2]:.4f} ms/it  all {['%.4f' % x for x in xs]}")


if __name__ == "__main__":
    main()
