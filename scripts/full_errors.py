"""Print the sampled relative errors of the GPU path against the full-size oracle goldens (see
tests/test_gpu_full.py): F-solve, K_F product, fixed-count PCG iterates.  python scripts/full_errors.py c3s"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import qpgen  # noqa: E402
from paper_2104_12916_b200.binding import from_qp  # noqa: E402


def err(got, z, pre, idx):
    e = got[idx] - z[pre + "s"]
    return np.sqrt(len(got) / len(idx)) * np.linalg.norm(e) / float(z[pre + "n2"])


for cfg in sys.argv[1:]:
    z = np.load(f"tests/golden/full/{cfg}.npz")
    qp = qpgen.make(cfg)
    pr = qpgen.probe_inputs(qp)
    s = from_qp(qp)
    s.ipm_factor_once("low")
    y, zz = s.f_solve(pr.f)
    out = {"F": err(np.concatenate([y, zz]), z, "F/", pr.idx_F), "KF": err(s.kf_apply(pr.D, pr.p), z, "KF/", pr.idx_m2)}
    for k in (1, 3, 7):
        x, *_ = s.pcg_solve(pr.D, pr.b, tol=0.0, maxit=k)
        out[f"PL{k}"] = err(x, z, f"PL/k{k}_", pr.idx_m2)
    x, it, rr, rc = s.pcg_solve(pr.D, pr.b, tol=1e-3, maxit=2000)
    out["PLeps_iters"] = (it, int(z["PL/eps_iters"]))
    print(cfg, {k: (f"{v:.2e}" if isinstance(v, float) else v) for k, v in out.items()}, flush=True)
    s.close()
