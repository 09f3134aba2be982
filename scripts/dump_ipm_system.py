"""Run the GPU PL-KF IPM for K iterations and dump the last reduced system (D_k, r_ν, ε_k) and the PCG
count the GPU needed on it (debug: compare with the oracle's PCG on the same system).
python scripts/dump_ipm_system.py CFG K OUT.npz"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import qpgen  # noqa: E402
from paper_2104_12916_b200.binding import from_qp  # noqa: E402

cfg, K, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
qp = qpgen.make(cfg)
s = from_qp(qp)
s.ipm_factor_once("low")
s.ipm_init(ipm_tol=1e-8, max_ipm=100, pcg_maxit=2000)
counts = []
for k in range(K):
    r = s.ipm_iterate(1)
    counts.append(int(r["pcg_iters"][-1]))
D, rnu, eps = s.ipm_last_system()
x, it, rr, rc = s.pcg_solve(D, rnu, tol=eps, maxit=2000)
np.savez(out, D=D, rnu=rnu, eps=eps, counts=np.array(counts), resolve_iters=it)
print(cfg, "counts", counts, "re-solve", it, "eps", eps)
