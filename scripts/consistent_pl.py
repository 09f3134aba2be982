"""PL-KF along a converging trajectory: the paper's benchmark protocol on the GPU.

P:L591–592: with ε = 1e-3 "the loss of accuracy in attained IPM objective value with respect to a
direct solver is below 6·10⁻⁷ ... In our comparative benchmarks, to ensure the IPM iteration count and
linear systems are consistent among the iterative methods used, we replace the computed inexact
solution with the result from direct solve at the end of each IPM step."  On the GPU the "direct" Δν is
PH-KF's PCG run to 1e-12 (P_H = D + C diag(H)⁻¹Cᵀ, Cholesky every IPM step; its spectrum stays
clustered, Theorem 2), and on every system (D_k, r_ν, ε_k = min(1e-3, μ_k)) of that trajectory a second
context runs PL-KF's PCG only to COUNT its iterations.  The IPM converges (it is PH-KF's), so the PL
counts are the paper's n_kr for PL-KF.  Oracle twin: oracle.ipm.ipm_solve(direct=True, consistent="low").

python scripts/consistent_pl.py CFG [pl_maxit]   → one JSON line
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def consistent_pl(qp, pl_maxit=2000, ipm_tol=1e-8, device=0, stream=None, max_ipm=100, keep_systems=False):
    from paper_2104_12916_b200.binding import from_qp
    ph = from_qp(qp, device=device, stream=stream)
    pl = from_qp(qp, device=device, stream=stream)
    t0 = time.perf_counter()
    ph.ipm_factor_once("high")
    pl.ipm_factor_once("low")
    t_setup = time.perf_counter() - t0
    ph.ipm_init(ipm_tol=ipm_tol, pcg_tol=1e-12, pcg_forcing=False, max_ipm=max_ipm, pcg_maxit=4000)
    counts, ph_counts, mus, systems = [], [], [], []
    t_pl = 0.0
    t1 = time.perf_counter()
    r = None
    for k in range(max_ipm):
        r = ph.ipm_iterate(1)
        if r["converged"]:
            break
        D, rnu, _ = ph.ipm_last_system()
        eps = min(1e-3, float(r["mu"]))
        ta = time.perf_counter()
        _, it, _, _ = pl.pcg_solve(D, rnu, tol=eps, maxit=pl_maxit)
        t_pl += time.perf_counter() - ta
        counts.append(it)
        if keep_systems:
            systems.append((D, rnu, eps))
        ph_counts.append(int(r["pcg_iters"][-1]))
        mus.append(float(r["mu"]))
    t_total = time.perf_counter() - t1
    out = {"converged": bool(r["converged"]), "n_ipm": int(r["n_ipm"]), "objective": float(r["objective"]),
           "pl_counts": counts, "pl_total": int(sum(counts)), "pl_maxit": pl_maxit,
           "pl_hit_maxit": int(sum(c >= pl_maxit for c in counts)),
           "ph_tight_counts": ph_counts, "mu": mus, "t_setup_s": t_setup, "t_total_s": t_total,
           "t_pl_counting_s": t_pl}
    if keep_systems:
        out["systems"] = systems
    ph.close()
    pl.close()
    return out


if __name__ == "__main__":
    import qpgen
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
    mx = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    res = consistent_pl(qpgen.make(cfg), pl_maxit=mx)
    res["config"] = cfg
    print(json.dumps(res))
