"""Oracle inexact IPM loop (TEST INFRASTRUCTURE ONLY).

The paper's IPM loop text (``quadratic-program.tex``) is missing from
PAPER.md, so the loop controls are readings (DESIGN.md §Readings,
SURVEY.md §8(c) c3):

* start x = 0, λ = 0, ν = 1, s = |d| + 1;
* σ = 0.1 fixed; one reduced solve per IPM iteration (cost model P:L149);
* per iteration: residuals (sign reading R1), D = V⁻¹S
  (P:L480–483), r_ν, PCG on K_F with P_L / P_H / none at
  relative tolerance ε_k = min(ε, μ_k), ε = 1e-3 (forcing
  reading R4: with a fixed ε the row-3 error of eq. augmented keeps ‖r_i‖
  at ≈ε·‖r_ν‖ and the 1e-8 stop is never met — "high accuracy may only be
  needed in late iterations"), recovery, Δs
  (P:L473–478), a common fraction-to-boundary step with τ = 0.995 (R3);
* stop when ‖Hx+g−Aᵀλ−Cᵀν‖∞ ≤ tol(1+‖g‖∞), ‖r_e‖∞ ≤ tol(1+‖b‖∞),
  ‖r_i‖∞ ≤ tol(1+‖d‖∞) and μ ≤ tol;
* objective ½xᵀHx + gᵀx.

The F factorization is computed once (setup phase) and reused.
"""
from __future__ import annotations

import dataclasses
import time
from typing import List, Optional

import numpy as np

from . import kkt, xspace
from .fsolve import make_fsolver
from .pcg import pcg


@dataclasses.dataclass
class IpmResult:
    x: np.ndarray
    lam: np.ndarray
    nu: np.ndarray
    s: np.ndarray
    objective: float
    n_ipm: int
    converged: bool
    pcg_iters: List[int]
    trace: List[dict]
    t_setup: float = 0.0
    t_solve: float = 0.0


def ipm_solve(qp, precond: str = "low", pcg_tol: float = 1e-3, ipm_tol: float = 1e-8,
              max_ipm: int = 100, sigma: float = 0.1, tau: float = 0.995,
              pcg_maxit: Optional[int] = None, fs=None, x_perm=None, record: bool = False,
              exact_ph: bool = False, direct: bool = False, forcing: bool = True,
              space: str = "nu", ph_opts: Optional[dict] = None,
              rnu_perturb: Optional[int] = None, consistent: Optional[str] = None,
              rnu_perturb_mag: float = 1e-15) -> IpmResult:
    """Run the single-factorization inexact IPM.

    precond ∈ {"none" (U-KF), "low" (PL-KF), "high" (PH-KF)}.
    ``direct=True`` replaces PCG by a dense solve of K_F (trajectory reference).
    ``record=True`` stores (D_k, r_ν, Δν, PCG iterations) per IPM iteration.
    ``consistent`` ∈ {"none", "low", "high"} (with ``direct=True``): the paper's benchmark protocol (P:L592,
    "we replace the computed inexact solution with the result from direct solve at the end of each IPM
    step"): the step uses the direct Δν while PCG with the named preconditioner is run on every system
    (D_k, r_ν, ε_k) only to record its iteration count — so the counts of PL-KF are reported along a
    trajectory that converges.
    ``rnu_perturb``: seed of a relative 1e-15 perturbation of every r_ν (a rounding-level variant of the
    same trajectory, used to measure how far rounding alone moves the PCG counts; DESIGN reading R12).
    ``ph_opts``: keyword options of ``kkt.PrecondH`` (sparse SuperLU factor / in-place dense factor
    for the full-size configs).
    ``space="x"``: the x-space twin — projected CG on the augmented system K_C with the constraint
    preconditioner [H Aᵀ; A 0] = the F factor (oracle.xspace; `precond` is then ignored).
    """
    n, m1, m2 = qp.n, qp.m1, qp.m2
    t0 = time.perf_counter()
    if fs is None:
        fs = make_fsolver(qp.H, qp.A, x_perm if x_perm is not None else None)
    T = kkt.T_matrix(qp) if precond == "high" and not exact_ph else None
    t_setup = time.perf_counter() - t0
    if pcg_maxit is None:
        pcg_maxit = 2000

    x = np.zeros(n)
    lam = np.zeros(m1)
    nu = np.ones(m2)
    s = np.abs(qp.d) + 1.0
    gmax = float(np.max(np.abs(qp.g))) if n else 0.0
    bmax = float(np.max(np.abs(qp.b))) if m1 else 0.0
    dmax = float(np.max(np.abs(qp.d))) if m2 else 0.0

    trace, iters = [], []
    CWCt = None
    converged = False
    t1 = time.perf_counter()
    k = 0
    for k in range(max_ipm + 1):
        res = kkt.residuals(qp, x, lam, nu, s, sigma)
        rg_inf = float(np.max(np.abs(res["grad"]))) if n else 0.0
        re_inf = float(np.max(np.abs(res["r_e"]))) if m1 else 0.0
        ri_inf = float(np.max(np.abs(res["r_i"])))
        if (rg_inf <= ipm_tol * (1 + gmax) and re_inf <= ipm_tol * (1 + bmax)
                and ri_inf <= ipm_tol * (1 + dmax) and res["mu"] <= ipm_tol):
            converged = True
            break
        if k == max_ipm:
            break
        D = kkt.diag_D(s, nu)
        if space == "x":
            eps = min(pcg_tol, res["mu"]) if forcing else pcg_tol
            f, e, W = xspace.x_rhs(qp, res, D)
            dx, dlam, it, _, _, _ = xspace.ppcg(qp, fs, W, f, e, eps, pcg_maxit)
            dnu, ds = xspace.newton_from_x(qp, res, D, nu, dx)
            alpha, amax = kkt.step_length(s, ds, nu, dnu, tau)
            trace.append(dict(k=k, mu=res["mu"], rg=rg_inf, re=re_inf, ri=ri_inf, pcg=it, alpha=alpha, eps=eps))
            iters.append(it)
            x, lam, nu, s = x + alpha * dx, lam + alpha * dlam, nu + alpha * dnu, s + alpha * ds
            continue
        rnu = kkt.r_nu(qp, fs, res)
        if rnu_perturb is not None:
            prng = np.random.default_rng([rnu_perturb, k])
            rnu = rnu * (1.0 + rnu_perturb_mag * prng.standard_normal(m2))
        if direct:
            if getattr(fs, "W", None) is not None:
                # K_F = D − C W Cᵀ with the written-out W = (F⁻¹)₁₁; C W Cᵀ is D-independent
                if CWCt is None:
                    Cd = qp.C.toarray() if m2 * n <= 4e8 else None
                    CWCt = (qp.C @ (qp.C @ fs.W).T).T if Cd is None else Cd @ fs.W @ Cd.T
                KF = -CWCt.copy() if m2 <= 8192 else np.negative(CWCt)
                KF[np.diag_indices_from(KF)] += D
                if m2 > 8192:
                    L = kkt.chol_blocked(KF)
                    dnu = kkt.chol_blocked_solve(L, rnu)
                    del L, KF
                else:
                    dnu = np.linalg.solve(KF, rnu)
            else:
                KF = np.column_stack([kkt.KF_apply(qp, fs, D, e) for e in np.eye(m2)])
                dnu = np.linalg.solve(KF, rnu)
            it = 0
            if consistent is not None:   # count the iterative method on the same system, step direct
                Mc = (kkt.PrecondL(D) if consistent == "low" else
                      kkt.PrecondH(qp, D, T=kkt.T_matrix(qp) if T is None else T) if consistent == "high"
                      else kkt.PrecondNone())
                eps_c = min(pcg_tol, res["mu"]) if forcing else pcg_tol
                _, it, _, _, _ = pcg(lambda p: kkt.KF_apply(qp, fs, D, p), rnu, Mc, eps_c, pcg_maxit)
        else:
            if precond == "low":
                M = kkt.PrecondL(D)
            elif precond == "high":
                M = kkt.PrecondH(qp, D, T=T, exact=exact_ph, **(ph_opts or {}))
            else:
                M = kkt.PrecondNone()
            eps = min(pcg_tol, res["mu"]) if forcing else pcg_tol
            dnu, it, _, _, _ = pcg(lambda p: kkt.KF_apply(qp, fs, D, p), rnu, M, eps, pcg_maxit)
        dx, dlam = kkt.recover(qp, fs, res, dnu)
        ds = kkt.delta_s(res, D, nu, dnu)
        alpha, amax = kkt.step_length(s, ds, nu, dnu, tau)
        rec = dict(k=k, mu=res["mu"], rg=rg_inf, re=re_inf, ri=ri_inf, pcg=it, alpha=alpha,
                   eps=(min(pcg_tol, res["mu"]) if forcing else pcg_tol))
        if record:
            rec.update(D=D.copy(), rnu=rnu.copy(), dnu=dnu.copy())
        trace.append(rec)
        iters.append(it)
        x = x + alpha * dx
        lam = lam + alpha * dlam
        nu = nu + alpha * dnu
        s = s + alpha * ds
    obj = float(0.5 * x @ (qp.H @ x) + qp.g @ x)
    return IpmResult(x=x, lam=lam, nu=nu, s=s, objective=obj, n_ipm=k, converged=converged,
                     pcg_iters=iters, trace=trace, t_setup=t_setup,
                     t_solve=time.perf_counter() - t1)
