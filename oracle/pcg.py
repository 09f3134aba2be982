"""Oracle PCG (TEST INFRASTRUCTURE ONLY).

Textbook left-preconditioned conjugate gradient (Hestenes–Stiefel with the
P-inner-product recurrence), equivalent to CG on P^{-1/2} K P^{-1/2}
(P:L284–285).  Zero initial guess; stop when the recursively updated
residual satisfies ‖r‖₂ ≤ ε‖b‖₂.  The iteration count is the
number of operator applications.  b = 0 returns 0 iterations.
"""
from __future__ import annotations

import numpy as np


def pcg(Kop, b, Minv, tol, maxit):
    """Return (x, iters, relres, converged, history of ‖r‖)."""
    b = np.asarray(b, dtype=float)
    x = np.zeros_like(b)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return x, 0, 0.0, True, []
    r = b.copy()
    z = Minv(r)
    p = z.copy()
    rho = float(r @ z)
    hist = []
    for j in range(1, maxit + 1):
        q = Kop(p)
        alpha = rho / float(p @ q)
        x = x + alpha * p
        r = r - alpha * q
        rn = float(np.linalg.norm(r))
        hist.append(rn)
        if rn <= tol * bnorm:
            return x, j, rn / bnorm, True, hist
        z = Minv(r)
        rho_new = float(r @ z)
        beta = rho_new / rho
        p = z + beta * p
        rho = rho_new
    return x, maxit, float(np.linalg.norm(r)) / bnorm, False, hist
