"""Oracle for the sharded (multi-rank) PCG — TEST INFRASTRUCTURE ONLY.

SURVEY §8(e): the m2 inequality rows (ν-space: C, D, p, r, z, q, Δν) are split into
contiguous nnz-balanced slices, one per rank; the x-space F-solve is replicated.  One
K_F product then reads

    u   = Σ_g C_gᵀ p_g                    (all-reduce of n doubles)
    w   = [F⁻¹ [u; 0]]_x                   (replicated)
    q_g = D_g p_g − C_g w                  (local)

and every PCG inner product (pᵀq, rᵀz, ‖r‖², ‖b‖²) is a sum of per-rank partial sums
(all-reduce).  Algebraically this is the unsharded PCG of oracle.pcg (P:L284–285,
P:L590–591); only the summation order of the reductions differs.

`partition_rows` is the plain definition of the split the library uses: the row
boundary r is the first row i whose prefix weight Σ_{k<i} (nnz_k + 1) reaches
r/world of the total.
"""
from __future__ import annotations

import numpy as np


def partition_rows(indptr, m2, world):
    """bounds[0..world]: bounds[r] = min{i : Σ_{k<i}(nnz_k + 1) ≥ total·r/world} (monotone)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    total = float(indptr[m2] - indptr[0]) + float(m2)
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        i = 0
        while i < m2 and float(indptr[i] - indptr[0]) + float(i) < target:
            i += 1
        bounds.append(max(i, bounds[-1]))
    bounds.append(m2)
    return np.array(bounds, dtype=np.int64)


def sharded_pcg(C_g, fs, D_g, b_g, Minv_g, tol, maxit, allreduce):
    """PCG on this rank's slice.  C_g: the rank's rows of C (scipy CSR); fs: the replicated
    F-solver (oracle.fsolve, fs.solve(r_x, r_λ) -> (y_x, y_λ)); allreduce(np.ndarray) -> the
    element-wise sum over ranks.  Returns (x_g, iters, relres, converged) with the textbook
    recurrence of oracle.pcg."""

    def K(p):
        u = allreduce(np.asarray(C_g.T @ p, dtype=float))   # Σ_g C_gᵀ p_g
        w, _ = fs.solve(u, None)                             # replicated F-solve
        return D_g * p - C_g @ w

    dot = lambda a, c: float(allreduce(np.array([float(a @ c)]))[0])
    x = np.zeros_like(b_g)
    bnorm = np.sqrt(dot(b_g, b_g))
    if bnorm == 0.0:
        return x, 0, 0.0, True
    r = b_g.copy()
    z = Minv_g(r)
    p = z.copy()
    rho = dot(r, z)
    for j in range(1, maxit + 1):
        q = K(p)
        alpha = rho / dot(p, q)
        x = x + alpha * p
        r = r - alpha * q
        rn = np.sqrt(dot(r, r))
        if rn <= tol * bnorm:
            return x, j, rn / bnorm, True
        z = Minv_g(r)
        rho_new = dot(r, z)
        p = z + (rho_new / rho) * p
        rho = rho_new
    return x, maxit, rn / bnorm, False
