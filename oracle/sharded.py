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


# ---------------------------------------------------------------- halo mode of the x-space operator
def halo_plan(H, C, row_bounds, world):
    """Owned x-ranges and windows of the halo mode (include/qp_b200.h qp_operator_halo_plan; BJ configs[4]:
    "rows are partitioned … with a halo exchange"; north_star: "boundary entries of p are exchanged").

    Written out from the definition:
    * cmin_g, cmax_g: the first / last column any of rank g's rows of C (rows row_bounds[g]..row_bounds[g+1]) touches;
    * owned boundaries b_0 = 0, b_W = n, b_g = ⌊(cmax_{g−1} + 1 + cmin_g)/2⌋ made monotone: rank g owns x[b_g : b_{g+1}];
    * q window of g = hull(owned range, [cmin_g, cmax_g]); p window = hull(q window, columns of H's owned rows);
    * enabled iff every owned range is non-empty and every window lies in [b_{g−1}, b_{g+2}] (only the two
      neighbours' parts of x are reached).
    Returns dict(enabled, b, p_lo, p_hi, q_lo, q_hi) with numpy int64 arrays."""
    H = H.tocsr()
    C = C.tocsr()
    n = H.shape[0]
    W = world
    cmin, cmax = np.zeros(W, dtype=np.int64), np.zeros(W, dtype=np.int64)
    ok = W >= 2 and n >= 4 * W
    for g in range(W):
        idx = C.indices[C.indptr[row_bounds[g]]:C.indptr[row_bounds[g + 1]]]
        if len(idx) == 0:
            return dict(enabled=False)
        cmin[g], cmax[g] = idx.min(), idx.max()
    b = np.zeros(W + 1, dtype=np.int64)
    b[W] = n
    for g in range(1, W):
        mid = int(np.floor((float(cmax[g - 1]) + 1.0 + float(cmin[g])) / 2.0))
        b[g] = max(b[g - 1], min(n, max(0, mid)))
    ok = ok and bool(np.all(np.diff(b) > 0))
    p_lo, p_hi, q_lo, q_hi = (np.zeros(W, dtype=np.int64) for _ in range(4))
    for g in range(W):
        q_lo[g], q_hi[g] = min(b[g], cmin[g]), max(b[g + 1], cmax[g] + 1)
        p_lo[g], p_hi[g] = q_lo[g], q_hi[g]
        if ok:
            cols = H.indices[H.indptr[b[g]]:H.indptr[b[g + 1]]]
            if len(cols):
                p_lo[g], p_hi[g] = min(p_lo[g], cols.min()), max(p_hi[g], cols.max() + 1)
    for g in range(W):
        left, right = b[max(0, g - 1)], b[min(W, g + 2)]
        ok = ok and p_lo[g] >= left and p_hi[g] <= right and q_lo[g] >= left and q_hi[g] <= right
    return dict(enabled=bool(ok), b=b, p_lo=p_lo, p_hi=p_hi, q_lo=q_lo, q_hi=q_hi)


def halo_operator(rank, plan, H, C_g, D_g, p, exchange):
    """One product q = H p + Cᵀ(D⁻¹∘(C p)) in halo mode on `rank`.  p: length-n array whose owned
    entries are valid; exchange(to_prev, to_next, n_from_prev, n_from_next) -> (from_prev, from_next) moves
    arrays between neighbouring ranks.  Returns (q, p): q valid on the owned range, p with the window filled."""
    b, W = plan["b"], len(plan["b"]) - 1
    g = rank
    lo, hi = int(b[g]), int(b[g + 1])
    p = np.array(p, dtype=float, copy=True)
    # 1. boundary entries of p
    tp = p[lo:int(plan["p_hi"][g - 1])] if g > 0 else p[:0]
    tn = p[int(plan["p_lo"][g + 1]):hi] if g + 1 < W else p[:0]
    fp, fn = exchange(tp, tn, lo - int(plan["p_lo"][g]), int(plan["p_hi"][g]) - hi)
    p[int(plan["p_lo"][g]):lo] = fp
    p[hi:int(plan["p_hi"][g])] = fn
    # 2. local products: C_g reaches only the q window, H's owned rows only the p window
    pw = np.zeros_like(p)
    pw[int(plan["p_lo"][g]):int(plan["p_hi"][g])] = p[int(plan["p_lo"][g]):int(plan["p_hi"][g])]
    t = (C_g @ pw) / D_g
    q = np.asarray(C_g.T @ t, dtype=float)
    q[lo:hi] += (H.tocsr()[lo:hi] @ pw)
    # 3. q outside the owned range goes to its owner
    qtp = q[int(plan["q_lo"][g]):lo]
    qtn = q[hi:int(plan["q_hi"][g])]
    nfp = int(plan["q_hi"][g - 1]) - lo if g > 0 else 0
    nfn = hi - int(plan["q_lo"][g + 1]) if g + 1 < W else 0
    fp, fn = exchange(qtp, qtn, max(0, nfp), max(0, nfn))
    q[lo:lo + len(fp)] += fp
    q[hi - len(fn):hi] += fn
    return q, p
