"""Oracle F-solves (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

F = [−H Aᵀ; A 0]  (eq. f-def) is nonsingular for SPD H
and full-row-rank A; its inertia is (n negative, m1 positive)
(Haynsworth).

Three ways to apply F⁻¹:

* ``DenseF``  — the explicit block inverse of P:L757–773 (eq. f-inv)
      F⁻¹ = [ −H⁻¹ + H⁻¹AᵀF_H⁻¹AH⁻¹ ,  H⁻¹AᵀF_H⁻¹ ]
            [        F_H⁻¹AH⁻¹        ,     F_H⁻¹   ],   F_H = AH⁻¹Aᵀ,
  applied with LAPACK Cholesky factors of H and of F_H (no LDLᵀ at all).
* ``BlockF``  — the same block formula with SuperLU's LU of the SPD H and a
  dense Cholesky of the m1 × m1 F_H: the full-size sparse configs;
* ``SparseF`` — SuperLU LU of F permuted to the x-block order ``x_perm``
  with the λ block last, NATURAL column order and no pivoting
  (diag_pivot_thresh = 0), for the sparse configs.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def assemble_F(H, A) -> sp.csr_matrix:
    """F = [−H Aᵀ; A 0]."""
    m1 = A.shape[0]
    if m1 == 0:
        return sp.csr_matrix(-H)
    return sp.bmat([[-H, A.T], [A, sp.csr_matrix((m1, m1))]], format="csr")


class DenseF:
    """F⁻¹ through the block-inverse formula f-inv."""

    def __init__(self, H, A, explicit_w=False):
        Hd = H.toarray() if sp.issparse(H) else np.asarray(H, dtype=float)
        Ad = A.toarray() if sp.issparse(A) else np.asarray(A, dtype=float)
        self.n, self.m1 = Hd.shape[0], Ad.shape[0]
        self.A = Ad
        self.cH = sla.cho_factor(Hd, lower=True)           # H = L Lᵀ (H SPD)
        HiAt = None
        if self.m1:
            HiAt = sla.cho_solve(self.cH, Ad.T)              # H⁻¹Aᵀ
            FH = Ad @ HiAt                                   # F_H = A H⁻¹ Aᵀ (SPD)
            self.cFH = sla.cho_factor(FH, lower=True)
        else:
            self.cFH = None
        self.W = None
        if explicit_w:
            # the (1,1) block of f-inv written out: W = −H⁻¹ + H⁻¹Aᵀ F_H⁻¹ A H⁻¹, so that
            # F⁻¹[u; 0] has x-part W u (one dense GEMV per K_F product on c1-size problems)
            W = -sla.cho_solve(self.cH, np.eye(self.n))
            if self.m1:
                W += HiAt @ sla.cho_solve(self.cFH, HiAt.T)
            self.W = 0.5 * (W + W.T)

    def solve_x(self, r1):
        """x-part of F⁻¹ (r1; 0) (row 1 of f-inv with r2 = 0)."""
        if self.W is not None:
            return self.W @ r1
        return self.solve(r1, None)[0]

    def Hinv(self, v):
        return sla.cho_solve(self.cH, v)

    def solve(self, r1, r2=None):
        """Return (y, z) = F⁻¹ (r1; r2), block by block as in f-inv."""
        t = self.Hinv(r1)                                    # H⁻¹ r1
        if self.m1 == 0:
            return -t, np.zeros((0,) + np.shape(r1)[1:])
        if r2 is None:
            r2 = np.zeros((self.m1,) + np.shape(r1)[1:])
        # row 2 of f-inv:  z = F_H⁻¹ A H⁻¹ r1 + F_H⁻¹ r2
        z = sla.cho_solve(self.cFH, self.A @ t) + sla.cho_solve(self.cFH, r2)
        # row 1 of f-inv:  y = (−H⁻¹ + H⁻¹AᵀF_H⁻¹AH⁻¹) r1 + H⁻¹AᵀF_H⁻¹ r2
        #                    = −t + H⁻¹Aᵀ z
        y = -t + self.Hinv(self.A.T @ z)
        return y, z


class SparseF:
    """F⁻¹ through SuperLU on P F Pᵀ (x block by ``x_perm``, λ block last).

    NATURAL ordering and diag_pivot_thresh=0 keep the given order and static
    diagonal pivots.
    """

    def __init__(self, H, A, x_perm=None):
        n, m1 = H.shape[0], A.shape[0]
        self.n, self.m1 = n, m1
        if x_perm is None:
            x_perm = np.arange(n)
        self.perm = np.concatenate([np.asarray(x_perm, dtype=np.int64), n + np.arange(m1)])
        F = assemble_F(H, A).tocsr()
        Fp = F[self.perm][:, self.perm].tocsc()
        self.lu = spla.splu(Fp, permc_spec="NATURAL", diag_pivot_thresh=0.0,
                            options=dict(SymmetricMode=True))

    def solve(self, r1, r2=None):
        n, m1 = self.n, self.m1
        if r2 is None:
            r2 = np.zeros((m1,) + np.shape(r1)[1:])
        rhs = np.concatenate([r1, r2])
        sol_p = self.lu.solve(rhs[self.perm])
        sol = np.empty_like(sol_p)
        sol[self.perm] = sol_p
        return sol[:n], sol[n:]


class BlockF:
    """F⁻¹ through the block-inverse formula f-inv with a SPARSE factor of H.

    Same algebra as ``DenseF`` — y = −H⁻¹r1 + H⁻¹Aᵀz, z = F_H⁻¹(AH⁻¹r1 + r2),
    F_H = AH⁻¹Aᵀ — but H⁻¹ is applied through SuperLU's LU of the SPD H (no
    pivoting needed: diag_pivot_thresh = 0) in a fill-reducing column order
    (``x_perm`` when given, e.g. the generator's grid nested dissection, else
    SuperLU's own minimum degree on H + Hᵀ, ``MMD_AT_PLUS_A``), and the small dense
    F_H (m1 × m1) by LAPACK Cholesky.  No factor of F itself is formed, so this
    route shares nothing with an LDLᵀ of F.  For the full-size configs
    ("sparse" configs), where the dense H of ``DenseF`` does
    not fit.
    """

    def __init__(self, H, A, x_perm=None, batch=256):
        H = sp.csc_matrix(H)
        A = sp.csr_matrix(A)
        self.n, self.m1 = H.shape[0], A.shape[0]
        self.A = A
        if x_perm is not None:
            p = np.asarray(x_perm, dtype=np.int64)
            self.hp = p
            Hp = H[p][:, p].tocsc()
            self.lu = spla.splu(Hp, permc_spec="NATURAL", diag_pivot_thresh=0.0,
                                options=dict(SymmetricMode=True))
        else:
            self.hp = None
            self.lu = spla.splu(H, permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                                options=dict(SymmetricMode=True))
        if self.m1:
            FH = np.empty((self.m1, self.m1))
            At = A.T.tocsc()
            for c0 in range(0, self.m1, batch):            # F_H = A (H⁻¹ Aᵀ), column batches
                c1 = min(self.m1, c0 + batch)
                HiAt = self.Hinv(At[:, c0:c1].toarray())
                FH[:, c0:c1] = A @ HiAt
            FH = 0.5 * (FH + FH.T)                            # exact symmetry of AH⁻¹Aᵀ
            self.cFH = sla.cho_factor(FH, lower=True, overwrite_a=True)
        else:
            self.cFH = None

    def Hinv(self, v):
        v = np.asarray(v, dtype=float)
        if self.hp is None:
            return self.lu.solve(v)
        out = np.empty_like(v)
        out[self.hp] = self.lu.solve(v[self.hp])
        return out

    def solve_x(self, r1):
        return self.solve(r1, None)[0]

    def solve(self, r1, r2=None):
        """Return (y, z) = F⁻¹ (r1; r2), block by block as in f-inv."""
        t = self.Hinv(r1)
        if self.m1 == 0:
            return -t, np.zeros((0,) + np.shape(r1)[1:])
        if r2 is None:
            r2 = np.zeros((self.m1,) + np.shape(r1)[1:])
        z = sla.cho_solve(self.cFH, self.A @ t + r2)
        y = -t + self.Hinv(self.A.T @ z)
        return y, z


def make_fsolver(H, A, x_perm=None, dense_limit=30000):
    """Dense block formula up to ``dense_limit`` unknowns, the sparse-H block formula beyond."""
    if H.shape[0] + A.shape[0] <= dense_limit and x_perm is None:
        return DenseF(H, A)
    return BlockF(H, A, x_perm)
