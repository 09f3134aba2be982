"""Dense spectral diagnostics (TEST INFRASTRUCTURE ONLY, tiny problems).

* KF_via_Finv      K_F = D − [C 0] F⁻¹ [Cᵀ; 0] with F⁻¹ = numpy.linalg.inv(F)
* KF_via_schur     K_F = D + C H⁻¹ (H − H̄_A) H⁻¹ Cᵀ, H̄_A = Aᵀ(AH⁻¹Aᵀ)⁻¹A
* precond_spectrum eigenvalues of P^{-1/2} K_F P^{-1/2}
"""
from __future__ import annotations

import numpy as np


def dense(M):
    return M.toarray() if hasattr(M, "toarray") else np.asarray(M, dtype=float)


def KF_via_Finv(qp, D):
    H, A, C = dense(qp.H), dense(qp.A), dense(qp.C)
    n, m1 = H.shape[0], A.shape[0]
    F = np.block([[-H, A.T], [A, np.zeros((m1, m1))]]) if m1 else -H
    Finv = np.linalg.inv(F)
    return np.diag(D) - C @ Finv[:n, :n] @ C.T


def HbarA(qp):
    H, A = dense(qp.H), dense(qp.A)
    Hi = np.linalg.inv(H)
    if A.shape[0] == 0:
        return np.zeros_like(H)
    return A.T @ np.linalg.inv(A @ Hi @ A.T) @ A


def KF_via_schur(qp, D):
    H, C = dense(qp.H), dense(qp.C)
    Hi = np.linalg.inv(H)
    return np.diag(D) + C @ Hi @ (H - HbarA(qp)) @ Hi @ C.T


def precond_spectrum(KF, P):
    w, V = np.linalg.eigh(P)
    Pmh = V @ np.diag(1.0 / np.sqrt(w)) @ V.T
    return np.linalg.eigvalsh(Pmh @ KF @ Pmh)
