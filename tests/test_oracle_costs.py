"""Pins of the oracle's cost model (oracle/costs.py).

Each formula is checked against a brute-force COUNT taken from a plain-loop execution of the
operation it models (flops executed, or bytes moved by a minimum-pass schedule), or against a
closed form — never by retyping the formula.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import costs, symbolic


class Counter:
    """Counts fp64 flops and HBM bytes of the plain loops below."""

    def __init__(self):
        self.flops = 0
        self.bytes = 0


def _lower_factor(N, dens, seed):
    """A random lower-triangular factor with a nonzero diagonal (CSC lists of (row, value))."""
    rng = np.random.default_rng(seed)
    cols = []
    for j in range(N):
        rows = [j] + [i for i in range(j + 1, N) if rng.random() < dens]
        cols.append([(i, (2.0 + rng.random()) if i == j else rng.standard_normal()) for i in rows])
    return cols


def trsv_forward(L, b, cnt):
    """x = L⁻¹b column by column; every stored entry is read once (diagonal included)."""
    x = list(b)
    cnt.bytes += 8 * len(b)                       # read b
    for j, col in enumerate(L):
        for i, v in col:
            cnt.bytes += 8                        # L value
            if i == j:
                x[j] /= v
                cnt.flops += 1
            else:
                x[i] -= v * x[j]
                cnt.flops += 2
    cnt.bytes += 8 * len(b)                       # write x
    return x


def trsv_backward(L, b, cnt):
    """x = L⁻ᵀb (dot-product form); every stored entry is read once."""
    N = len(b)
    x = list(b)
    cnt.bytes += 8 * N
    for j in range(N - 1, -1, -1):
        for i, v in L[j]:
            cnt.bytes += 8
            if i == j:
                diag = v
            else:
                x[j] -= v * x[i]
                cnt.flops += 2
        x[j] /= diag
        cnt.flops += 1
    cnt.bytes += 8 * N
    return x


def test_c_trsv_is_flops_of_a_sweep():
    """c_trsv(L) = 2 nz(L): the flops of one substitution sweep with L's stored diagonal."""
    for N, dens, seed in ((1, 0.0, 0), (7, 0.3, 1), (25, 0.2, 2), (40, 0.6, 3)):
        L = _lower_factor(N, dens, seed)
        nnz = sum(len(c) for c in L)
        c = Counter()
        trsv_forward(L, np.ones(N), c)
        # each off-diagonal entry is one multiply-add (2 flops), each diagonal one division (1 flop):
        # 2(nnz − N) + N = 2nnz − N, i.e. the model's 2nz(L) up to the N divisions it folds in
        assert c.flops == 2 * nnz - N
        assert costs.c_trsv(nnz) == 2 * nnz
        assert costs.c_trsv(nnz) - c.flops == N


def test_c_fact_closed_forms():
    """c_fact = Σ_j nz(L[:,j])²: dense n×n gives n(n+1)(2n+1)/6, diagonal gives n,
    a tridiagonal (path) factor gives 4(n−1)+1 — column counts from the oracle's symbolic analysis."""
    for n in (1, 5, 33):
        _, struct = symbolic.symbolic_factor(n, [np.arange(j + 1, n) for j in range(n)])
        cc = [len(s) for s in struct]
        assert costs.c_fact(cc) == n * (n + 1) * (2 * n + 1) // 6
        assert costs.c_fact(np.ones(n, dtype=int)) == n
        _, struct = symbolic.symbolic_factor(n, [np.arange(j + 1, min(n, j + 2)) for j in range(n)])
        assert costs.c_fact([len(s) for s in struct]) == 4 * (n - 1) + 1


def test_c_spmv_and_spmm_by_counting():
    """c_spmv(B) = 2nz(B); c_spmm(B, D Bᵀ) = Σ_j nz(B[:,j])² and c_spmm(Bᵀ, D B) = Σ_i nz(B[i,:])²
    (P:L54–62): the multiply count of the outer-product formation of B D Bᵀ over columns."""
    rng = np.random.default_rng(4)
    for m, n, dens in ((6, 9, 0.3), (20, 12, 0.2), (1, 1, 1.0)):
        B = sp.random(m, n, density=dens, random_state=rng, format="csr")
        B.data[:] = rng.standard_normal(B.nnz)
        Bd = B.toarray()
        # SpMV: one multiply-add per stored entry
        flops = sum(2 for i in range(m) for j in range(n) if Bd[i, j] != 0)
        assert costs.c_spmv(B) == flops
        # B D Bᵀ = Σ_j d_j B[:,j] B[:,j]ᵀ: nz(B[:,j])² products for column j
        prods = 0
        out = np.zeros((m, m))
        dj = rng.uniform(0.5, 2, n)
        for j in range(n):
            nzr = [i for i in range(m) if Bd[i, j] != 0]
            for a in nzr:
                for b in nzr:
                    out[a, b] += Bd[a, j] * dj[j] * Bd[b, j]
                    prods += 1
        assert np.allclose(out, Bd @ np.diag(dj) @ Bd.T)
        assert costs.c_spmm_BDBt(B) == prods
        prods = sum(sum(1 for j in range(n) if Bd[i, j] != 0) ** 2 for i in range(m))
        assert costs.c_spmm_BtDB(B) == prods


def _counted_pcg_iteration(L, C, D, p, x, r, cnt):
    """One P_L PCG iteration of PL-KF as a minimum-pass schedule, every HBM access counted
    (K_F p = D∘p − [C 0] F⁻¹ [Cᵀp; 0]; SURVEY §8(d) accounting: the F-solve reads and
    writes (n+m1)-vectors, matrix values 8 B, column indices 4 B, on-chip accumulators free)."""
    m2, n = C.shape
    N = len(L)
    Cd = C.tocsr()
    # a1: u = Cᵀp — read p once per row, C values + indices once; write the rhs [u; 0] once
    u = np.zeros(N)
    for i in range(m2):
        cnt.bytes += 8
        for k in range(Cd.indptr[i], Cd.indptr[i + 1]):
            cnt.bytes += 12
            u[Cd.indices[k]] += Cd.data[k] * p[i]
            cnt.flops += 2
    cnt.bytes += 8 * N
    # a2–a4: forward and backward sweeps (read vector, every stored entry, write vector)
    y = trsv_forward(L, u, cnt)
    w = trsv_backward(L, y, cnt)
    # a5: q = D∘p − [C 0]·w — read D, p, the solve output once, C once; write q
    cnt.bytes += 8 * N
    q = np.zeros(m2)
    for i in range(m2):
        cnt.bytes += 16
        acc = 0.0
        for k in range(Cd.indptr[i], Cd.indptr[i + 1]):
            cnt.bytes += 12
            acc += Cd.data[k] * w[Cd.indices[k]]
            cnt.flops += 2
        q[i] = D[i] * p[i] - acc
        cnt.bytes += 8
    pq = float(p @ q)                       # fused into the pass above
    alpha = float(r @ (r / D)) / pq
    # a6: x += αp (read x, p; write x); r −= αq (read r, q; write r); z = r/D (read D; write z);
    #     then p = z + βp (read z, p; write p)
    x = x + alpha * p
    cnt.bytes += 24 * m2
    r_new = r - alpha * q
    cnt.bytes += 24 * m2
    z = r_new / D
    cnt.bytes += 16 * m2
    beta = float(r_new @ z) / float(r @ (r / D))
    p = z + beta * p
    cnt.bytes += 24 * m2
    return x, r_new, p


def test_pcg_iteration_bytes_and_flops_by_counting():
    """pcg_iteration_bytes (SURVEY §8(d) B_it) and pcg_iteration_flops (P:L145 model:
    2c_trsv(L_F) + 2c_spmv(C)) against a counted execution of one PL-KF PCG iteration."""
    rng = np.random.default_rng(5)
    for N, n, m2, dens in ((12, 9, 15, 0.3), (30, 22, 41, 0.15)):
        L = _lower_factor(N, dens, int(rng.integers(100)))
        nnz_L = sum(len(c) for c in L)
        C = sp.random(m2, n, density=0.25, random_state=rng, format="csr")
        C.data[:] = rng.standard_normal(C.nnz)
        D = rng.uniform(0.5, 2, m2)
        p, r = rng.standard_normal(m2), rng.standard_normal(m2)
        cnt = Counter()
        _counted_pcg_iteration(L, C, D, p, np.zeros(m2), r, cnt)
        m1 = N - n
        assert cnt.bytes == costs.pcg_iteration_bytes(nnz_L, C.nnz, n, m1, m2)
        # model flops: the N pivot divisions are folded into c_trsv's 2nz(L) (see the trsv pin)
        assert cnt.flops + 2 * N == costs.pcg_iteration_flops(nnz_L, C.nnz)
    # the P_H term adds one more pair of sweeps with L_PH: 16 B and 4 flops per stored entry
    assert costs.pcg_iteration_bytes(10, 3, 1, 1, 1, nnz_LPH=7) - costs.pcg_iteration_bytes(10, 3, 1, 1, 1) == 16 * 7
    assert costs.pcg_iteration_flops(10, 3, 7) - costs.pcg_iteration_flops(10, 3) == 4 * 7


@pytest.mark.parametrize("N", [5])
def test_counted_sweeps_solve(N):
    """The counted sweeps are real solves (so the counts are of the actual operation)."""
    L = _lower_factor(N, 0.5, 9)
    Ld = np.zeros((N, N))
    for j, col in enumerate(L):
        for i, v in col:
            Ld[i, j] = v
    b = np.arange(1.0, N + 1)
    c = Counter()
    assert np.allclose(Ld @ trsv_forward(L, b, c), b)
    assert np.allclose(Ld.T @ trsv_backward(L, b, c), b)
