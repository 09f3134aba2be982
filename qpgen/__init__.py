"""Seeded synthetic QP instance generator (shared input module).

This module is the ONLY code shared by the CPU oracle (``oracle/``) and the
CUDA path (``paper_2104_12916_b200``).  It builds problem DATA only — the
matrices H, A, C and vectors g, b, d of

    min ½xᵀHx + gᵀx   s.t.  Ax = b,  Cx ≥ d

— and holds none of the method's arithmetic (no factorization, no Krylov
solve, no IPM step).  Feasibility is constructed from a random interior point
(x0, s0): b = A·x0, d = C·x0 − s0 (BASELINE.json configs).

Recipes (readings c5#9–#14), all numpy PCG64:

* ``c0``  n=200,  m1=50,   m2=300,     H=GᵀG+0.1I (G 5 nnz/row), A 3/row, C 4/row
* ``c1``  n=2e4,  m1=5e3,  m2=4e4,     G 8/row, A 4/row, C 6/row
* ``c2``  1000×1000 grid, H = 5-point Laplacian + 0.01I, A 1e4 rows × 8,
          C = [I; −I; 2e5 random rows × 5]
* ``c3``  n=4e6, m1=2e5, m2=8e6, H = diag U(0.1,10) + GᵀG (G 2/row),
          A 6/row, C row degrees min(512, Zipf(2.1)+2)
* ``c3s`` the c3 recipe at 1/100 scale (end-to-end stand-in)
* ``c4``  5657×5657 grid, A 1e6 × 8, C 6.4e7 × 4, columns in a ±64 band
* ``c4s`` 512×512 grid, m1 = n/32, m2 = 2n, same bands (stand-in)
* ``syqp`` the paper's SyQPⁿ_{m1} family: block-diagonal H of
          4×4 MᵀM blocks, banded A ~ U[0,1), C = I, d = 0.

Draw order is fixed and documented in each builder; the same seed gives the
bit-identical problem.  Matrices are canonical CSR (sorted column indices,
no duplicates, float64 values); H is stored as
the full symmetric matrix.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import scipy.sparse as sp

__all__ = ["QP", "make", "make_random_qp", "make_grid_qp", "make_powerlaw_qp",
           "make_syqp", "CONFIGS", "grid_nd_perm", "canonical_csr"]


@dataclasses.dataclass
class QP:
    """A convex QP instance: min ½xᵀHx+gᵀx s.t. Ax=b, Cx≥d."""
    H: sp.csr_matrix
    A: sp.csr_matrix
    C: sp.csr_matrix
    g: np.ndarray
    b: np.ndarray
    d: np.ndarray
    name: str = ""
    x_perm: Optional[np.ndarray] = None   # optional fill-reducing order of the x block
    x0: Optional[np.ndarray] = None       # the interior point the data was built from
    s0: Optional[np.ndarray] = None

    @property
    def n(self) -> int:
        return self.H.shape[0]

    @property
    def m1(self) -> int:
        return self.A.shape[0]

    @property
    def m2(self) -> int:
        return self.C.shape[0]


def canonical_csr(M) -> sp.csr_matrix:
    """Sorted, duplicate-free CSR (scipy index dtypes; the binding widens indptr to int64)."""
    M = sp.csr_matrix(M, dtype=np.float64)
    M.sum_duplicates()
    M.sort_indices()
    M.eliminate_zeros()
    return M


def _distinct_cols(rng, nrows, ncols, k):
    """k distinct uniform columns in [0, ncols) per row (rejection redraw)."""
    k = min(k, ncols)
    cols = rng.integers(0, ncols, size=(nrows, k), dtype=np.int64)
    cols.sort(axis=1)
    while k > 1:
        dup = (np.diff(cols, axis=1) == 0).any(axis=1)
        if not dup.any():
            break
        idx = np.nonzero(dup)[0]
        new = rng.integers(0, ncols, size=(len(idx), k), dtype=np.int64)
        new.sort(axis=1)
        cols[idx] = new
    return cols


def _fixed_degree(rng, nrows, ncols, k, values="normal"):
    cols = _distinct_cols(rng, nrows, ncols, k)
    kk = cols.shape[1]
    if values == "normal":
        vals = rng.standard_normal(size=(nrows, kk))
    else:
        vals = rng.random(size=(nrows, kk))
    rows = np.repeat(np.arange(nrows, dtype=np.int64), kk)
    M = sp.csr_matrix((vals.ravel(), (rows, cols.ravel())), shape=(nrows, ncols))
    return canonical_csr(M)


def _banded_rows(rng, nrows, ncols, k, half=64):
    """Row i: k distinct columns in a ±half window around ⌊i·ncols/nrows⌋ (reading c5#10)."""
    anchor = (np.arange(nrows, dtype=np.int64) * ncols) // max(nrows, 1)
    width = min(2 * half + 1, ncols)
    lo = np.clip(anchor - half, 0, ncols - width)
    off = _distinct_cols(rng, nrows, width, k)
    cols = lo[:, None] + off
    kk = cols.shape[1]
    vals = rng.standard_normal(size=(nrows, kk))
    rows = np.repeat(np.arange(nrows, dtype=np.int64), kk)
    return canonical_csr(sp.csr_matrix((vals.ravel(), (rows, cols.ravel())), shape=(nrows, ncols)))


def _variable_degree(rng, degs, ncols):
    """Rows with the given degrees; distinct uniform columns, N(0,1) values."""
    nrows = len(degs)
    rows_l, cols_l, vals_l = [], [], []
    for k in np.unique(degs):
        idx = np.nonzero(degs == k)[0]
        c = _distinct_cols(rng, len(idx), ncols, int(k))
        v = rng.standard_normal(size=c.shape)
        rows_l.append(np.repeat(idx, c.shape[1]))
        cols_l.append(c.ravel())
        vals_l.append(v.ravel())
    M = sp.csr_matrix((np.concatenate(vals_l), (np.concatenate(rows_l), np.concatenate(cols_l))),
                      shape=(nrows, ncols))
    return canonical_csr(M)


def grid_laplacian(k: int, shift: float = 0.01) -> sp.csr_matrix:
    """5-point Laplacian on a k×k grid, Dirichlet boundary, + shift·I (reading c5#13)."""
    n = k * k
    idx = np.arange(n, dtype=np.int64)
    r, c = idx // k, idx % k
    rows = [idx]
    cols = [idx]
    vals = [np.full(n, 4.0 + shift)]
    for dr, dc in ((0, 1), (0, -1), (1, 0), (-1, 0)):
        ok = (r + dr >= 0) & (r + dr < k) & (c + dc >= 0) & (c + dc < k)
        rows.append(idx[ok])
        cols.append((r[ok] + dr) * k + (c[ok] + dc))
        vals.append(np.full(int(ok.sum()), -1.0))
    M = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    return canonical_csr(M)


def grid_nd_perm(k: int, leaf: int = 64) -> np.ndarray:
    """Geometric nested-dissection order of a k×k grid (new→old).

    Recursive coordinate bisection: split the longer side at its middle line,
    order part 1, part 2, then the separator line.  A fill-reducing ordering
    heuristic only (no method arithmetic); the library accepts it as x_perm.
    """
    out = []

    def rec(r0, r1, c0, c1):
        h, w = r1 - r0, c1 - c0
        if h <= 0 or w <= 0:
            return
        if h * w <= leaf or (h <= 2 and w <= 2):
            for r in range(r0, r1):
                out.extend(range(r * k + c0, r * k + c1))
            return
        if w >= h:
            m = (c0 + c1) // 2
            rec(r0, r1, c0, m)
            rec(r0, r1, m + 1, c1)
            out.extend(r * k + m for r in range(r0, r1))
        else:
            m = (r0 + r1) // 2
            rec(r0, m, c0, c1)
            rec(m + 1, r1, c0, c1)
            out.extend(range(m * k + c0, m * k + c1))

    import sys
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 10000))
    try:
        rec(0, k, 0, k)
    finally:
        sys.setrecursionlimit(old)
    p = np.asarray(out, dtype=np.int64)
    assert len(p) == k * k and len(np.unique(p)) == k * k
    return p


def _finish(name, H, A, C, g, x0, s0, x_perm=None):
    b = A @ x0
    d = C @ x0 - s0
    return QP(H=H, A=A, C=C, g=np.ascontiguousarray(g, dtype=np.float64),
              b=np.ascontiguousarray(b, dtype=np.float64),
              d=np.ascontiguousarray(d, dtype=np.float64), name=name,
              x_perm=x_perm, x0=x0, s0=s0)


def make_random_qp(n, m1, m2, g_nnz, a_nnz, c_nnz, seed=0, name="random"):
    """Configs 0 and 1 of BASELINE.json.

    Draw order: G (cols, vals), A (cols, vals), C (cols, vals), g, x0, s0.
    """
    rng = np.random.default_rng(seed)
    G = _fixed_degree(rng, n, n, g_nnz)
    A = _fixed_degree(rng, m1, n, a_nnz) if m1 > 0 else canonical_csr(sp.csr_matrix((0, n)))
    C = _fixed_degree(rng, m2, n, c_nnz)
    H = canonical_csr(G.T @ G + 0.1 * sp.identity(n, format="csr"))
    g = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    s0 = rng.uniform(0.1, 1.0, size=m2)
    return _finish(name, H, A, C, g, x0, s0)


def make_grid_qp(k, m1, n_rand, a_nnz=8, r_nnz=5, seed=0, name="grid", box=True, band=None,
                 m2_band=None, c_nnz_band=4):
    """Config 2 (box + random rows) and config 4 / c4s (banded rows).

    Draw order: g, x0, A (cols, vals), C-rows (cols, vals), s0.
    """
    rng = np.random.default_rng(seed)
    n = k * k
    H = grid_laplacian(k)
    g = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    if band is None:
        A = _fixed_degree(rng, m1, n, a_nnz)
        blocks = []
        if box:
            I = sp.identity(n, format="csr")
            blocks += [I, -I]
        if n_rand > 0:
            blocks.append(_fixed_degree(rng, n_rand, n, r_nnz))
        C = canonical_csr(sp.vstack(blocks, format="csr"))
    else:
        A = _banded_rows(rng, m1, n, a_nnz, half=band)
        C = _banded_rows(rng, m2_band, n, c_nnz_band, half=band)
    s0 = rng.uniform(0.1, 1.0, size=C.shape[0])
    return _finish(name, H, A, C, g, x0, s0, x_perm=grid_nd_perm(k))


def make_powerlaw_qp(n, m1, m2, seed=0, name="powerlaw", zipf_a=2.1, cap=512, shift=2):
    """Config 3 / c3s: H = diag U(0.1,10) + GᵀG (G 2/row), A 6/row, Zipf C rows (reading c5#9).

    Draw order: hdiag, G (cols, vals), A (cols, vals), C degrees, C (cols, vals), g, x0, s0.
    """
    rng = np.random.default_rng(seed)
    hdiag = rng.uniform(0.1, 10.0, size=n)
    G = _fixed_degree(rng, n, n, 2)
    A = _fixed_degree(rng, m1, n, 6)
    degs = np.minimum(cap, rng.zipf(zipf_a, size=m2) + shift).astype(np.int64)
    degs = np.minimum(degs, n)
    C = _variable_degree(rng, degs, n)
    H = canonical_csr(sp.diags(hdiag) + G.T @ G)
    g = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    s0 = rng.uniform(0.1, 1.0, size=m2)
    return _finish(name, H, A, C, g, x0, s0)


def make_syqp(n=64, m1=32, seed=0, block=4, bandwidth=3, name=None):
    """SyQPⁿ_{m1}: block-diagonal H from 4×4 MᵀM, M ~ U[0,1];
    banded full-rank A ~ U[0,1); C = I, d = 0.

    Readings: the band of A is A[i, i : i+bandwidth] (leading m1×m1 block upper
    triangular with a nonzero diagonal ⇒ full row rank); b = A·x0 with
    x0 ~ U(0.1, 1) so the family is strictly feasible (the paper draws b at
    random, which can be infeasible for x ≥ 0); the shared-H rule
    is honoured by drawing H from its own stream (seed, n).
    """
    rngH = np.random.default_rng([seed, n])
    nb = (n + block - 1) // block
    blocks = []
    for _ in range(nb):
        M = rngH.random((block, block))
        blocks.append(M.T @ M)
    H = canonical_csr(sp.block_diag([sp.csr_matrix(bk) for bk in blocks], format="csr").tocsr()[:n, :n])
    rng = np.random.default_rng([seed, n, m1])
    rows, cols = [], []
    for i in range(m1):
        for j in range(i, min(i + bandwidth, n)):
            rows.append(i)
            cols.append(j)
    vals = rng.random(len(rows))
    vals[np.asarray(cols) == np.asarray(rows)] += 0.5  # keep the diagonal away from 0
    A = canonical_csr(sp.csr_matrix((vals, (rows, cols)), shape=(m1, n)))
    c = rng.random(n)
    x0 = rng.uniform(0.1, 1.0, size=n)
    C = canonical_csr(sp.identity(n, format="csr"))
    b = A @ x0
    return QP(H=H, A=A, C=C, g=c, b=b, d=np.zeros(n), name=name or f"syqp{n}_{m1}",
              x0=x0, s0=x0.copy())


def _c0(seed=0):
    return make_random_qp(200, 50, 300, 5, 3, 4, seed, "c0")


def _c1(seed=0):
    return make_random_qp(20000, 5000, 40000, 8, 4, 6, seed, "c1")


def _c2(seed=0):
    return make_grid_qp(1000, 10000, 200000, seed=seed, name="c2")


def _c3(seed=0):
    return make_powerlaw_qp(4_000_000, 200_000, 8_000_000, seed, "c3")


def _c3s(seed=0):
    return make_powerlaw_qp(40_000, 2_000, 80_000, seed, "c3s")


def _c4(seed=0):
    k = 5657
    return make_grid_qp(k, 1_000_000, 0, seed=seed, name="c4", band=64, m2_band=64_000_000)


def _c4s(seed=0):
    k = 512
    n = k * k
    return make_grid_qp(k, n // 32, 0, seed=seed, name="c4s", band=64, m2_band=2 * n)


CONFIGS = {"c0": _c0, "c1": _c1, "c2": _c2, "c3": _c3, "c3s": _c3s, "c4": _c4, "c4s": _c4s}


def make(name: str, seed: int = 0) -> QP:
    """Build a named configuration (see module docstring)."""
    if name.startswith("syqp"):
        # syqp<n>_<m1>
        n_s, m_s = name[4:].split("_")
        return make_syqp(int(n_s), int(m_s), seed)
    return CONFIGS[name](seed)


def scaled_random_qp(n, m1, m2, seed=0, g_nnz=5, a_nnz=3, c_nnz=4, name=None):
    """Small random QPs of the config-0 family at other sizes (tests)."""
    return make_random_qp(n, m1, m2, g_nnz, a_nnz, c_nnz, seed, name or f"rand{n}_{m1}_{m2}")


@dataclasses.dataclass
class Probe:
    """Seeded probe inputs for parity at full size (shared by the golden script and the GPU tests).

    Data only — no method arithmetic.  Draw order (numpy PCG64, seed [seed, 7]): f (n+m1, N(0,1)),
    D (m2, exp U(−4, 4): a six-decade spread like mid-IPM D = V⁻¹S), p (m2, N(0,1)), b (m2, N(0,1));
    then the sample index sets (sorted, without replacement) for vectors of length n+m1 and m2.
    """
    f: np.ndarray
    D: np.ndarray
    p: np.ndarray
    b: np.ndarray
    idx_F: np.ndarray
    idx_m2: np.ndarray


def probe_inputs(qp: QP, seed: int = 0, nsample: int = 8192) -> Probe:
    rng = np.random.default_rng([seed, 7])
    N, m2 = qp.n + qp.m1, qp.m2
    f = rng.standard_normal(N)
    D = np.exp(rng.uniform(-4.0, 4.0, size=m2))
    p = rng.standard_normal(m2)
    b = rng.standard_normal(m2)
    idx_F = np.sort(rng.choice(N, size=min(N, nsample), replace=False)).astype(np.int64)
    idx_m2 = np.sort(rng.choice(m2, size=min(m2, nsample), replace=False)).astype(np.int64)
    return Probe(f=f, D=D, p=p, b=b, idx_F=idx_F, idx_m2=idx_m2)
