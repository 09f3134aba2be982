"""Oracle symbolic structures of the LDLᵀ factor of F (TEST INFRASTRUCTURE ONLY).

The paper factors F once with an LDLᵀ whose factor L_F has
nz(L_F[:,j]) entries per column.  The structures here
are what the library's symbolic phase must reproduce bit-exactly, given the
same x-block permutation:

* ordering: x block by ``x_perm``, then the λ block last in row order;
* elimination tree and column structures by the definition of symbolic
  elimination: struct(L[:,j]) = {j} ∪ {i>j : F_ij ≠ 0}
  ∪ ⋃_{c : parent(c)=j} struct(L[:,c]) \\ {c},   parent(j) = min(struct(j) \\ {j});
* column counts cc(j) = |struct(L[:,j])| (diagonal included);
* fundamental supernodes: column j joins j−1's supernode iff
  parent(j−1) = j and cc(j−1) = cc(j) + 1 (then struct(j−1) = {j−1} ∪ struct(j));
* relaxed amalgamation, repeated passes in increasing
  supernode order until no merge happens: merge J into its parent P when J's columns end right before P's and
  the merged block's explicit zeros are small — merged width w ≤ 4, or
  w ≤ 16 and zeros ≤ 80 %, or w ≤ 48 and zeros ≤ 10 %, or zeros ≤ 5 % of
  the stored w·m − w(w−1)/2 entries (m = w_J + m_P rows);  a relaxed
  supernode's rows are its columns followed by the rows below its topmost
  fundamental supernode;
* forced dense trailing supernode (input `trailing_from`; ``analyse_auto`` derives it with
  ``choose_trailing`` from the oracle's own structures): after amalgamation every supernode reaching
  that column merges with the last one;
* supernodal tree: parent of supernode J = supernode of parent(last col of J);
  level(J) = 0 for leaves, else 1 + max level(children);
* row levels: lev(i) = 1 + max{lev(j) : j < i, L_ij ≠ 0}, 0 for rows with no
  off-diagonal entry.
"""
from __future__ import annotations

import hashlib

import numpy as np
import scipy.sparse as sp


def permuted_lower_pattern(H, A, x_perm=None):
    """Column lists of the strictly-lower pattern of P F Pᵀ, F = [−H Aᵀ; A 0]."""
    n, m1 = H.shape[0], A.shape[0]
    if x_perm is None:
        x_perm = np.arange(n)
    x_perm = np.asarray(x_perm, dtype=np.int64)
    pinv = np.empty(n, dtype=np.int64)
    pinv[x_perm] = np.arange(n)
    N = n + m1
    Hc = sp.coo_matrix(H)
    Ac = sp.coo_matrix(A)
    rows = np.concatenate([pinv[Hc.row], n + Ac.row])
    cols = np.concatenate([pinv[Hc.col], pinv[Ac.col]])
    lo = rows > cols
    P = sp.csc_matrix((np.ones(int(lo.sum())), (rows[lo], cols[lo])), shape=(N, N))
    P.sum_duplicates()
    P.sort_indices()
    return N, [P.indices[P.indptr[j]:P.indptr[j + 1]].astype(np.int64) for j in range(N)]


def symbolic_factor(N, lower_cols):
    """Elimination tree and full column structures (definition, in column order)."""
    parent = np.full(N, -1, dtype=np.int64)
    children = [[] for _ in range(N)]
    struct = [None] * N
    for j in range(N):
        parts = [np.array([j], dtype=np.int64), lower_cols[j]]
        for c in children[j]:
            sc = struct[c]
            parts.append(sc[sc != c])
        sj = np.unique(np.concatenate(parts))
        struct[j] = sj
        if len(sj) > 1:
            parent[j] = int(sj[1])
            children[int(sj[1])].append(j)
    return parent, struct


def supernodes(parent, cc):
    """Fundamental supernode start columns (with a final sentinel N)."""
    N = len(parent)
    starts = [0]
    for j in range(1, N):
        if not (parent[j - 1] == j and cc[j - 1] == cc[j] + 1):
            starts.append(j)
    starts.append(N)
    return np.asarray(starts, dtype=np.int64)


def _col2sn(starts, N):
    col2sn = np.empty(N, dtype=np.int64)
    for J in range(len(starts) - 1):
        col2sn[starts[J]:starts[J + 1]] = J
    return col2sn


def relax(parent, cc, struct, fstart, trailing_from=-1):
    """Relaxed amalgamation of the fundamental supernodes; returns (starts, rows-per-supernode)."""
    N = len(parent)
    nf = len(fstart) - 1
    col2f = _col2sn(fstart, N)
    fpar = [int(col2f[parent[fstart[J + 1] - 1]]) if parent[fstart[J + 1] - 1] >= 0 else -1 for J in range(nf)]
    below = [struct[fstart[J]][fstart[J + 1] - fstart[J]:] for J in range(nf)]
    c0 = [int(fstart[J]) for J in range(nf)]
    w = [int(fstart[J + 1] - fstart[J]) for J in range(nf)]
    m = [w[J] + len(below[J]) for J in range(nf)]
    true = [int(cc[fstart[J]:fstart[J + 1]].sum()) for J in range(nf)]
    alive = [True] * nf
    # passes over the current partition until no merge happens
    while True:
        own = np.empty(N, dtype=np.int64)
        for J in range(nf):
            if alive[J]:
                own[c0[J]:c0[J] + w[J]] = J
        merged = 0
        for J in range(nf):
            if not alive[J]:
                continue
            pc = parent[c0[J] + w[J] - 1]
            if pc < 0:
                continue
            P = int(own[pc])
            if not alive[P] or c0[J] + w[J] != c0[P]:
                continue
            ww = w[J] + w[P]
            mm = w[J] + m[P]
            stored = ww * mm - ww * (ww - 1) // 2
            zeros = stored - (true[J] + true[P])
            if ww <= 4 or (ww <= 16 and 100 * zeros <= 80 * stored) or (ww <= 48 and 100 * zeros <= 10 * stored) \
                    or 100 * zeros <= 5 * stored:
                c0[P], w[P], m[P], true[P] = c0[J], ww, mm, true[P] + true[J]
                alive[J] = False
                own[c0[P]:c0[P] + w[P]] = P
                merged += 1
        if merged == 0:
            break
    # forced dense trailing supernode: every supernode reaching column trailing_from merges with the last
    if 0 <= trailing_from < N:
        live = [J for J in range(nf) if alive[J]]
        first = next(J for J in live if c0[J] + w[J] > trailing_from)
        last = live[-1]
        if first != last:
            group = [J for J in live if J >= first]
            wsum = sum(w[J] for J in group)
            tsum = sum(true[J] for J in group)
            for J in group[:-1]:
                alive[J] = False
            c0[last], w[last], m[last], true[last] = N - wsum, wsum, wsum, tsum
            assert len(below[last]) == 0
    starts = [c0[J] for J in range(nf) if alive[J]] + [N]
    rows = [np.concatenate([np.arange(c0[J], c0[J] + w[J]), below[J]]).astype(np.int64)
            for J in range(nf) if alive[J]]
    return np.asarray(starts, dtype=np.int64), rows


def supernode_tree(parent, sn_start):
    ns = len(sn_start) - 1
    col2sn = np.empty(sn_start[-1], dtype=np.int64)
    for J in range(ns):
        col2sn[sn_start[J]:sn_start[J + 1]] = J
    sparent = np.full(ns, -1, dtype=np.int64)
    for J in range(ns):
        p = parent[sn_start[J + 1] - 1]
        if p >= 0:
            sparent[J] = col2sn[p]
    level = np.zeros(ns, dtype=np.int64)
    for J in range(ns):               # children have smaller indices than parents
        if sparent[J] >= 0:
            level[sparent[J]] = max(level[sparent[J]], level[J] + 1)
    return sparent, level


def row_levels(N, struct):
    lev = np.zeros(N, dtype=np.int64)
    for j in range(N):
        sj = struct[j]
        below = sj[sj > j]
        if len(below):
            lev[below] = np.maximum(lev[below], lev[j] + 1)
    return lev


def choose_trailing(sn_start, sn_parent, sn_level, sn_rowptr, budget_frac=0.02, bw=64):
    """Top-level absorption rule (DESIGN.md §4 "Top-level absorption"), decided from the oracle's
    own supernodal structures: if the factor ends in a dense root R (no parent, width w_R > 64, no
    rows below its columns) and the tree has more than 3 levels, take the lowest cut level L ≥ 1 such
    that merging every supernode J ≠ R of level ≥ L into R adds at most 2 % of R's w_R(w_R+1)/2
    entries as explicit zeros — Σ_J w_J·(w_R − (m_J − w_J)) for the rows of R each absorbed column
    lacks, plus wsum²/2 for the triangle between the absorbed columns — and return the first column
    of the absorbed block plus R (−1 when nothing is absorbed).  The absorbed columns must already be
    contiguous before R (the library's reordering, an equivalent order with the same fill)."""
    ns = len(sn_start) - 1
    if ns < 2:
        return -1
    R = ns - 1
    wR = int(sn_start[R + 1] - sn_start[R])
    mR = int(sn_rowptr[R + 1] - sn_rowptr[R])
    n_levels = int(np.max(sn_level)) + 1
    if not (sn_parent[R] < 0 and wR > bw and mR == wR and n_levels > 3):
        return -1
    w = np.diff(np.asarray(sn_start, dtype=np.int64))[:R]
    m = np.diff(np.asarray(sn_rowptr, dtype=np.int64))[:R]
    lev = np.asarray(sn_level)[:R]
    budget = budget_frac * wR * (wR + 1) / 2
    best = n_levels - 1
    for L in range(n_levels - 2, 0, -1):
        sel = lev >= L
        wsum = int(w[sel].sum())
        zeros = float(np.sum(w[sel].astype(float) * (wR - (m[sel] - w[sel])))) + wsum * wsum / 2
        if zeros > budget:
            break
        best = L
    if best >= n_levels - 1:
        return -1
    sel = lev >= best
    cols = np.concatenate([np.arange(sn_start[J], sn_start[J + 1]) for J in np.nonzero(sel)[0]] or [np.zeros(0, np.int64)])
    first = int(sn_start[R]) - int(w[sel].sum())
    if not np.array_equal(np.sort(cols), np.arange(first, int(sn_start[R]))):
        return -1                                  # not contiguous before the root: no absorption in this order
    return first


def analyse(H, A, x_perm=None, trailing_from=-1):
    """All structures, as a dict of int64 arrays.  trailing_from: first column of a forced dense
    trailing supernode (the library's absorbed tree top, exported as structure 9), or -1."""
    N, lower = permuted_lower_pattern(H, A, x_perm)
    parent, struct = symbolic_factor(N, lower)
    cc = np.array([len(s) for s in struct], dtype=np.int64)
    fsn = supernodes(parent, cc)
    sn, rows = relax(parent, cc, struct, fsn, trailing_from)
    sparent, slevel = supernode_tree(parent, sn)
    sn_rows = np.concatenate(rows) if N else np.zeros(0, np.int64)
    sn_rowptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    rlev = row_levels(N, struct)
    w = np.diff(sn)
    m = np.diff(sn_rowptr)
    nnz_stored = int(np.sum(w * m - w * (w - 1) // 2))
    return dict(N=N, parent=parent, colcount=cc, sn_start=sn, fsn_start=fsn, nnz_stored=nnz_stored,
                trailing_from=int(trailing_from) if 0 <= trailing_from < N else -1,
                sn_parent=sparent,
                sn_level=slevel, sn_rowptr=sn_rowptr, sn_rows=sn_rows, row_level=rlev,
                nnz_L=int(cc.sum()), struct=struct)


def struct_hash(arr) -> str:
    """64-bit hash of an int64 array together with its length."""
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.int64))
    h = hashlib.blake2b(digest_size=8)
    h.update(np.int64(len(a)).tobytes())
    h.update(a.tobytes())
    return h.hexdigest()


def analyse_auto(H, A, x_perm, absorb=True):
    """``analyse`` with the trailing column chosen by the oracle itself (``choose_trailing`` on the
    structures of the same order without a forced trailing supernode).  ``absorb`` = the library
    chose the ordering itself (it never reorders a caller-supplied x_perm)."""
    tf = -1
    if absorb:
        a0 = analyse(H, A, x_perm, trailing_from=-1)
        tf = choose_trailing(a0["sn_start"], a0["sn_parent"], a0["sn_level"], a0["sn_rowptr"])
        if tf < 0:
            return a0
    return analyse(H, A, x_perm, trailing_from=tf)
