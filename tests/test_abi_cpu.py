"""CPU-side checks of the C-ABI library: it builds, loads, exports every symbol
declared in include/qp_b200.h, refuses to compute without a GPU (no CPU
fallback), and its host symbolic analysis (qp_analyse) matches the oracle's
structures bit-exactly."""
import numpy as np
import pytest

import qpgen
from oracle import costs, symbolic

P = pytest.importorskip("paper_2104_12916_b200")

KEYS = ("parent", "colcount", "sn_start", "sn_parent", "sn_level", "sn_rowptr", "sn_rows", "row_level")


def test_library_exports_header_symbols():
    P.load_library()
    exported = set(P.exported_symbols())
    declared = P.header_functions()
    assert declared, "no functions parsed from include/qp_b200.h"
    missing = [f for f in declared if f not in exported]
    assert not missing, missing


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    qp = qpgen.make("c0")
    with pytest.raises(P.QPError) as ei:
        P.binding.from_qp(qp)
    assert ei.value.code == -5     # QP_ECUDA


def _path30():
    import scipy.sparse as sp
    n = 30
    H = sp.diags([np.full(n - 1, -1.0), np.full(n, 4.0), np.full(n - 1, -1.0)], [-1, 0, 1], format="csr")
    return qpgen.QP(H=qpgen.canonical_csr(H), A=qpgen.canonical_csr(sp.csr_matrix((0, n))),
                    C=qpgen.canonical_csr(sp.identity(n, format="csr")), g=np.zeros(n), b=np.zeros(0),
                    d=np.zeros(n), x_perm=np.arange(n))


@pytest.mark.parametrize("name", ["c0", "tiny", "m1_zero", "m1_eq_n", "ragged", "grid", "syqp", "path30", "absorb",
                                  "c3s"])
def test_host_symbolic_matches_oracle(name):
    qp = {"c0": lambda: qpgen.make("c0"),
          "tiny": lambda: qpgen.scaled_random_qp(9, 4, 12, seed=1, g_nnz=3, a_nnz=3, c_nnz=3),
          "m1_zero": lambda: qpgen.scaled_random_qp(30, 0, 40, seed=2, g_nnz=3, a_nnz=3, c_nnz=3),
          "m1_eq_n": lambda: qpgen.make_syqp(24, 24),
          "ragged": lambda: qpgen.scaled_random_qp(700, 130, 900, seed=3),
          "grid": lambda: qpgen.make_grid_qp(24, 40, 60, seed=4, name="grid24"),
          "syqp": lambda: qpgen.make_syqp(64, 20),
          "path30": _path30,                                                   # hand-worked relax example
          "absorb": lambda: qpgen.scaled_random_qp(2000, 500, 3000, seed=5, g_nnz=8, a_nnz=4, c_nnz=6),
          "c3s": lambda: qpgen.make("c3s")}[name]()
    a = P.Analysis(qp.H, qp.A, qp.x_perm)
    perm = a.structure("perm")
    assert sorted(perm[:qp.n].tolist()) == list(range(qp.n))
    assert perm[qp.n:].tolist() == list(range(qp.n, qp.n + qp.m1))      # λ block last, in row order
    # the oracle decides the forced trailing supernode itself (symbolic.choose_trailing); the library
    # absorbs only under its own ordering (x_perm None)
    ref = symbolic.analyse_auto(qp.H, qp.A, perm[:qp.n], absorb=qp.x_perm is None)
    assert int(a.structure("trailing_from")[0]) == ref["trailing_from"]
    for k in KEYS:
        assert symbolic.struct_hash(a.structure(k)) == symbolic.struct_hash(ref[k]), k
    st = a.stats()
    assert st["nnz_LF"] == ref["nnz_L"] and st["nnz_LF_stored"] == ref["nnz_stored"]
    # the paper's cost model: the library's c_fact(F) equals the oracle's Σ_j cc(j)² exactly
    assert int(st["c_fact_F"]) == costs.c_fact(ref["colcount"])
    if name == "path30":
        assert a.structure("sn_start").tolist() == [0, 16, 30]
    if name == "absorb":
        assert ref["trailing_from"] > 0          # the case exercises the absorption rule


def test_min_degree_reduces_fill():
    qp = qpgen.scaled_random_qp(400, 50, 100, seed=9)
    nat = P.Analysis(qp.H, qp.A, np.arange(qp.n)).stats()["nnz_LF"]
    md = P.Analysis(qp.H, qp.A).stats()["nnz_LF"]
    assert md < nat


def test_setup_rejects_bad_inputs_before_touching_a_gpu():
    """qp_setup validates shapes, CSR canonicality, symmetry and finiteness first (QP_EINVAL), so these
    errors are reported identically with or without a GPU."""
    import numpy as np
    import scipy.sparse as sp
    from paper_2104_12916_b200.binding import QPError, QPSolver
    qp = qpgen.make("c0")
    bad_g = qp.g.copy()
    bad_g[0] = np.nan
    H_asym = sp.csr_matrix(qp.H.toarray() + np.triu(np.ones((qp.n, qp.n)), 1) * 1e-3)
    for args in ((qp.H, qp.A, qp.C, bad_g, qp.b, qp.d),
                 (H_asym, qp.A, qp.C, qp.g, qp.b, qp.d),
                 (qp.H, qp.A, sp.csr_matrix((0, qp.n)), qp.g, qp.b, np.zeros(0)),
                 (qp.H, sp.csr_matrix((qp.n + 1, qp.n)), qp.C, qp.g, np.zeros(qp.n + 1), qp.d)):
        with pytest.raises(QPError) as e:
            QPSolver(*args)
        assert e.value.code == -1, e.value
