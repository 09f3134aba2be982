"""GPU parity of the alternative K_F / PCG paths, each against the CPU oracle.

The library picks its K_F product path at setup (include/qp_b200.h qp_stats): the explicit x-block
W = (F⁻¹)₁₁ when it reads fewer bytes than an F-solve, else the flattened forest or the sweeps; the
P_L PCG runs as one fused cooperative step per iteration, with long rows of C (> 32 entries) warp per
row.  The A/B switches QPB_DENSE_W=0 / QPB_FUSED_PCG=0 are read once per process, so every variant
runs in its own subprocess; each must match the oracle on the same (D, rhs) at a fixed iteration count
(reading c5#16: 1e-8 relative) and, on c0, reach the oracle's IPM objective (1e-8 relative).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import qpgen
from oracle import kkt
from oracle.fsolve import DenseF
from oracle.ipm import ipm_solve as oracle_ipm
from oracle.pcg import pcg as oracle_pcg

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import qpgen
from paper_2104_12916_b200.binding import from_qp
qp = eval(sys.argv[2])
s = from_qp(qp)
s.ipm_factor_once('low')
st = s.stats()
rng = np.random.default_rng(8)
D = rng.uniform(0.5, 2.0, qp.m2)
b = rng.standard_normal(qp.m2)
out = {"dense_w": st["dense_w_enabled"], "flat": st["flat_enabled"], "pi": st["pi_enabled"],
       "pi_levels": st["pi_levels"], "lvl": st["lvl_levels_F"], "st": st["pi_subtrees"], "xs": {}}
if len(sys.argv) > 4 and sys.argv[4] == 'fsolve':
    f = np.random.default_rng(12).standard_normal(qp.n + qp.m1)
    out["fsolve"] = np.concatenate(s.f_solve(f)).tolist()
for k in (1, 3, 7):
    x, it, rr, rc = s.pcg_solve(D, b, tol=0.0, maxit=k)
    out["xs"][str(k)] = [it, x.tolist()]
if sys.argv[3] == '1':
    res = s.ipm_solve(ipm_tol=1e-10)
    out["obj"] = res["objective"]
    out["converged"] = bool(res["converged"])
print("RESULT " + json.dumps(out))
'''

CASES = {
    "c0": "qpgen.make('c0')",
    "ragged": "qpgen.scaled_random_qp(700, 130, 900, seed=3)",
    # every row of C has 40 entries: the fused step's warp-per-row branch
    "long_rows": "qpgen.scaled_random_qp(300, 60, 400, seed=5, c_nnz=40)",
    # dense F with a large λ block: W (n²/2 words) reads fewer bytes than an F-solve ((n+m1)²/2 words)
    "dense_m1": "qpgen.scaled_random_qp(400, 200, 500, seed=6, g_nnz=8)",
}
VARIANTS = {"default": {}, "no_dense_w": {"QPB_DENSE_W": "0"}, "force_w": {"QPB_DENSE_W": "2"},
            "unfused": {"QPB_FUSED_PCG": "0"}, "unfused_no_w": {"QPB_FUSED_PCG": "0", "QPB_DENSE_W": "0"},
            "unfused_force_w": {"QPB_FUSED_PCG": "0", "QPB_DENSE_W": "2"}}


def run_child(expr, env_extra, ipm, extra=()):
    env = dict(os.environ)
    env.update(env_extra)
    p = subprocess.run([sys.executable, "-c", CHILD, ROOT, expr, "1" if ipm else "0", *extra], capture_output=True,
                       text=True, env=env,
                       timeout=600, cwd=ROOT)
    line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    assert p.returncode == 0 and line, p.stderr[-2000:]
    return json.loads(line[-1][7:])


@pytest.fixture(scope="module", params=list(CASES))
def oracle_case(request):
    qp = eval(CASES[request.param])
    fs = DenseF(qp.H, qp.A)
    rng = np.random.default_rng(8)
    D = rng.uniform(0.5, 2.0, qp.m2)
    b = rng.standard_normal(qp.m2)
    ref = {}
    for k in (1, 3, 7):
        xr, itr, *_ = oracle_pcg(lambda v: kkt.KF_apply(qp, fs, D, v), b, kkt.PrecondL(D), 0.0, k)
        ref[k] = xr
    obj = None
    if request.param == "c0":   # PL-KF oracle IPMs at the other sizes take thousands of dense PCG steps
        r = oracle_ipm(qp, precond="low", ipm_tol=1e-10, fs=fs)
        assert r.converged
        obj = r.objective
    return request.param, qp, ref, obj


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_path_variant_matches_oracle(oracle_case, variant):
    name, qp, ref, obj = oracle_case
    out = run_child(CASES[name], VARIANTS[variant], obj is not None)
    if name == "dense_m1" and variant in ("default", "unfused"):
        assert out["dense_w"] == 1.0          # chosen by bytes
    if name == "c0" and variant == "default":
        assert out["dense_w"] == 1.0          # c0 (N = 250): the small-N explicit F⁻¹, W its x-block
    if VARIANTS[variant].get("QPB_DENSE_W") == "0":
        assert out["dense_w"] == 0.0
    if VARIANTS[variant].get("QPB_DENSE_W") == "2":
        assert out["dense_w"] == 1.0
    for k, xr in ref.items():
        it, x = out["xs"][str(k)]
        assert it == k
        x = np.asarray(x)
        assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr), (k, np.linalg.norm(x - xr) / np.linalg.norm(xr))
    if obj is not None:
        assert out["converged"]
        assert abs(out["obj"] - obj) <= 1e-8 * max(1.0, abs(obj))


PI_ENV = {"QPB_PI_MINN": "0", "QPB_DENSE_FINV": "0", "QPB_DENSE_W": "0", "QPB_FLAT": "0", "QPB_PI": "2"}


@pytest.mark.parametrize("variant", ["subtrees", "subtrees32", "subtrees_fused_rhs", "leaf_phase", "all_levels", "off"])
def test_level_products_match_oracle(variant):
    """Level products (Z_J = [L_JJ⁻¹; L_ext L_JJ⁻¹], one kernel per elimination-tree level) on a
    grid QP small enough for the dense oracle: the F-solve and the P_L PCG iterates against the oracle with
    (a) subtrees swept by one CTA each below them (16 and 32 lanes per supernode), (b) the leaf phase below
    them, (c) every level swept as a product, (d) switched off (the task graph)."""
    expr = "qpgen.make_grid_qp(48, 80, 200, seed=9, name='grid48')"
    qp = eval(expr)
    env = dict(PI_ENV)
    env.update({"subtrees": {"QPB_ST_MIN": "1", "QPB_ST_KB": "8", "QPB_ST": "2"},
                "subtrees32": {"QPB_ST_MIN": "1", "QPB_ST_KB": "40", "QPB_ST": "2"},
                # Cᵀp gathered inside the sweep kernels (no pregather SpMV, no phase D in the fused step)
                "subtrees_fused_rhs": {"QPB_ST_MIN": "1", "QPB_ST_KB": "8", "QPB_PREGATHER": "0", "QPB_ST": "2"},
                "leaf_phase": {"QPB_LVL_MIN": "16", "QPB_ST": "0"}, "all_levels": {"QPB_LVL": "0", "QPB_ST": "0"},
                "off": {"QPB_PI": "0"}}[variant])
    out = run_child(expr, env, False, extra=("fsolve",))
    assert out["dense_w"] == 0.0 and out["flat"] == 0.0
    if variant == "off":
        assert out["pi"] == 0.0
    else:
        assert out["pi"] == 1.0 and out["pi_levels"] >= 2
        assert (out["lvl"] > 0) == (variant == "leaf_phase") or variant.startswith("subtrees")
        assert (out["st"] > 0) == variant.startswith("subtrees")
    fs = DenseF(qp.H, qp.A)
    f = np.random.default_rng(12).standard_normal(qp.n + qp.m1)
    yr = np.concatenate(fs.solve(f[:qp.n], f[qp.n:]))
    y = np.asarray(out["fsolve"])
    assert np.linalg.norm(y - yr) <= 1e-9 * np.linalg.norm(yr), np.linalg.norm(y - yr) / np.linalg.norm(yr)
    rng = np.random.default_rng(8)
    D = rng.uniform(0.5, 2.0, qp.m2)
    b = rng.standard_normal(qp.m2)
    for k in (1, 3, 7):
        xr, itr, *_ = oracle_pcg(lambda v: kkt.KF_apply(qp, fs, D, v), b, kkt.PrecondL(D), 0.0, k)
        it, x = out["xs"][str(k)]
        assert it == k
        assert np.linalg.norm(np.asarray(x) - xr) <= 1e-8 * np.linalg.norm(xr)


def test_debug_timeline_records_pcg_launches():
    """qp_debug_timeline: one fused PCG step per iteration (inside and outside the CUDA graph), every
    recorded launch has start ≤ end, and launches of one kernel do not overlap (stream order)."""
    from paper_2104_12916_b200.binding import from_qp
    qp = qpgen.make("c0")
    s = from_qp(qp)
    s.ipm_factor_once("low")
    rng = np.random.default_rng(3)
    D, b = rng.uniform(0.5, 2.0, qp.m2), rng.standard_normal(qp.m2)
    s.pcg_solve(D, b, tol=0.0, maxit=10)          # graph captured
    s.debug_timeline(True)
    x, it, rr, rc = s.pcg_solve(D, b, tol=0.0, maxit=10)
    ev = s.debug_timeline(False)
    assert it == 10
    assert sum(1 for k, a, e in ev if k == 4) == 10     # k_pcg_step
    assert sum(1 for k, a, e in ev if k == 2) >= 10     # the dense GEMV of every F-solve (S⁻¹ or W)
    assert all(a <= e for k, a, e in ev)
    for kk in {k for k, a, e in ev}:
        spans = sorted((a, e) for k, a, e in ev if k == kk)
        assert all(e0 <= a1 for (a0, e0), (a1, e1) in zip(spans, spans[1:]))
    s.close()
