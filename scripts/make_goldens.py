"""Write the full-size parity goldens (tests/golden/full/<cfg>.npz) from the CPU ORACLE only.

Calls only ``oracle/`` and the shared input module ``qpgen`` — nothing from the CUDA path.
For each BASELINE config (c1, c2) and stand-in (c3s, c4s) it stores, on the seeded probe
inputs of ``qpgen.probe_inputs`` (D with a six-decade spread, N(0,1) vectors):

* ``F``        y = F⁻¹f, sampled at idx_F, plus ‖y‖₂;
* ``KF``       q = K_F(D)·p, sampled at idx_m2, plus ‖q‖₂;
* ``PL<k>``    the P_L PCG iterate after k = 1, 3, 7 steps (tol 0) on K_F(D) x = b;
* ``PLeps``    the P_L PCG iteration count at ε = 1e-3 and its solution's samples;
* ``PH<k>``, ``PHeps``  the same with P_H = D + C diag(H)⁻¹Cᵀ where the oracle can
               factor P_H (c1 dense LAPACK, c4s SuperLU in the banded row order);
* ``PLeps_var`` the ε = 1e-3 P_L count with b perturbed by 1e-15 relative (seeds 1–4): the rounding spread;
* ``ipm_pl``   the oracle PL-KF IPM's first 15 iterations (μ, residual norms, α, PCG counts);
* ``ipm_pl_var`` the same with r_ν perturbed by 1e-15 (seeds 1–4): the rounding spread of the counts;
* ``ipm_ph``   the oracle PH-KF IPM at ipm_tol 1e-10 (objective, counts, trace) — c4s;
* ``ipm_direct`` c1: the oracle IPM with DIRECT K_F solves (K_F = D − C W Cᵀ formed densely with the
               written-out W = (F⁻¹)₁₁ and Cholesky-factored) at ipm_tol 1e-10 — the optimum's objective,
               which is unique (H SPD), for the GPU PH-KF objective parity; the oracle's own PH-KF IPM
               on c1 would take ~7 h on the host (a 40 000² dense P_H factor and apply per step).

Usage: python scripts/make_goldens.py CFG [stage ...]   (stages: F KF PL PH ipm_pl ipm_ph; default all)
Each stage is saved as it finishes, so a long run can be resumed stage by stage.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import qpgen  # noqa: E402
from oracle import kkt  # noqa: E402
from oracle.fsolve import BlockF, DenseF  # noqa: E402
from oracle.ipm import ipm_solve  # noqa: E402
from oracle.pcg import pcg  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "full")
PH_OK = {"c1": dict(sparse=False, keep=False), "c4s": dict(sparse=True, order="natural")}
IPM_PH = ("c4s",)
VARIANTS = tuple(int(v) for v in os.environ.get("GOLD_VARIANTS", "1,2,3,4").split(","))
KS = (1, 3, 7)


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def fsolver(qp):
    if qp.name == "c1":
        return DenseF(qp.H, qp.A, explicit_w=True)     # K_F products through the written-out (F⁻¹)₁₁
    return BlockF(qp.H, qp.A, qp.x_perm)          # grid configs: the generator's ND order; c3s: SuperLU MMD


def sample(v, idx):
    return dict(s=v[idx].copy(), n2=float(np.linalg.norm(v)), ninf=float(np.max(np.abs(v))))


def save(cfg, stage, payload):
    """Merge `payload` into tests/golden/full/<cfg>.npz (under a file lock: stages may run in parallel)."""
    import fcntl
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, f"{cfg}.npz")
    with open(path + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        old = dict(np.load(path, allow_pickle=False)) if os.path.exists(path) else {}
        for k, v in payload.items():
            old[f"{stage}/{k}"] = np.asarray(v)
        np.savez_compressed(path + ".tmp.npz", **old)
        os.replace(path + ".tmp.npz", path)
    log("saved", cfg, stage, sorted(payload))


def flat(prefix, d):
    return {f"{prefix}_{k}": v for k, v in d.items()}


def main():
    cfg = sys.argv[1]
    stages = sys.argv[2:] or ["F", "KF", "PL", "PH", "ipm_pl", "ipm_pl_var", "ipm_ph", "ipm_direct"]
    qp = qpgen.make(cfg)
    pr = qpgen.probe_inputs(qp)
    log(cfg, "n", qp.n, "m1", qp.m1, "m2", qp.m2)
    t = time.time()
    fs = fsolver(qp)
    t_f = time.time() - t
    log("F factor", round(t_f, 1), "s")
    n = qp.n
    meta = dict(cfg=cfg, t_factor_s=t_f)
    if "F" in stages:
        t = time.time()
        y, z = fs.solve(pr.f[:n], pr.f[n:])
        meta["t_fsolve_s"] = time.time() - t
        save(cfg, "F", sample(np.concatenate([y, z]), pr.idx_F))
    Kop = lambda v: kkt.KF_apply(qp, fs, pr.D, v)  # noqa: E731
    if "KF" in stages:
        t = time.time()
        q = Kop(pr.p)
        meta["t_kf_s"] = time.time() - t
        save(cfg, "KF", sample(q, pr.idx_m2))
    precs = []
    if "PL" in stages:
        precs.append(("PL", kkt.PrecondL(pr.D)))
    if "PH" in stages and cfg in PH_OK:
        t = time.time()
        precs.append(("PH", kkt.PrecondH(qp, pr.D, **PH_OK[cfg])))
        meta["t_ph_factor_s"] = time.time() - t
        log("P_H factor", round(meta["t_ph_factor_s"], 1), "s")
    for name, M in precs:
        pay = {}
        for k in KS:
            x, it, rr, ok, _ = pcg(Kop, pr.b, M, 0.0, k)
            pay.update(flat(f"k{k}", sample(x, pr.idx_m2)))
            log(name, "k", k, "done")
        t = time.time()
        x, it, rr, ok, hist = pcg(Kop, pr.b, M, 1e-3, 2000)
        meta[f"t_{name}_eps_s"] = time.time() - t
        pay.update(flat("eps", sample(x, pr.idx_m2)))
        pay.update(eps_iters=it, eps_relres=rr, eps_converged=int(ok))
        log(name, "eps count", it, "relres", rr)
        save(cfg, name, pay)
    if "PLeps_var" in stages:
        # rounding-level variants of the ε-count solve: b perturbed by 1e-15 relative (seeds 1..4), the same
        # perturbation the IPM variants apply to r_ν — what rounding alone does to the count (reading R12)
        pay = {}
        M = kkt.PrecondL(pr.D)
        for v in VARIANTS:
            bv = pr.b * (1.0 + 1e-15 * np.random.default_rng([v, 0]).standard_normal(len(pr.b)))
            t = time.time()
            x, it, rr, ok, _ = pcg(Kop, bv, M, 1e-3, 2000)
            meta[f"t_PLeps_var{v}_s"] = time.time() - t
            pay[f"eps_iters_v{v}"] = it
            log("PLeps variant", v, "count", it)
        save(cfg, "PLeps_var", pay)
    if "ipm_pl" in stages:
        t = time.time()
        r = ipm_solve(qp, precond="low", max_ipm=15, fs=fs)
        meta["t_ipm_pl_s"] = time.time() - t
        tr = r.trace
        save(cfg, "ipm_pl", dict(k=[d["k"] for d in tr], mu=[d["mu"] for d in tr], rg=[d["rg"] for d in tr],
                                 re=[d["re"] for d in tr], ri=[d["ri"] for d in tr], pcg=[d["pcg"] for d in tr],
                                 alpha=[d["alpha"] for d in tr], eps=[d["eps"] for d in tr]))
    if "ipm_pl_var" in stages:
        # rounding-level variants of the same trajectory (r_ν perturbed by 1e-15 relative): the spread of
        # their PCG counts is what rounding alone does to the counts (DESIGN reading R12)
        pay = {}
        vmax = int(os.environ.get("GOLD_VAR_MAXIPM", "15"))   # the count gate covers counts ≤ 100 only
        for v in VARIANTS:
            t = time.time()
            r = ipm_solve(qp, precond="low", max_ipm=vmax, fs=fs, rnu_perturb=v,
                          rnu_perturb_mag=float(os.environ.get("GOLD_VAR_MAG", "1e-15")))   # reading R12: 1e-15 or 1e-14
            meta[f"t_ipm_pl_var{v}_s"] = time.time() - t
            pay[f"pcg_v{v}"] = [d["pcg"] for d in r.trace]
            pay[f"mu_v{v}"] = [d["mu"] for d in r.trace]
        save(cfg, "ipm_pl_var", pay)
    if "ipm_pl_opv" in stages:
        # operator variants: the same trajectory with the F-solves through another exact route (SuperLU's
        # LU of H in a different column order — other rounding in every K_F product)
        from oracle.fsolve import BlockF as _BF
        import scipy.sparse.linalg as _spla
        pay = {}
        for v, spec in enumerate(("COLAMD", "MMD_ATA"), start=1):
            fs2 = _BF(qp.H, qp.A, None) if qp.x_perm is None else _BF(qp.H, qp.A, qp.x_perm)
            if qp.x_perm is None:
                fs2.lu = _spla.splu(qp.H.tocsc(), permc_spec=spec, diag_pivot_thresh=0.0,
                                    options=dict(SymmetricMode=True))
            t = time.time()
            r = ipm_solve(qp, precond="low", max_ipm=15, fs=fs2, rnu_perturb=10 + v if qp.x_perm is not None else None)
            meta[f"t_ipm_pl_opv{v}_s"] = time.time() - t
            pay[f"pcg_v{10 + v}"] = [d["pcg"] for d in r.trace]
        save(cfg, "ipm_pl_var", pay)
    if "ipm_direct" in stages and cfg == "c1":
        t = time.time()
        r = ipm_solve(qp, precond="low", ipm_tol=1e-10, fs=fs, direct=True)
        meta["t_ipm_direct_s"] = time.time() - t
        tr = r.trace
        save(cfg, "ipm_direct", dict(objective=r.objective, n_ipm=r.n_ipm, converged=int(r.converged),
                                     mu=[d["mu"] for d in tr], alpha=[d["alpha"] for d in tr]))
    if "ipm_ph" in stages and cfg in IPM_PH:
        t = time.time()
        kw = {k: v for k, v in PH_OK[cfg].items()}
        r = ipm_solve(qp, precond="high", ipm_tol=1e-10, fs=fs, ph_opts=kw)
        meta["t_ipm_ph_s"] = time.time() - t
        tr = r.trace
        save(cfg, "ipm_ph", dict(objective=r.objective, n_ipm=r.n_ipm, converged=int(r.converged),
                                 mu=[d["mu"] for d in tr], pcg=[d["pcg"] for d in tr],
                                 alpha=[d["alpha"] for d in tr]))
    mpath = os.path.join(OUT, f"{cfg}.meta.json")
    old = json.load(open(mpath)) if os.path.exists(mpath) else {}
    old.update(meta)
    import platform
    model = next((ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name")),
                 platform.processor())
    old["host"] = dict(cpu=model, nproc=os.cpu_count(), note="the build container, not the GPU box")
    json.dump(old, open(mpath, "w"), indent=1)
    log("done", cfg, meta)


if __name__ == "__main__":
    main()
