#!/usr/bin/env python
"""bench.py — PCG iterations/s of the single-factorization inexact IPM (arXiv 2104.12916) on B200.

Workload (BASELINE.json configs[1], "c1"): random sparse convex QP, n = 20 000,
m1 = 5 000, m2 = 40 000, H = GᵀG + 0.1 I (G 8 nnz/row), A 4 / C 6 nnz/row,
seed 0, fp64, preconditioner P_L (PL-KF).  A *step* is one IPM iteration of
the hot path — residuals (a9), r_ν F-solve (a10), PCG on K_F to ε_k (a1–a6),
recovery F-solve + Δs + step (a11) — on the device-resident iterate.  The
one-time F factorization (a12) is setup, timed and reported separately.

  value      PCG iterations / s over the K timed IPM steps (after W warm-up
             steps), CUDA events on the library's stream, max over ranks.
  e2e        the same metric through the public C ABI from pinned HOST
             buffers: pcg_solve(D_k, r_ν) replayed for the same K steps, with
             the host→device copy of (D_k, r_ν) and device→host copy of Δν in
             the timed region.
  roofline   the F-solve (forward + backward sweep kernels, ~90 % of the step):
             the bytes one F-solve must read in this formulation — L_F outside
             the symmetric root twice, the root's S⁻¹ lower triangle once
              — ÷ the CUDA-event durations inside the timed
             region, against MEASURED_PEAKS.json's HBM copy bandwidth; the
             survey's 2·8·nnz(L_F) per F-solve is reported beside it.
  cpu_baseline  the CPU oracle (oracle/, NumPy/SciPy fp64) on the box's host
             cores: PCG iterations of IPM step 0 on the same c1 problem.

Multi-GPU (torchrun, N > 1), --mode replicas (default): one independent replica
per GPU (the F-solve, ≥ 95 % of the bytes, is replicated, so the
path scales as weak-scaling replicas), value = Σ PCG iterations / max-over-ranks
time.  --mode sharded: ONE IPM with the inequality rows split over the ranks
(NCCL all-reduce of Cᵀp and the PCG reductions, replicated F-solve; strong
scaling), value = PCG iterations / max-over-ranks time.

``--impl reference`` times the CPU oracle as the reference arm (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG iterations/s (fp64, K_F = D - [C 0] F^-1 [C^T; 0], IPM hot path)"
UNIT = "PCG iterations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1")
    ap.add_argument("--precond", default="low", choices=["none", "low", "high"])
    ap.add_argument("--cpu-iters", type=int, default=6, help="oracle PCG iterations per sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ipm-solve", action="store_true",
                    help="skip the full IPM solve timing (BJ metric 'IPM solve time'; c1 PH-KF, rank 0, ~1 min)")
    ap.add_argument("--space", default="nu", choices=["nu", "x"],
                    help="nu: PCG on K_F (the paper's PL-KF, default); x: the x-space twin (projected CG on K_C)")
    ap.add_argument("--mode", default=None, choices=["replicas", "sharded"],
                    help="N > 1: one IPM with the inequality rows sharded over the ranks (default; strong "
                         "scaling, W's chunks split over the ranks on c1) or independent replicas (weak)")
    ap.add_argument("--secondary", default="c2",
                    help="N = 1: also measure this config's PL-KF IPM steps (the sparse-sweep path; '' = off)")
    ap.add_argument("--secondary-steps", type=int, default=4)
    ap.add_argument("--profile-traffic", default=os.path.join(ROOT, "profiles", "traffic.json"))
    return ap.parse_args()


# ----------------------------------------------------------------------------- distributed plumbing
def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def dist_init(world, local):
    import torch
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world > 1


def barrier(use_dist):
    if use_dist:
        import torch.distributed as dist
        dist.barrier()


def allreduce(vals, op, use_dist):
    if not use_dist:
        return vals
    import torch
    import torch.distributed as dist
    dev = "cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return t.cpu().tolist()


def aggregate(pcg_iters, ms, use_dist, shared=False):
    """Whole-job throughput: Σ PCG iterations over ranks ÷ the slowest rank's time (max over ranks).
    shared=True (sharded mode): the ranks run the SAME iterations, so they are counted once."""
    tot, mx = float(pcg_iters), float(ms)
    if use_dist:
        import torch.distributed as dist
        tot = allreduce([tot], dist.ReduceOp.MAX if shared else dist.ReduceOp.SUM, True)[0]
        mx = allreduce([mx], dist.ReduceOp.MAX, True)[0]
    return (tot / (mx / 1e3) if mx > 0 else 0.0), tot, mx


# ----------------------------------------------------------------------------- clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for ln in open(self.path):
            p = [x.strip() for x in ln.split(",")]
            if len(p) >= 9:
                rows.append(p)
        os.unlink(self.path)
        if not rows:
            return None
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------------------- CPU oracle timing
class OracleSampler:
    """The CPU oracle as it stands: F factorization once, then PCG samples on IPM step 0's system."""

    def __init__(self, qp, x_perm=None):
        import numpy as np
        from oracle import kkt
        from oracle.fsolve import make_fsolver
        try:
            from threadpoolctl import threadpool_info
            self.cores = max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
        except Exception:
            self.cores = os.cpu_count()
        t0 = time.perf_counter()
        self.qp = qp
        self.fs = make_fsolver(qp.H, qp.A, x_perm)
        self.t_setup = time.perf_counter() - t0
        x, lam, nu = np.zeros(qp.n), np.zeros(qp.m1), np.ones(qp.m2)
        s = np.abs(qp.d) + 1.0
        res = kkt.residuals(qp, x, lam, nu, s, 0.1)
        self.D = kkt.diag_D(s, nu)
        self.rnu = kkt.r_nu(qp, self.fs, res)

    def sample(self, iters):
        from oracle import kkt
        from oracle.pcg import pcg
        t1 = time.perf_counter()
        _, it, _, _, _ = pcg(lambda p: kkt.KF_apply(self.qp, self.fs, self.D, p), self.rnu, kkt.PrecondL(self.D),
                             0.0, iters)
        return it, time.perf_counter() - t1


def host_info():
    """The host the oracle runs on: CPU model (lscpu / /proc/cpuinfo), cores, BLAS threads."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        model = next((ln.split(":", 1)[1].strip() for ln in out.splitlines() if ln.startswith("Model name")), None)
    except Exception:
        pass
    if model is None:
        try:
            model = next(ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name"))
        except Exception:
            model = "unknown"
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads")} for d in threadpool_info()]
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "blas": blas,
            "superlu": "single-threaded (scipy.sparse.linalg.splu)"}


def cpu_oracle_sample(qp, iters, x_perm=None):
    o = OracleSampler(qp, x_perm)
    it, dt = o.sample(iters)
    return it, dt, o.t_setup, o.cores


def run_reference(args, rank, world):
    """The reference arm: the CPU oracle, timed on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import qpgen
    qp = qpgen.make(args.config)
    o = OracleSampler(qp, qp.x_perm)
    _, t_it = o.sample(1)                         # warm-up; also sizes the per-step sample
    # bounded sample: at most --cpu-iters PCG iterations per step, fewer when K steps of them would take
    # more than about three minutes on this host (the metric, iterations/s, does not depend on the count)
    per_step = max(1, min(args.cpu_iters, int(180.0 / max(args.steps * t_it, 1e-9))))
    its, dts = 0, 0.0
    for k in range(args.steps):
        it, dt = o.sample(per_step)
        its += it
        dts += dt
    value = its / dts if dts > 0 else 0.0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dts / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} PL-KF (CPU oracle: dense block-inverse F-solve, textbook PCG)",
                   "n": qp.n, "m1": qp.m1, "m2": qp.m2},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": o.cores, "kind": "oracle",
                         "sample": f"{args.steps} x {per_step} PCG iterations of IPM step 0 on {args.config} "
                                   f"(oracle F setup {o.t_setup:.1f} s excluded)", "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)



# ----------------------------------------------------------------------------- secondary workload (sparse sweeps)
def measure_secondary(cfg, args, local, stream, peak, peak_src):
    """PL-KF IPM steps on `cfg` (default c2, the largest single-GPU config of BASELINE.json): the path where
    every K_F product runs the sparse supernodal sweeps (a2–a4) instead of c1's explicit W.  Same protocol
    as the headline (W warm-up IPM steps, K timed, CUDA events on the library stream), plus a profiled pass
    for the sweep kernels' durations.  GB/s on SURVEY §8(d)'s algorithmic B_it per PCG iteration."""
    import torch
    import qpgen
    from paper_2104_12916_b200.binding import from_qp
    dev = torch.device("cuda", local)
    qp = qpgen.make(cfg)
    s = from_qp(qp, device=local, stream=stream.cuda_stream)
    t0 = time.perf_counter()
    s.ipm_factor_once("low")
    t_setup = time.perf_counter() - t0
    st = s.stats()
    W, K = 2, args.secondary_steps
    s.ipm_init()
    s.ipm_iterate(W)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    r = s.ipm_iterate(K)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    pcg = int(sum(r["pcg_iters"][W:W + K]))
    steps = max(0, min(K, r["n_ipm"] - W))
    # profiled pass (CUDA events around every launch): sweep kernel durations
    s.ipm_init()
    s.ipm_iterate(W)
    s.profile(True)
    s.profile_read()
    r2 = s.ipm_iterate(K)
    torch.cuda.synchronize(dev)
    prof = s.profile_read()
    s.profile(False)
    pcg2 = int(sum(r2["pcg_iters"][W:W + K]))
    solves = pcg2 + 2 * max(0, min(K, r2["n_ipm"] - W))
    ss = s.structure("sn_start")
    w_root = int(ss[-1] - ss[-2]) if st["sym_enabled"] else 0
    root_bytes = 8.0 * w_root * (w_root + 1) / 2
    forest_bytes = (st["fsolve_bytes_F"] - root_bytes) / 2          # L_F outside the root, per sweep
    (fwd_ms, _), (bwd_ms, _), (root_ms, _) = prof["f_fwd"], prof["f_bwd"], prof["f_root"]
    gbs = lambda b, t: b * solves / (t / 1e3) / 1e9 if t > 0 else None  # noqa: E731
    b_it = st["pcg_bytes_per_iter"]
    value = pcg / (ms / 1e3) if ms > 0 else 0.0
    ach_it = pcg * b_it / (ms / 1e3) / 1e9 if ms > 0 else 0.0
    fsolve_ms = fwd_ms + bwd_ms + root_ms
    traffic = None
    if os.path.exists(args.profile_traffic):
        try:
            traffic = json.load(open(args.profile_traffic)).get(cfg, {}).get("dram_bytes_per_fsolve")
        except Exception:
            traffic = None
    if st.get("pi_enabled"):   # level products: leaf levels / subtrees, then one product kernel per level
        leaf = "k_st16_fwd" if st.get("pi_subtrees") else "k_lvl_fwd x%d" % int(st["lvl_levels_F"])
        kf = "k_pi_init + %s + k_pi_fwd x%d levels" % (leaf, int(st["pi_levels"]))
        kb = "k_pi_bwd x%d levels + %s" % (int(st["pi_levels"]), leaf.replace("fwd", "bwd"))
    else:
        kf, kb = "k_trsv_fwd", "k_trsv_bwd"
    out = {
        "config": cfg, "workload": f"{cfg} PL-KF: one IPM iteration per step (sparse supernodal sweeps for every "
                                   f"K_F product, symmetric-root GEMV, fused PCG step)",
        "sweep_path": "level products" if st.get("pi_enabled") else "task graph",
        "n": qp.n, "m1": qp.m1, "m2": qp.m2, "nnz_LF": st["nnz_LF"], "metric": METRIC, "unit": UNIT,
        "value": value, "ms_per_step": ms / max(1, steps), "steps": steps, "warmup": W, "pcg_iters_timed": pcg,
        "ms_per_pcg_iter": ms / max(1, pcg),
        "achieved_GBps_Bit": ach_it, "frac_Bit": ach_it / peak, "frac_Bit_8TBps": ach_it / 8000.0,
        "B_it_bytes": b_it,
        "B_it_note": "SURVEY 8(d): 16 nnz(L_F) + 24 nnz(C) + 8(15 m2 + 6(n+m1)) per PCG iteration; the timed step "
                     "also holds the IPM step's r_nu / recovery F-solves and residuals, so this is a lower bound",
        "roofline": {"bound": "hbm", "unit": "GB/s", "peak": peak, "peak_source": peak_src,
                     "kernel": f"[{kf}] + k_symroot_gemv + [{kb}] (one F-solve)",
                     "achieved": gbs(st["fsolve_bytes_F"], fsolve_ms),
                     "frac": (gbs(st["fsolve_bytes_F"], fsolve_ms) or 0) / peak,
                     "algorithmic_bytes_per_fsolve": st["fsolve_bytes_F"],
                     "traffic": traffic if st.get("pi_enabled") else None,
                     "traffic_note": "DRAM read + write bytes of one F-solve from the ncu --set full capture in "
                                     "profiles/r2_ncu_c2_levels.txt (level products: the panels Z_J hold L_JJ^-1 as "
                                     "full w x w squares and the relaxed supernodes' explicit zeros (stored 2.23e8 entries against 2.09e8 true), "
                                     "plus row lists and the vector gathers: +24 % over the algorithmic bytes, no re-reads)",
                     "per_kernel": {"forward": {"kernels": kf, "bytes": forest_bytes, "ms": fwd_ms / max(1, solves),
                                                "GBps": gbs(forest_bytes, fwd_ms)},
                                    "k_symroot_gemv": {"bytes": root_bytes, "ms": root_ms / max(1, solves),
                                                       "GBps": gbs(root_bytes, root_ms)},
                                    "backward": {"kernels": kb, "bytes": forest_bytes, "ms": bwd_ms / max(1, solves),
                                                 "GBps": gbs(forest_bytes, bwd_ms)}},
                     "fsolve_share_of_step": fsolve_ms / sum(v[0] for v in prof.values()) if prof else None},
        "setup_s": t_setup, "l2": "no flush: the factor read by every sweep (%.2f GB) exceeds L2" % (
            st["factor_bytes"] / 1e9),
    }
    s.close()
    return out

# ----------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local, use_dist):
    import numpy as np
    import torch
    import qpgen
    from paper_2104_12916_b200.binding import from_qp

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    qp = qpgen.make(args.config)
    stream = torch.cuda.Stream(device=dev)
    sharded = args.mode == "sharded"
    if sharded:
        from paper_2104_12916_b200.binding import nccl_unique_id
        uid = [nccl_unique_id() if rank == 0 else None]
        if use_dist:
            import torch.distributed as dist
            dist.broadcast_object_list(uid, src=0)
        s = from_qp(qp, device=local, stream=stream.cuda_stream, rank=rank, world=world, nccl_uid=uid[0])
    else:
        s = from_qp(qp, device=local, stream=stream.cuda_stream)
    t0 = time.perf_counter()
    s.ipm_factor_once(args.precond)
    t_setup = time.perf_counter() - t0
    st = s.stats()
    W, K = args.warmup, args.steps

    # ---------------------------------------------------------------- device-resident value run
    # (no profiling events inside the timed region: they add ~40 µs per PCG iteration)
    s.ipm_init(space=args.space)
    s.ipm_iterate(W)
    torch.cuda.synchronize(dev)
    clocks = Clocks(local)
    clocks.start()
    l0 = s.launch_count()
    barrier(use_dist)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof_region = bool(os.environ.get("QPB_PROFILE_TIMED"))   # ncu --profile-from-start off: the timed steps only
    if prof_region:
        torch.cuda.cudart().cudaProfilerStart()
    e0.record(stream)
    r = s.ipm_iterate(K)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if prof_region:
        torch.cuda.cudart().cudaProfilerStop()
    barrier(use_dist)
    ck = clocks.stop()
    launches = s.launch_count() - l0
    ms = e0.elapsed_time(e1)
    hist = r["pcg_iters"]
    pcg_timed = int(sum(hist[W:W + K]))
    steps_done = max(0, min(K, r["n_ipm"] - W))

    # ---------------------------------------------------------------- kernel durations (same steps, replayed
    # with CUDA events around every launch on the library stream) for the roofline
    s.ipm_init(space=args.space)
    s.ipm_iterate(W)
    s.profile(True)
    s.profile_read()
    torch.cuda.synchronize(dev)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    r_prof = s.ipm_iterate(K)
    p1.record(stream)
    torch.cuda.synchronize(dev)
    ms_prof = p0.elapsed_time(p1)
    prof = s.profile_read()
    s.profile(False)
    pcg_prof = int(sum(r_prof["pcg_iters"][W:W + K]))

    # ---------------------------------------------------------------- device launch timeline (third pass, the
    # production path with CUDA graphs): per kernel the earliest block start and latest block end by
    # %globaltimer, so launch durations and the idle gaps between dependent launches are both visible
    TLN = ["flat_rhs", "flat_fwd", "root_gemv", "flat_bwd", "pcg_step", "trsv_fwd", "trsv_bwd", "spmv", "lvl_fwd", "lvl_bwd"]
    s.ipm_init(space=args.space)
    s.ipm_iterate(W)
    torch.cuda.synchronize(dev)
    s.debug_timeline(True)
    s.ipm_iterate(1)
    torch.cuda.synchronize(dev)
    tl_ev = s.debug_timeline(False)
    # the first 256 launches per kernel are recorded: keep the events before the first kernel's ring filled
    if tl_ev:
        last = {}
        for k, a, b in tl_ev:
            last[k] = last.get(k, 0) + 1
        full = [k for k, c in last.items() if c >= 256]
        if full:
            cut = min(max(a for k, a, b in tl_ev if k == kk) for kk in full)
            tl_ev = [e for e in tl_ev if e[1] <= cut]
    tl = {}
    if len(tl_ev) > 8:
        span_us = (tl_ev[-1][2] - tl_ev[0][1]) / 1e3
        busy = {}
        for (k0, a0, b0), (k1, a1, b1) in zip(tl_ev, tl_ev[1:]):
            d = busy.setdefault(TLN[k1], [0, 0.0, 0.0])
            d[0] += 1
            d[1] += (b1 - a1) / 1e3
            d[2] += (a1 - b0) / 1e3
        tl = {"span_us": span_us, "note": "first <=256 launches per kernel of one IPM step, graphs on",
              "kernels": {k: {"n": v[0], "avg_us": v[1] / v[0], "avg_gap_before_us": v[2] / v[0],
                              "share_of_span": v[1] / span_us} for k, v in busy.items()}}

    # ---------------------------------------------------------------- e2e replay through the C ABI
    e2e = None
    if not args.no_e2e and args.space == "nu":
        systems = []
        s.ipm_init()
        for k in range(W + K):
            rr = s.ipm_iterate(1)
            if rr["converged"]:
                break
            if k >= W:
                D, rnu, eps = s.ipm_last_system()
                Dp = torch.from_numpy(D).pin_memory()
                rp = torch.from_numpy(rnu).pin_memory()
                systems.append((Dp, rp, eps))
        outp = torch.empty(s.m2, dtype=torch.float64).pin_memory()
        for (Dp, rp, eps) in systems[:1]:   # warm the host path
            s.pcg_solve(Dp.numpy(), rp.numpy(), tol=eps, maxit=2000)
        barrier(use_dist)
        torch.cuda.synchronize(dev)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its = 0
        f0.record(stream)
        for (Dp, rp, eps) in systems:
            x, it, rel, rc = s.pcg_solve(Dp.numpy(), rp.numpy(), tol=eps, maxit=2000)
            outp.numpy()[:] = x
            its += it
        f1.record(stream)
        torch.cuda.synchronize(dev)
        barrier(use_dist)
        ms_e2e = f0.elapsed_time(f1)
        e2e_value, _, _ = aggregate(its, ms_e2e, use_dist, sharded)
        e2e = {"value": e2e_value, "unit": UNIT,
               "h2d_bytes_per_step": 2 * 8 * s.m2, "d2h_bytes_per_step": 8 * s.m2 + 16,
               "steps": len(systems), "pcg_iters": its}

    # ---------------------------------------------------------------- aggregate over ranks
    value, tot_pcg, ms_max = aggregate(pcg_timed, ms, use_dist, sharded)

    # ---------------------------------------------------------------- roofline of the L_F sweeps
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        try:
            peak = float(json.load(open(peaks_path))["hbm_gbs"])
            peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    fwd_ms, fwd_n = prof["f_fwd"]
    bwd_ms, bwd_n = prof["f_bwd"]
    root_ms, root_n = prof["f_root"]
    n_ipm_timed = max(0, min(K, r_prof["n_ipm"] - W))
    # F-solves in the profiled pass: ν-space — one per K_F product + r_ν and recovery per IPM step;
    # x-space — one projection per PCG iteration + the first projection and the particular solution
    real_solves = pcg_prof + 2 * n_ipm_timed
    solve_ms = fwd_ms + root_ms + bwd_ms
    ss = s.structure("sn_start")
    w_root = int(ss[-1] - ss[-2]) if st["sym_enabled"] else 0
    root_bytes = 8.0 * w_root * (w_root + 1) / 2           # lower triangle of S⁻¹, read once per F-solve
    fsolve_bytes = st["fsolve_bytes_F"]
    achieved = real_solves * fsolve_bytes / (solve_ms / 1e3) / 1e9 if solve_ms > 0 else 0.0
    paper_bytes = 2 * 8.0 * st["nnz_LF"]                # L_F values read twice per F-solve
    traffic = None
    if os.path.exists(args.profile_traffic):
        try:
            traffic = json.load(open(args.profile_traffic)).get(args.config, {}).get("dram_bytes_per_fsolve")
        except Exception:
            traffic = None
    flat = bool(st.get("flat_enabled", 0))
    kname = ("F-solve = k_flat_fwd_t + k_symroot_gemv + k_flat_bwd_t (+ k_flat_rhs outside PCG; inside PCG the "
             "fused step prepares C^T p)" if flat else
             "F-solve = k_pi_init + leaf levels / subtrees + k_pi_fwd per level + k_symroot_gemv + k_pi_bwd per "
             "level + leaf levels / subtrees (level products)" if st.get("pi_enabled") else
             "F-solve = (C^T p SpMV +) k_trsv_fwd + k_symroot_gemv + k_trsv_bwd")
    roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved,
                "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "peak_source": peak_src,
                "algorithmic_bytes_per_fsolve": fsolve_bytes,
                "algorithmic_bytes_note": ("8*(w(w+1)/2 of the root's S^-1 + 2*nnz(M) + 2*nnz(L11^-1)), the flattened "
                                           "forest M = L21 L11^-1 read forward and backward" if flat else
                                           "8*(2*nnz(L_F) outside the symmetric root + w(w+1)/2 of the root's "
                                           "S^-1, read once per F-solve)"),
                "paper_bytes_per_fsolve": paper_bytes,
                "paper_formulation_GBps": real_solves * paper_bytes / (solve_ms / 1e3) / 1e9 if solve_ms > 0 else 0,
                "fsolve_ms_avg": solve_ms / max(1, real_solves),
                "fsolve_split_ms": {"forward": fwd_ms / max(1, real_solves), "root_gemv": root_ms / max(1, real_solves),
                                    "backward": bwd_ms / max(1, real_solves)},
                "root_gemv": {"kernel": "k_symroot_gemv", "bytes": root_bytes,
                              "achieved": (root_n * root_bytes / (root_ms / 1e3) / 1e9) if root_ms > 0 else None,
                              "frac": (root_n * root_bytes / (root_ms / 1e3) / 1e9 / peak) if root_ms > 0 else None},
                "flattened_forest": bool(st.get("flat_enabled", 0)),
                "fsolve_share_of_step": solve_ms / ms_prof if ms_prof > 0 else None,
                "timing": "kernel durations from a second pass over the same IPM steps with CUDA events "
                          "around every launch (the headline pass runs without events)",
                "device_timeline": tl}
    if st.get("dense_w_enabled", 0) and prof.get("kf_W", (0, 0))[1] > 0:
        # PCG's K_F products use the explicit x-block W = (F^-1)_11: the dominant kernel is its symmetric GEMV
        w_ms, w_n = prof["kf_W"]
        wb = st["kf_bytes_W"]
        w_ach = w_n * wb / (w_ms / 1e3) / 1e9
        fs = {k: roofline[k] for k in ("kernel", "achieved", "frac", "traffic", "algorithmic_bytes_per_fsolve",
                                       "algorithmic_bytes_note", "fsolve_ms_avg", "fsolve_split_ms", "root_gemv")}
        fs["note"] = "full F-solves (r_nu and recovery, 2 per IPM step) keep the flattened / sweep path"
        n_full = 2 * n_ipm_timed
        if solve_ms > 0 and n_full > 0:
            fs["achieved"] = n_full * fsolve_bytes / (solve_ms / 1e3) / 1e9
            fs["frac"] = fs["achieved"] / peak
            fs["fsolve_ms_avg"] = solve_ms / n_full
            fs["fsolve_split_ms"] = {"forward": fwd_ms / n_full, "root_gemv": root_ms / n_full,
                                     "backward": bwd_ms / n_full}
        roofline.update({
            "kernel": "k_dense_symv: w = W C^T p with W = (F^-1)_11 explicit (every PCG K_F product)",
            "achieved": w_ach, "frac": w_ach / peak, "traffic": None,
            "algorithmic_bytes_per_kf": wb,
            "algorithmic_bytes_note": "8*n(n+1)/2: the lower triangle of W (n x n), read once per K_F product",
            "kf_W_ms_avg": w_ms / w_n, "kf_W_launches": w_n,
            "kf_W_share_of_step": w_ms / ms_prof if ms_prof > 0 else None,
            "dense_w_discrepancy": st.get("dense_w_discrepancy"),
            "fsolve": fs})
        for k in ("algorithmic_bytes_per_fsolve", "fsolve_split_ms", "fsolve_ms_avg", "fsolve_share_of_step"):
            roofline.pop(k, None)
        roofline["paper_formulation_GBps"] = w_n * paper_bytes / (w_ms / 1e3) / 1e9
        roofline["paper_formulation_note"] = ("the paper's 2*8*nnz(L_F) bytes per K_F product over the measured "
                                              "time of one W product (what the F-solve formulation would need)")
        if args.profile_traffic and os.path.exists(args.profile_traffic):
            try:
                roofline["traffic"] = json.load(open(args.profile_traffic)).get(args.config, {}).get(
                    "dram_bytes_per_kf_W")
            except Exception:
                pass
    if tl and "root_gemv" in tl.get("kernels", {}):
        g_us = tl["kernels"]["root_gemv"]["avg_us"]
        gb = st["kf_bytes_W"] if st.get("dense_w_enabled", 0) else root_bytes
        tl["dominant_gemv_achieved_GBps"] = gb / (g_us / 1e6) / 1e9
        tl["dominant_gemv_frac"] = gb / (g_us / 1e6) / 1e9 / peak

    # ---------------------------------------------------------------- CPU baseline (rank 0)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        it, dt, t_or, cores = cpu_oracle_sample(qp, args.cpu_iters, s.structure("perm")[:qp.n]
                                                if qp.n + qp.m1 > 30000 else None)
        cpu = {"value": it / dt if dt > 0 else 0.0, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{it} PCG iterations of IPM step 0 on {args.config} (oracle F setup {t_or:.1f} s excluded)",
               "host": host_info(), "oracle_factor_s": t_or, "oracle_ms_per_pcg_iter": 1e3 * dt / max(1, it)}
        # per-config oracle times measured when the full-size goldens were made (scripts/make_goldens.py,
        # the build container's host, stated in each record) — BASELINE.md §4's factor / PCG / IPM times
        gold = {}
        for cfg in ("c1", "c2", "c3s", "c4s"):
            mp = os.path.join(ROOT, "tests", "golden", "full", f"{cfg}.meta.json")
            if os.path.exists(mp):
                try:
                    gold[cfg] = json.load(open(mp))
                except Exception:
                    pass
        cpu["oracle_times_full_size"] = gold or None

    # ---------------------------------------------------------------- secondary workload (N = 1)
    secondary = None
    if world == 1 and args.secondary and args.secondary != args.config:
        secondary = measure_secondary(args.secondary, args, local, stream, peak, peak_src)

    # ---------------------------------------------------------------- IPM solve time (BJ metric, rank 0)
    # c1 PL-KF does not converge, so the full solve is timed with P_H (PH-KF), the paper's
    # other preconditioner, from the first P_H numeric factor to the 1e-8 KKT stop.
    ipm = None
    if rank == 0 and not args.no_ipm_solve and args.config == "c1" and not sharded:
        del s
        torch.cuda.synchronize(dev)
        sp = from_qp(qp, device=local, stream=stream.cuda_stream)
        t0 = time.perf_counter()
        sp.ipm_factor_once("high")
        t_set = time.perf_counter() - t0
        r_ph = sp.ipm_solve(ipm_tol=1e-8, with_vectors=False)
        stp = sp.stats()
        ipm = {"config": args.config, "precond": "high", "converged": bool(r_ph["converged"]),
               "n_ipm": r_ph["n_ipm"], "pcg_total": r_ph["pcg_total"], "solve_s": r_ph["t_solve_s"],
               "setup_s": t_set, "p_h_refactor_s": stp["t_factor_ph_s"], "objective": r_ph["objective"],
               "note": "full PH-KF IPM solve to the 1e-8 KKT test, setup (orderings, symbolic, factors) separate"}
        sp.close()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_max / max(1, steps_done), "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": (f"{args.config} x-space twin: one IPM iteration per step (residuals, K_C rhs, "
                                f"projected CG with the F factor as constraint preconditioner, step)"
                                if args.space == "x" else
                                f"{args.config} PL-KF: one IPM iteration per step (residuals, r_nu F-solve, "
                                f"PCG to eps_k, recovery, step)" if args.precond == "low" else
                                f"{args.config} {args.precond.upper()}-KF IPM iteration per step"),
                   "space": args.space,
                   "n": qp.n, "m1": qp.m1, "m2": qp.m2, "nnz_LF": st["nnz_LF"], "precond": args.precond,
                   "ipm_steps_timed": steps_done, "pcg_iters_timed": pcg_timed,
                   "l2": ("no flush: every K_F product reads W (%.2f GB) and every full F-solve the factor (%.2f GB), both exceed L2" % (st["kf_bytes_W"] / 1e9, st["factor_bytes"] / 1e9)) if st.get("dense_w_enabled", 0) else ("no flush: the factor read every sweep (%.2f GB) exceeds L2" % (st["factor_bytes"] / 1e9)),
                   "parallelism": (f"sharded inequality rows x{world} (NCCL all-reduce; " + ("W chunks split over ranks" if st.get("dense_w_enabled", 0) else "replicated F-solve") + ")"
                                   if sharded else (f"replicas x{world}" if world > 1 else "single GPU"))},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": ck,
        "ipm_solve": ipm, "secondary": secondary,
        "setup_s": {"symbolic": st["t_symbolic_s"], "factor": st["t_factor_s"], "factor_once_total": t_setup},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def spawn(args):
    """`bench.py --gpus N` without a torchrun environment: re-run this command under torchrun with N ranks
    (one process per GPU, rendezvous on 127.0.0.1) and pass its output through."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    rank, world, local = dist_info()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    if args.mode is None:
        args.mode = "sharded" if world > 1 else "replicas"
    use_dist = dist_init(world, local)
    run_ours(args, rank, world, local, use_dist)
    if use_dist:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
