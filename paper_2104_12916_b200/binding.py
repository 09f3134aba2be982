"""ctypes binding of include/qp_b200.h (argument marshalling only).

Names mirror the C ABI: ``qp_setup`` → ``QPSolver(...)``, ``ipm_factor_once``
→ ``QPSolver.ipm_factor_once``, ``pcg_solve``, ``ipm_solve``, ``f_solve``,
``kf_apply``, ``structure``, ``stats``.  Vectors may be NumPy arrays (host
path: the library copies in/out) or, with ``vectors_on_device=True``, CUDA
torch tensors whose ``data_ptr()`` is passed straight through.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from typing import Optional

import numpy as np

from . import build as _build

HERE = os.path.dirname(os.path.abspath(__file__))
HEADER = os.path.join(os.path.dirname(HERE), "include", "qp_b200.h")

PREC = {"none": 0, "low": 1, "high": 2}
STATUS = {0: "QP_OK", 1: "QP_MAXIT", -1: "QP_EINVAL", -2: "QP_ENOTSPD", -3: "QP_EBREAKDOWN",
          -4: "QP_ENOMEM", -5: "QP_ECUDA", -6: "QP_ENCCL", -7: "QP_ESTATE"}
STRUCTURES = {"perm": 0, "parent": 1, "colcount": 2, "sn_start": 3, "sn_parent": 4, "sn_level": 5,
              "sn_rowptr": 6, "sn_rows": 7, "row_level": 8, "trailing_from": 9}


class QPError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class _CSR(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("indptr", C.c_void_p),
                ("indices", C.c_void_p), ("values", C.c_void_p)]


# int (*)(void* user, double* buf, int64_t count, int32_t op, void* stream)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p)
# int (*)(void* user, const double* to_prev, int64_t, const double* to_next, int64_t,
#         double* from_prev, int64_t, double* from_next, int64_t, void* stream)
HALO_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                      C.c_void_p, C.c_int64, C.c_void_p)


class _SetupOpts(C.Structure):
    _fields_ = [("device", C.c_int), ("stream", C.c_void_p), ("rank", C.c_int), ("world", C.c_int),
                ("nccl_uid", C.c_void_p), ("x_perm", C.c_void_p), ("vectors_on_device", C.c_int),
                ("workspace_limit_bytes", C.c_int64), ("allreduce", ALLREDUCE_FN),
                ("allreduce_user", C.c_void_p), ("halo", HALO_FN), ("halo_user", C.c_void_p)]


class _IpmOpts(C.Structure):
    _fields_ = [("ipm_tol", C.c_double), ("pcg_tol", C.c_double), ("sigma", C.c_double),
                ("tau", C.c_double), ("max_ipm", C.c_int32), ("pcg_maxit", C.c_int32),
                ("pcg_forcing", C.c_int32), ("space", C.c_int32)]


class _IpmResult(C.Structure):
    _fields_ = [("x", C.c_void_p), ("lam", C.c_void_p), ("nu", C.c_void_p), ("s", C.c_void_p),
                ("objective", C.c_double), ("n_ipm", C.c_int32), ("pcg_iters", C.c_void_p),
                ("status", C.c_int32), ("pcg_total", C.c_int32), ("t_setup_s", C.c_double),
                ("t_solve_s", C.c_double), ("mu", C.c_double), ("rg_inf", C.c_double),
                ("re_inf", C.c_double), ("ri_inf", C.c_double), ("alpha", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("n", "m1", "m2", "nnz_H", "nnz_A", "nnz_C", "nnz_LF",
                                         "n_supernodes_F", "n_blocks_F", "n_levels_F", "row_levels_F",
                                         "nnz_LPH", "n_supernodes_PH", "workspace_bytes", "factor_bytes",
                                         "nnz_LF_stored")] + \
               [(k, C.c_double) for k in ("c_fact_F", "c_fact_PH", "t_symbolic_s", "t_factor_s",
                                          "t_factor_ph_s", "pcg_bytes_per_iter", "pcg_flops_per_iter",
                                          "sweep_bytes_F", "fsolve_bytes_F", "sym_discrepancy", "sym_enabled",
                                          "flat_discrepancy", "flat_enabled", "flat_nnz_M", "dense_w_enabled",
                                          "dense_w_discrepancy", "kf_bytes_W", "dense_finv_enabled",
                                          "dense_finv_discrepancy", "lvl_levels_F", "lvl_levels_PH",
                                          "lvl_supernodes_F", "lvl_supernodes_PH", "pi_enabled", "pi_discrepancy",
                                          "pi_levels", "pi_subtrees", "pi_fsolve_ms", "sweep_fsolve_ms")]


_LIB = None


def header_functions():
    """Function names declared in include/qp_b200.h."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+(\w+)\s*\(", txt, flags=re.M)))


def load_library(build: bool = True):
    """Load libqp_b200.so (building it first if sources are newer)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = _build.build() if build else _build.LIB
    if not os.path.exists(path):
        raise OSError(f"{path} not built — run paper_2104_12916_b200/build.py (no CPU fallback exists)")
    lib = C.CDLL(path)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    lib.qp_setup.argtypes = [C.POINTER(vp), C.POINTER(_CSR), C.POINTER(_CSR), C.POINTER(_CSR), vp, vp, vp,
                             C.POINTER(_SetupOpts)]
    lib.ipm_factor_once.argtypes = [vp, vp, C.c_int]
    lib.pcg_solve.argtypes = [vp, vp, vp, dbl, i32, vp, C.POINTER(i32), C.POINTER(dbl)]
    lib.pcg_solve_x.argtypes = [vp, vp, vp, vp, dbl, i32, vp, vp, C.POINTER(i32), C.POINTER(dbl)]
    lib.ipm_solve.argtypes = [vp, C.POINTER(_IpmOpts), C.POINTER(_IpmResult)]
    lib.qp_ipm_init.argtypes = [vp, C.POINTER(_IpmOpts)]
    lib.qp_ipm_iterate.argtypes = [vp, i32, C.POINTER(_IpmResult), C.POINTER(i32)]
    lib.qp_f_solve.argtypes = [vp, vp, vp]
    lib.qp_kf_apply.argtypes = [vp, vp, vp, vp]
    lib.qp_operator_apply.argtypes = [vp, vp, vp, vp]
    lib.qp_operator_halo_plan.argtypes = [vp, vp]
    lib.qp_operator_apply_halo.argtypes = [vp, vp, vp, vp]
    lib.qp_analyse.argtypes = [C.POINTER(vp), C.POINTER(_CSR), C.POINTER(_CSR), vp]
    lib.qp_partition_rows.argtypes = [vp, i64, i32, vp]
    lib.qp_get_partition.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
    lib.qp_nccl_unique_id.argtypes = [vp]
    lib.qp_get_structure.argtypes = [vp, i32, vp, C.POINTER(i64)]
    lib.qp_get_stats.argtypes = [vp, C.POINTER(_Stats)]
    lib.qp_profile.argtypes = [vp, i32]
    lib.qp_profile_read.argtypes = [vp, vp, vp]
    lib.qp_debug_sweep_profile.argtypes = [vp, i32, vp]
    lib.qp_debug_sweep_trace.argtypes = [vp, i32, vp, i64]
    lib.qp_debug_sweep_trace.restype = i64
    lib.qp_debug_timeline.argtypes = [vp, i32, vp, i64]
    lib.qp_debug_timeline.restype = i64
    lib.qp_ipm_last_system.argtypes = [vp, vp, vp, C.POINTER(dbl)]
    lib.qp_launch_count.argtypes = [vp]
    lib.qp_launch_count.restype = i64
    lib.qp_last_error.argtypes = [vp]
    lib.qp_last_error.restype = C.c_char_p
    lib.qp_free.argtypes = [vp]
    lib.qp_free.restype = None
    _LIB = lib
    return lib


def exported_symbols():
    """Dynamic symbols exported by the built library (reads the ELF via nm -D)."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True, text=True).stdout
    return sorted({ln.split()[-1] for ln in out.splitlines() if " T " in ln})


def partition_rows(indptr, m2, world):
    """qp_partition_rows: contiguous nnz-balanced split of m2 rows over `world` ranks (host only)."""
    lib = load_library()
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    out = np.zeros(world + 1, dtype=np.int64)
    rc = lib.qp_partition_rows(ip.ctypes.data, int(m2), int(world), out.ctypes.data)
    if rc != 0:
        raise QPError(rc, "qp_partition_rows")
    return out


def nccl_unique_id():
    """qp_nccl_unique_id: 128 bytes for QPSolver(nccl_uid=...) (rank 0 creates, caller broadcasts)."""
    buf = C.create_string_buffer(128)
    rc = load_library().qp_nccl_unique_id(buf)
    if rc != 0:
        raise QPError(rc, "qp_nccl_unique_id (NCCL unavailable)")
    return buf.raw


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class QPSolver:
    """One qp_ctx: ``qp_setup`` on construction, ``qp_free`` on close."""

    def __init__(self, H, A, Cm, g, b, d, x_perm=None, device=0, stream=None, vectors_on_device=False,
                 workspace_limit_bytes=0, rank=0, world=1, nccl_uid=None, allreduce=None, halo=None):
        """rank / world / nccl_uid / allreduce select the sharded mode (qp_b200.h): every rank passes
        the same global problem; m2-length vectors are then this rank's row slice
        (``self.row0 : self.row0 + self.m2`` of ``self.m2_global``).  ``allreduce`` is a Python
        callable ``f(buf_ptr, count, op, stream_ptr) -> int`` used instead of NCCL; ``halo`` a callable
        ``f(to_prev, n, to_next, n, from_prev, n, from_next, n, stream_ptr) -> int`` (qp_halo_fn)."""
        import scipy.sparse as sp
        self.lib = load_library()
        self.vectors_on_device = bool(vectors_on_device)
        self._keep = []

        def csr(M):
            M = sp.csr_matrix(M)
            ip = np.ascontiguousarray(M.indptr, dtype=np.int64)
            ix = np.ascontiguousarray(M.indices, dtype=np.int32)
            vv = np.ascontiguousarray(M.data, dtype=np.float64)
            self._keep += [ip, ix, vv]
            return _CSR(M.shape[0], M.shape[1], ip.ctypes.data, ix.ctypes.data, vv.ctypes.data)

        self.n, self.m1, self.m2 = H.shape[0], A.shape[0], Cm.shape[0]
        cH, cA, cC = csr(H), csr(A), csr(Cm)
        g, b, d = _f64(g), _f64(b), _f64(d)
        opts = _SetupOpts()
        opts.device = device
        opts.stream = stream
        opts.rank = rank
        opts.world = world
        if nccl_uid is not None:
            uid = C.create_string_buffer(bytes(nccl_uid), 128)
            self._keep.append(uid)
            opts.nccl_uid = C.cast(uid, C.c_void_p)
        if allreduce is not None:
            self._ar = ALLREDUCE_FN(lambda user, buf, cnt, op, st: int(allreduce(buf, cnt, op, st)))
            opts.allreduce = self._ar
        if halo is not None:
            self._halo = HALO_FN(lambda user, a, na, b, nb, c_, nc, d_, nd, st: int(halo(a, na, b, nb, c_, nc, d_, nd, st)))
            opts.halo = self._halo
        opts.vectors_on_device = 1 if vectors_on_device else 0
        opts.workspace_limit_bytes = workspace_limit_bytes
        if x_perm is not None:
            xp = np.ascontiguousarray(x_perm, dtype=np.int64)
            self._keep.append(xp)
            opts.x_perm = xp.ctypes.data
        self.ctx = C.c_void_p()
        rc = self.lib.qp_setup(C.byref(self.ctx), C.byref(cH), C.byref(cA), C.byref(cC), g.ctypes.data,
                               b.ctypes.data if b.size else g.ctypes.data, d.ctypes.data, C.byref(opts))
        self._keep = []
        self._check(rc)
        r0, r1, mg = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.qp_get_partition(self.ctx, C.byref(r0), C.byref(r1), C.byref(mg)))
        self.row0, self.m2, self.m2_global = int(r0.value), int(r1.value - r0.value), int(mg.value)

    # -------------------------------------------------------------- plumbing
    def _check(self, rc, ok=(0,)):
        if rc not in ok:
            msg = self.lib.qp_last_error(self.ctx).decode() if self.ctx else ""
            raise QPError(rc, msg)
        return rc

    def _ptr(self, v, n, out=False):
        if self.vectors_on_device:
            return v.data_ptr(), v
        a = np.zeros(n) if out else _f64(v)
        assert a.size == n, (a.size, n)
        return a.ctypes.data, a

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.qp_free(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- ABI
    def ipm_factor_once(self, precond="low", D0=None):
        p = None
        if D0 is not None:
            p, keep = self._ptr(D0, self.m2)
        return self._check(self.lib.ipm_factor_once(self.ctx, p, PREC[precond]))

    def pcg_solve(self, D, rhs, tol=1e-3, maxit=2000, out=None):
        pD, kD = self._ptr(D, self.m2)
        pb, kb = self._ptr(rhs, self.m2)
        if self.vectors_on_device:
            assert out is not None
            po, ko = out.data_ptr(), out
        else:
            ko = np.zeros(self.m2)
            po = ko.ctypes.data
        it = C.c_int32()
        rr = C.c_double()
        rc = self._check(self.lib.pcg_solve(self.ctx, pD, pb, float(tol), int(maxit), po, C.byref(it),
                                            C.byref(rr)), ok=(0, 1))
        return ko, int(it.value), float(rr.value), rc

    def _opts(self, ipm_tol=1e-8, pcg_tol=1e-3, sigma=0.1, tau=0.995, max_ipm=100, pcg_maxit=2000,
              pcg_forcing=True, space="nu"):
        return _IpmOpts(ipm_tol, pcg_tol, sigma, tau, max_ipm, pcg_maxit, 1 if pcg_forcing else 0,
                        {"nu": 0, "x": 1}[space])

    def pcg_solve_x(self, D, f, e, tol=1e-3, maxit=2000):
        """x-space twin: G Δx − AᵀΔλ = f, AΔx = e, G = H + CᵀD⁻¹C (projected CG).
        Returns (Δx, Δλ, iters, relres, status)."""
        pD, kD = self._ptr(D, self.m2)
        pf, kf = self._ptr(f, self.n)
        pe, ke = self._ptr(e, self.m1) if self.m1 else (None, None)
        if self.vectors_on_device:
            raise NotImplementedError("device vectors: call the C ABI directly")
        dx, dl = np.zeros(self.n), np.zeros(max(self.m1, 1))
        it = C.c_int32()
        rr = C.c_double()
        rc = self._check(self.lib.pcg_solve_x(self.ctx, pD, pf, pe, float(tol), int(maxit), dx.ctypes.data,
                                              dl.ctypes.data, C.byref(it), C.byref(rr)), ok=(0, 1))
        return dx, dl[:self.m1], int(it.value), float(rr.value), rc

    def _result(self, with_vectors=True, max_ipm=100):
        r = _IpmResult()
        bufs = {}
        if with_vectors and not self.vectors_on_device:
            for k, n in (("x", self.n), ("lam", self.m1), ("nu", self.m2), ("s", self.m2)):
                bufs[k] = np.zeros(n)
                setattr(r, k, bufs[k].ctypes.data)
        it = np.zeros(max(1, max_ipm), dtype=np.int32)
        r.pcg_iters = it.ctypes.data
        return r, bufs, it

    @staticmethod
    def _pack(r, bufs, it):
        out = dict(objective=r.objective, n_ipm=r.n_ipm, status=r.status, pcg_total=r.pcg_total,
                   t_setup_s=r.t_setup_s, t_solve_s=r.t_solve_s, mu=r.mu, rg_inf=r.rg_inf,
                   re_inf=r.re_inf, ri_inf=r.ri_inf, alpha=r.alpha,
                   pcg_iters=it[:min(r.n_ipm, len(it))].tolist())
        out.update(bufs)
        return out

    def ipm_solve(self, with_vectors=True, **kw):
        o = self._opts(**kw)
        r, bufs, it = self._result(with_vectors, o.max_ipm)
        rc = self._check(self.lib.ipm_solve(self.ctx, C.byref(o), C.byref(r)), ok=(0, 1))
        d = self._pack(r, bufs, it)
        d["converged"] = rc == 0
        return d

    def ipm_init(self, **kw):
        self._iter_opts = self._opts(**kw)
        return self._check(self.lib.qp_ipm_init(self.ctx, C.byref(self._iter_opts)))

    def ipm_iterate(self, nsteps, with_vectors=False):
        r, bufs, it = self._result(with_vectors, self._iter_opts.max_ipm)
        done = C.c_int32()
        self._check(self.lib.qp_ipm_iterate(self.ctx, int(nsteps), C.byref(r), C.byref(done)))
        d = self._pack(r, bufs, it)
        d["converged"] = bool(done.value)
        return d

    def f_solve(self, rhs):
        N = self.n + self.m1
        p, k = self._ptr(rhs, N)
        out = np.zeros(N)
        self._check(self.lib.qp_f_solve(self.ctx, p, out.ctypes.data))
        return out[:self.n], out[self.n:]

    def operator_apply(self, D, p, out=None):
        """q = H p + Cᵀ(D⁻¹∘(C p)) (qp_operator_apply; no factorization needed)."""
        pD, kD = self._ptr(D, self.m2)
        pp, kp = self._ptr(p, self.n)
        if self.vectors_on_device:
            assert out is not None
            self._check(self.lib.qp_operator_apply(self.ctx, pD, pp, out.data_ptr()))
            return out
        q = np.zeros(self.n)
        self._check(self.lib.qp_operator_apply(self.ctx, pD, pp, q.ctypes.data))
        return q

    def operator_halo_plan(self):
        """qp_operator_halo_plan (collective): dict(enabled, own=(lo, hi), p_window, q_window, sent_doubles)."""
        info = np.zeros(8, dtype=np.int64)
        self._check(self.lib.qp_operator_halo_plan(self.ctx, info.ctypes.data))
        return dict(enabled=bool(info[0]), own=(int(info[1]), int(info[2])), p_window=(int(info[3]), int(info[4])),
                    q_window=(int(info[5]), int(info[6])), sent_doubles=int(info[7]))

    def operator_apply_halo(self, D, p):
        """qp_operator_apply_halo with host vectors: p full length with this rank's owned entries valid;
        returns q (full length; valid on the owned range) and p with the rank's window filled in."""
        assert not self.vectors_on_device
        D = _f64(D)
        p = np.array(p, dtype=np.float64, copy=True)
        q = np.zeros(self.n)
        self._check(self.lib.qp_operator_apply_halo(self.ctx, D.ctypes.data, p.ctypes.data, q.ctypes.data))
        return q, p

    def kf_apply(self, D, p):
        pD, kD = self._ptr(D, self.m2)
        pp, kp = self._ptr(p, self.m2)
        out = np.zeros(self.m2)
        self._check(self.lib.qp_kf_apply(self.ctx, pD, pp, out.ctypes.data))
        return out

    def structure(self, name, ph=False):
        which = STRUCTURES[name] + (10 if ph else 0)
        n = C.c_int64(0)
        self._check(self.lib.qp_get_structure(self.ctx, which, None, C.byref(n)))
        buf = np.zeros(n.value, dtype=np.int64)
        self._check(self.lib.qp_get_structure(self.ctx, which, buf.ctypes.data, C.byref(n)))
        return buf

    def debug_sweep_profile(self, enable):
        out = np.zeros(80, dtype=np.int64)
        self._check(self.lib.qp_debug_sweep_profile(self.ctx, 1 if enable else 0, out.ctypes.data))
        return out.reshape(2, 8, 5)

    def debug_sweep_trace(self, sweep, cap=1 << 20):
        out = np.zeros((cap, 6), dtype=np.int64)
        n = int(self.lib.qp_debug_sweep_trace(self.ctx, int(sweep), out.ctypes.data, cap))
        if n < 0:
            self._check(n)
        return out[:n]

    def debug_timeline(self, enable):
        """enable=True: start recording; enable=False: stop and return a list of (kernel, start_ns, end_ns)
        per recorded launch (the first 256 per kernel), sorted by start (kernels: 0 flat rhs … 7 SpMV, 8/9 leaf-phase levels fwd/bwd,
        include/qp_b200.h)."""
        K, R = 10, 256
        W = 2 * K + 2 * K * R
        if enable:
            rc = int(self.lib.qp_debug_timeline(self.ctx, 1, None, 0))
            if rc < 0:
                self._check(rc)
            return None
        out = np.zeros(W, dtype=np.uint64)
        rc = int(self.lib.qp_debug_timeline(self.ctx, 0, out.ctypes.data, W))
        if rc < 0:
            self._check(rc)
        st = out[2 * K:2 * K + K * R].reshape(K, R)
        en = out[2 * K + K * R:].reshape(K, R)
        ev = [(k, int(st[k, s]), int(en[k, s])) for k in range(K) for s in range(R)
              if st[k, s] != np.uint64(2**64 - 1) and en[k, s] != 0]
        return sorted(ev, key=lambda e: e[1])

    def ipm_last_system(self):
        D, r = np.zeros(self.m2), np.zeros(self.m2)
        eps = C.c_double()
        self._check(self.lib.qp_ipm_last_system(self.ctx, D.ctypes.data, r.ctypes.data, C.byref(eps)))
        return D, r, float(eps.value)

    def launch_count(self):
        return int(self.lib.qp_launch_count(self.ctx))

    def stats(self):
        s = _Stats()
        self._check(self.lib.qp_get_stats(self.ctx, C.byref(s)))
        return {k: getattr(s, k) for k, _ in _Stats._fields_}

    def profile(self, enable=True):
        self._check(self.lib.qp_profile(self.ctx, 1 if enable else 0))

    def profile_read(self):
        ms = np.zeros(10)
        cnt = np.zeros(10, dtype=np.int64)
        self._check(self.lib.qp_profile_read(self.ctx, ms.ctypes.data, cnt.ctypes.data))
        names = ["f_fwd", "f_bwd", "kf_q", "pcg_vec", "ph_sweeps", "ph_refactor", "ipm_rhs", "other", "f_root",
                 "kf_W"]
        return {nm: (float(m), int(c)) for nm, m, c in zip(names, ms, cnt)}


class Analysis(QPSolver):
    """Host-only symbolic analysis context (``qp_analyse``): structures and stats, no GPU."""

    def __init__(self, H, A, x_perm=None):
        import scipy.sparse as sp
        self.lib = load_library()
        self.vectors_on_device = False
        keep = []

        def csr(M):
            M = sp.csr_matrix(M)
            ip = np.ascontiguousarray(M.indptr, dtype=np.int64)
            ix = np.ascontiguousarray(M.indices, dtype=np.int32)
            vv = np.ascontiguousarray(M.data, dtype=np.float64)
            keep.extend([ip, ix, vv])
            return _CSR(M.shape[0], M.shape[1], ip.ctypes.data, ix.ctypes.data, vv.ctypes.data)

        self.n, self.m1, self.m2 = H.shape[0], A.shape[0], 0
        cH, cA = csr(H), csr(A)
        xp = None
        if x_perm is not None:
            xp = np.ascontiguousarray(x_perm, dtype=np.int64)
        self.ctx = C.c_void_p()
        rc = self.lib.qp_analyse(C.byref(self.ctx), C.byref(cH), C.byref(cA),
                                 xp.ctypes.data if xp is not None else None)
        self._check(rc)


def from_qp(qp, **kw):
    """QPSolver from a ``qpgen.QP`` instance (uses its x_perm when present)."""
    xp = kw.pop("x_perm", qp.x_perm)
    return QPSolver(qp.H, qp.A, qp.C, qp.g, qp.b, qp.d, x_perm=xp, **kw)
