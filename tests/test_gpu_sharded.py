"""Sharded ν-row mode on one GPU (qp_b200.h "Sharded mode").

The round's GPU budget is one device, so two ranks run as two threads of this process, each
with its own qp_ctx (own stream, own replicated F factor) on cuda:0, and the collective is the
C ABI's qp_allreduce_fn implemented here on the host: every call synchronises the rank's
stream, copies the buffer out, sums in rank order (bit-identical on both ranks) and copies it
back.  No kernel of one rank ever waits on the other's.  The NCCL path itself is exercised
with world = 1 (a one-rank communicator: all-reduce is the identity, but every collective of
the sharded code path is issued through NCCL).

Checks: the concatenated sharded PCG solution equals the oracle's (1e-8 relative, reading
R16 at fixed iterations) and the unsharded library's; the sharded IPM reaches the oracle's
objective (1e-8 relative) with replicated x identical on both ranks and the KKT conditions.
"""
import threading

import numpy as np
import pytest

import qpgen
from oracle.fsolve import make_fsolver
from oracle.kkt import KF_apply
from oracle.pcg import pcg

pytestmark = pytest.mark.gpu


class ThreadComm:
    """qp_allreduce_fn for `world` ranks living in threads of one process."""

    def __init__(self, world):
        self.world = world
        self.slots = [None] * world
        self.bar = threading.Barrier(world)

    def fn(self, rank):
        from cuda.bindings import runtime as rt

        def allreduce(buf, count, op, stream):
            (err,) = rt.cudaStreamSynchronize(stream)
            assert int(err) == 0, err
            host = np.empty(count)
            (err,) = rt.cudaMemcpy(host.ctypes.data, buf, count * 8, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
            assert int(err) == 0, err
            self.slots[rank] = host
            self.bar.wait()
            res = self.slots[0].copy()
            for r in range(1, self.world):
                res = res + self.slots[r] if op == 0 else (np.maximum(res, self.slots[r]) if op == 1
                                                           else np.minimum(res, self.slots[r]))
            self.bar.wait()
            # on the caller's stream and complete before returning (a plain cudaMemcpy from pageable memory may
            # return before its DMA lands and is not ordered with the library's non-blocking stream)
            (err,) = rt.cudaMemcpyAsync(buf, res.ctypes.data, count * 8, rt.cudaMemcpyKind.cudaMemcpyHostToDevice,
                                        stream)
            assert int(err) == 0, err
            (err,) = rt.cudaStreamSynchronize(stream)
            return int(err)
        return allreduce

    def halo(self, rank):
        """qp_halo_fn for threads: every rank posts what it sends, then reads what its neighbours posted."""
        from cuda.bindings import runtime as rt

        def d2h(ptr, n):
            host = np.empty(n)
            if n:
                (err,) = rt.cudaMemcpy(host.ctypes.data, ptr, n * 8, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
                assert int(err) == 0, err
            return host

        def exchange(to_prev, n_tp, to_next, n_tn, from_prev, n_fp, from_next, n_fn, stream):
            (err,) = rt.cudaStreamSynchronize(stream)
            assert int(err) == 0, err
            self.slots[rank] = (d2h(to_prev, n_tp), d2h(to_next, n_tn))
            self.bar.wait()
            if n_fp:
                src = self.slots[rank - 1][1]
                assert len(src) == n_fp
                (err,) = rt.cudaMemcpyAsync(from_prev, src.ctypes.data, n_fp * 8,
                                            rt.cudaMemcpyKind.cudaMemcpyHostToDevice, stream)
                assert int(err) == 0, err
            if n_fn:
                src = self.slots[rank + 1][0]
                assert len(src) == n_fn
                (err,) = rt.cudaMemcpyAsync(from_next, src.ctypes.data, n_fn * 8,
                                            rt.cudaMemcpyKind.cudaMemcpyHostToDevice, stream)
                assert int(err) == 0, err
            (err,) = rt.cudaStreamSynchronize(stream)
            assert int(err) == 0, err
            self.bar.wait()
            return 0
        return exchange


def run_ranks(world, body):
    """body(rank, comm) in `world` threads; returns the per-rank results (re-raises errors)."""
    comm = ThreadComm(world)
    out, errs = [None] * world, []

    def run(r):
        try:
            out[r] = body(r, comm)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            comm.bar.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    if errs:
        raise errs[0]
    return out


def _solver(qp, rank, world, comm):
    from paper_2104_12916_b200.binding import from_qp
    s = from_qp(qp, rank=rank, world=world, allreduce=comm.fn(rank))
    s.ipm_factor_once("low")
    return s


@pytest.mark.parametrize("world,name", [(2, "c0"), (3, "c0"), (4, "ragged")])
def test_sharded_pcg_matches_oracle(world, name):
    qp = qpgen.make("c0") if name == "c0" else qpgen.scaled_random_qp(700, 130, 900, seed=3)
    rng = np.random.default_rng(11)
    D = rng.uniform(0.5, 2.0, qp.m2)
    b = rng.standard_normal(qp.m2)
    fs = make_fsolver(qp.H, qp.A)
    for tol, maxit in ((0.0, 12), (1e-12, 300)):
        def body(rank, comm):
            s = _solver(qp, rank, world, comm)
            sl = slice(s.row0, s.row0 + s.m2)
            x, it, rr, rc = s.pcg_solve(D[sl], b[sl], tol=tol, maxit=maxit)
            s.close()
            return s.row0, x, it, rr
        res = run_ranks(world, body)
        assert [r[0] for r in res] == sorted(r[0] for r in res) and res[0][0] == 0
        xs = np.concatenate([r[1] for r in res])
        its = {r[2] for r in res}
        assert len(its) == 1                                   # every rank took the same decisions
        xo, ito, _, _, _ = pcg(lambda p: KF_apply(qp, fs, D, p), b, lambda r: r / D, tol, maxit)
        if tol == 0.0:
            assert its == {maxit} and ito == maxit
        else:
            assert abs(its.pop() - ito) <= 2
        assert np.linalg.norm(xs - xo) <= 1e-8 * np.linalg.norm(xo)


def test_sharded_ipm_matches_oracle():
    from oracle.ipm import ipm_solve as oracle_ipm
    qp = qpgen.make("c0")
    ref = oracle_ipm(qp, precond="low", ipm_tol=1e-10)

    def body(rank, comm):
        s = _solver(qp, rank, 2, comm)
        r = s.ipm_solve(ipm_tol=1e-10, max_ipm=100)
        r["row0"] = s.row0
        s.close()
        return r

    res = run_ranks(2, body)
    for r in res:
        assert r["converged"]
        assert abs(r["objective"] - ref.objective) <= 1e-8 * max(1.0, abs(ref.objective))
    assert res[0]["n_ipm"] == res[1]["n_ipm"] and res[0]["pcg_iters"] == res[1]["pcg_iters"]
    assert np.abs(res[0]["x"] - res[1]["x"]).max() <= 1e-12 * (1 + np.abs(res[0]["x"]).max())
    x, lam = res[0]["x"], res[0]["lam"]
    nu = np.concatenate([r["nu"] for r in res])
    s_ = np.concatenate([r["s"] for r in res])
    assert s_.min() > 0 and nu.min() > 0
    tol = 1e-8
    assert np.abs(qp.H @ x + qp.g - qp.A.T @ lam - qp.C.T @ nu).max() <= tol * (1 + np.abs(qp.g).max())
    assert np.abs(qp.A @ x - qp.b).max() <= tol * (1 + np.abs(qp.b).max())
    assert np.abs(qp.C @ x - s_ - qp.d).max() <= tol * (1 + np.abs(qp.d).max())


def test_sharded_rejects_ph_and_bad_rank():
    from paper_2104_12916_b200.binding import QPError, from_qp
    qp = qpgen.make("c0")
    with pytest.raises(QPError):
        from_qp(qp, rank=2, world=2, allreduce=lambda *a: 0)

    def body(rank, comm):
        s = from_qp(qp, rank=rank, world=2, allreduce=comm.fn(rank))
        with pytest.raises(QPError):
            s.ipm_factor_once("high")
        s.close()
        return True

    assert all(run_ranks(2, body))


def test_nccl_world1_matches_unsharded():
    """world = 1 through a real one-rank NCCL communicator: identical to the unsharded path up
    to reduction order."""
    from paper_2104_12916_b200.binding import from_qp, nccl_unique_id
    qp = qpgen.make("c0")
    rng = np.random.default_rng(5)
    D = rng.uniform(0.5, 2.0, qp.m2)
    b = rng.standard_normal(qp.m2)
    s1 = from_qp(qp)
    s1.ipm_factor_once("low")
    s2 = from_qp(qp, rank=0, world=1, nccl_uid=nccl_unique_id())
    s2.ipm_factor_once("low")
    # same iterates up to rounding order (Cᵀp summed in another order, fp64 atomics): counts ±2 at a
    # tight tolerance (late CG steps are rounding-decided, DESIGN R12), 5 fixed iterations to 1e-10
    x1, it1, _, _ = s1.pcg_solve(D, b, tol=1e-12, maxit=300)
    x2, it2, _, _ = s2.pcg_solve(D, b, tol=1e-12, maxit=300)
    assert abs(it1 - it2) <= 2 and np.linalg.norm(x1 - x2) <= 1e-9 * np.linalg.norm(x1)
    x1, _, _, _ = s1.pcg_solve(D, b, tol=0.0, maxit=5)
    x2, _, _, _ = s2.pcg_solve(D, b, tol=0.0, maxit=5)
    assert np.linalg.norm(x1 - x2) <= 1e-10 * np.linalg.norm(x1)
    r1 = s1.ipm_solve(ipm_tol=1e-10)
    r2 = s2.ipm_solve(ipm_tol=1e-10)
    assert r1["converged"] and r2["converged"]
    assert abs(r1["objective"] - r2["objective"]) <= 1e-10 * max(1.0, abs(r1["objective"]))


DENSE_M1 = dict(n=400, m1=200, m2=500, seed=6, g_nnz=8)   # W = (F⁻¹)₁₁ chosen by bytes (tests/test_gpu_paths.py)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_dense_w_pcg_matches_oracle(world):
    """Sharded rows with the explicit W: every rank applies its contiguous run of W's lower-triangle
    chunks and the partial w are summed by the all-reduce; the concatenated PCG solution matches the
    oracle at fixed iterations (1e-8, reading R16) and every rank took the same decisions."""
    d = dict(DENSE_M1)
    qp = qpgen.scaled_random_qp(d.pop("n"), d.pop("m1"), d.pop("m2"), **d)
    rng = np.random.default_rng(11)
    D = rng.uniform(0.5, 2.0, qp.m2)
    b = rng.standard_normal(qp.m2)
    fs = make_fsolver(qp.H, qp.A)

    def body(rank, comm):
        s = _solver(qp, rank, world, comm)
        assert s.stats()["dense_w_enabled"] == 1.0
        sl = slice(s.row0, s.row0 + s.m2)
        x, it, rr, rc = s.pcg_solve(D[sl], b[sl], tol=0.0, maxit=12)
        s.close()
        return s.row0, x, it
    res = run_ranks(world, body)
    xs = np.concatenate([r[1] for r in res])
    assert {r[2] for r in res} == {12}
    xo, ito, _, _, _ = pcg(lambda p: KF_apply(qp, fs, D, p), b, lambda r: r / D, 0.0, 12)
    assert np.linalg.norm(xs - xo) <= 1e-8 * np.linalg.norm(xo)


def test_sharded_dense_w_ipm_matches_oracle(monkeypatch):
    """c0 with W forced (QPB_DENSE_W=2) on two ranks: the sharded IPM reaches the oracle's objective."""
    from oracle.ipm import ipm_solve as oracle_ipm
    monkeypatch.setenv("QPB_DENSE_W", "2")
    qp = qpgen.make("c0")
    ref = oracle_ipm(qp, precond="low", ipm_tol=1e-10)

    def body(rank, comm):
        s = _solver(qp, rank, 2, comm)
        assert s.stats()["dense_w_enabled"] == 1.0
        r = s.ipm_solve(ipm_tol=1e-10, max_ipm=100)
        s.close()
        return r
    res = run_ranks(2, body)
    for r in res:
        assert r["converged"]
        assert abs(r["objective"] - ref.objective) <= 1e-8 * max(1.0, abs(ref.objective))
    assert res[0]["pcg_iters"] == res[1]["pcg_iters"]


@pytest.mark.parametrize("world", [2, 3])
def test_operator_halo_mode_matches_oracle(world):
    """Halo mode of the sharded operator (qp_operator_apply_halo; BJ configs[4], north_star "boundary entries
    of p are exchanged"): on a band-local grid QP every rank plans the same owned ranges and windows as the
    oracle's definition (oracle.sharded.halo_plan, bit-exact), its product equals H p + Cᵀ D⁻¹ C p on the
    owned range (1e-12), only the owned entries of p are read, and it sends far fewer than n doubles."""
    from oracle.sharded import halo_plan, partition_rows
    from paper_2104_12916_b200.binding import from_qp
    qp = qpgen.make_grid_qp(24, 16, 0, seed=5, name="band24", band=8, m2_band=1500)
    C = qp.C.tocsr()
    rng = np.random.default_rng(3)
    D = rng.uniform(0.5, 2.0, qp.m2)
    p = rng.standard_normal(qp.n)
    ref = qp.H @ p + C.T @ ((C @ p) / D)
    oplan = halo_plan(qp.H, C, partition_rows(C.indptr, qp.m2, world), world)
    assert oplan["enabled"]

    def body(rank, comm):
        s = from_qp(qp, rank=rank, world=world, allreduce=comm.fn(rank), halo=comm.halo(rank))
        plan = s.operator_halo_plan()
        lo, hi = plan["own"]
        pin = np.full(qp.n, 1e300)         # poison: only the owned entries may be used as given
        pin[lo:hi] = p[lo:hi]
        q, pw = s.operator_apply_halo(D[s.row0:s.row0 + s.m2], pin)
        q_ar = s.operator_apply(D[s.row0:s.row0 + s.m2], p)     # the all-reduce path, same context
        s.close()
        return plan, q[lo:hi], pw, q_ar
    res = run_ranks(world, body)
    for g, (plan, qg, pw, q_ar) in enumerate(res):
        assert plan["enabled"]
        assert plan["own"] == (int(oplan["b"][g]), int(oplan["b"][g + 1]))
        assert plan["p_window"] == (int(oplan["p_lo"][g]), int(oplan["p_hi"][g]))
        assert plan["q_window"] == (int(oplan["q_lo"][g]), int(oplan["q_hi"][g]))
        a, b = plan["p_window"]
        assert np.array_equal(pw[a:b], p[a:b])                   # the window of p was filled exactly
        assert plan["sent_doubles"] < qp.n // 2
        assert np.linalg.norm(q_ar - ref) <= 1e-12 * np.linalg.norm(ref)
    got = np.concatenate([r[1] for r in res])
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_operator_halo_mode_rejected_for_random_rows():
    """c0's rows of C reach all of x: with 4 ranks the plan is disabled on every rank and the halo call
    returns QP_ESTATE; the all-reduce path still serves."""
    from paper_2104_12916_b200.binding import QPError, from_qp
    qp = qpgen.make("c0")

    def body(rank, comm):
        s = from_qp(qp, rank=rank, world=4, allreduce=comm.fn(rank), halo=comm.halo(rank))
        plan = s.operator_halo_plan()
        with pytest.raises(QPError):
            s.operator_apply_halo(np.ones(s.m2), np.zeros(qp.n))
        s.close()
        return plan["enabled"]
    assert run_ranks(4, body) == [False] * 4
