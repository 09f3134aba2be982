"""World-size-2 gloo test of the multi-GPU host logic (CPU only).

bench.py --gpus N runs one replica of the c1 IPM per GPU (the F-solve carries
≥ 95 % of the bytes and is replicated, so ν-row sharding cannot scale; throughput scales by
replicas).  The whole-job value is Σ PCG iterations over ranks ÷ the slowest rank's time; this
test runs that aggregation and the barrier/all-reduce plumbing in two gloo processes.
"""
import os
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    use = True
    bench.barrier(use)
    iters = [1000, 1200][rank]
    ms = [500.0, 800.0][rank]
    value, tot, mx = bench.aggregate(iters, ms, use)
    shared = bench.aggregate(1000, ms, use, True)   # sharded mode: same iterations on every rank
    out[rank] = (value, tot, mx, shared)
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_replica_aggregation_two_ranks():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        value, tot, mx, shared = out[r]
        assert tot == 2200 and mx == 800.0
        assert abs(value - 2200 / 0.8) < 1e-9      # Σ iterations / max-over-ranks seconds
        assert shared[1] == 1000 and abs(shared[0] - 1000 / 0.8) < 1e-9   # counted once


# ---------------------------------------------------------------- sharded ν rows
def _sharded_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist
    import qpgen
    from oracle.fsolve import make_fsolver
    from oracle.sharded import partition_rows, sharded_pcg
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    qp = qpgen.make("c0")
    fs = make_fsolver(qp.H, qp.A)
    C = qp.C.tocsr()
    bounds = partition_rows(C.indptr, qp.m2, world)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    rng = np.random.default_rng(7)
    D = rng.uniform(0.5, 2.0, qp.m2)
    b = rng.standard_normal(qp.m2)
    x_g, it, rr, conv = sharded_pcg(C[r0:r1], fs, D[r0:r1], b[r0:r1], lambda r: r / D[r0:r1], 1e-10, 500,
                                    allreduce)
    out[rank] = (r0, r1, x_g, it, rr, conv)
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_sharded_pcg_two_ranks_matches_unsharded():
    """Two gloo ranks, each owning a contiguous slice of the c0 inequality rows, run the sharded
    PCG (Cᵀp all-reduced before the replicated F-solve, inner products all-reduced): the
    concatenated solution and the iteration count equal the single-process PCG's."""
    import numpy as np
    import qpgen
    from oracle.fsolve import make_fsolver
    from oracle.kkt import KF_apply
    from oracle.pcg import pcg
    world = 2
    port = 30500 + (os.getpid() % 1000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sharded_worker, args=(world, port, out), nprocs=world, join=True)
    qp = qpgen.make("c0")
    fs = make_fsolver(qp.H, qp.A)
    rng = np.random.default_rng(7)
    D = rng.uniform(0.5, 2.0, qp.m2)
    b = rng.standard_normal(qp.m2)
    x, it, rr, conv, _ = pcg(lambda p: KF_apply(qp, fs, D, p), b, lambda r: r / D, 1e-10, 500)
    assert out[0][1] == out[1][0] and out[0][0] == 0 and out[1][1] == qp.m2
    xs = np.concatenate([out[0][2], out[1][2]])
    assert out[0][3] == out[1][3] and abs(out[0][3] - it) <= 1
    assert np.linalg.norm(xs - x) <= 1e-9 * np.linalg.norm(x)


# ---------------------------------------------------------------- halo mode of the operator (BJ configs[4])
def _band_qp():
    import qpgen
    return qpgen.make_grid_qp(24, 16, 0, seed=5, name="band24", band=8, m2_band=1500)


def _halo_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist
    from oracle.sharded import halo_operator, halo_plan, partition_rows
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def exchange(to_prev, to_next, n_fp, n_fn):
        fp, fn = torch.zeros(n_fp, dtype=torch.float64), torch.zeros(n_fn, dtype=torch.float64)
        ops = []
        if rank > 0 and len(to_prev):
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(to_prev)), rank - 1))
        if rank + 1 < world and len(to_next):
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(to_next)), rank + 1))
        if n_fp:
            ops.append(dist.P2POp(dist.irecv, fp, rank - 1))
        if n_fn:
            ops.append(dist.P2POp(dist.irecv, fn, rank + 1))
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()
        return fp.numpy(), fn.numpy()

    qp = _band_qp()
    C = qp.C.tocsr()
    bounds = partition_rows(C.indptr, qp.m2, world)
    plan = halo_plan(qp.H, C, bounds, world)
    assert plan["enabled"]
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    rng = np.random.default_rng(3)
    D = rng.uniform(0.5, 2.0, qp.m2)
    p = rng.standard_normal(qp.n)
    lo, hi = int(plan["b"][rank]), int(plan["b"][rank + 1])
    pin = np.full(qp.n, np.nan)            # only the owned entries are valid on entry
    pin[lo:hi] = p[lo:hi]
    q, pw = halo_operator(rank, plan, qp.H, C[r0:r1], D[r0:r1], pin, exchange)
    sent = (max(0, int(plan["p_hi"][rank - 1]) - lo) + lo - int(plan["q_lo"][rank]) if rank > 0 else 0) + \
           (max(0, hi - int(plan["p_lo"][rank + 1])) + int(plan["q_hi"][rank]) - hi if rank + 1 < world else 0)
    out[rank] = (lo, hi, q[lo:hi], sent)
    dist.destroy_process_group()


@pytest.mark.timeout(180)
@pytest.mark.parametrize("world", [2, 3])
def test_halo_operator_gloo_matches_dense(world):
    """The halo-mode product on gloo ranks (boundary entries of p in, foreign parts of q out and added)
    equals H p + Cᵀ D⁻¹ C p computed in one piece, on each rank's owned range, and moves far fewer than
    the n doubles of the all-reduce."""
    import numpy as np
    port = 31500 + (os.getpid() % 1000) + world
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_halo_worker, args=(world, port, out), nprocs=world, join=True)
    qp = _band_qp()
    rng = np.random.default_rng(3)
    D = rng.uniform(0.5, 2.0, qp.m2)
    p = rng.standard_normal(qp.n)
    ref = qp.H @ p + qp.C.T @ ((qp.C @ p) / D)
    got = np.concatenate([out[r][2] for r in range(world)])
    assert out[0][0] == 0 and out[world - 1][1] == qp.n
    assert all(out[r][1] == out[r + 1][0] for r in range(world - 1))
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    assert max(out[r][3] for r in range(world)) < qp.n // 2


def test_halo_plan_rejects_unstructured_rows():
    """Random columns (c0) reach every part of x: with more than two ranks (two are always neighbours) the
    plan must say so and keep the all-reduce."""
    import qpgen
    from oracle.sharded import halo_plan, partition_rows
    qp = qpgen.make("c0")
    C = qp.C.tocsr()
    assert not halo_plan(qp.H, C, partition_rows(C.indptr, qp.m2, 4), 4)["enabled"]
