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
    out[rank] = (value, tot, mx)
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_replica_aggregation_two_ranks():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        value, tot, mx = out[r]
        assert tot == 2200 and mx == 800.0
        assert abs(value - 2200 / 0.8) < 1e-9      # Σ iterations / max-over-ranks seconds
