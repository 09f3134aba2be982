"""Halo mode of the sharded operator (qp_operator_apply_halo) at FULL c4 size (n = 32e6, m2 = 6.4e7, rows of C
within ±64 of their anchor, H the 5657² grid Laplacian) with WORLD ranks as threads of this process on one
GPU: the collective hooks (qp_allreduce_fn / qp_halo_fn) go through host memory, so this run shows the
plan, the halo volumes and the result at full size — not NVLink timing (this pod has one GPU).  Each rank's
owned part of q is compared with the same context's all-reduce product (qp_operator_apply).
python scripts/operator_halo_full.py [c4] [WORLD]"""
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import qpgen  # noqa: E402
from paper_2104_12916_b200.binding import from_qp  # noqa: E402
from test_gpu_sharded import ThreadComm  # noqa: E402  (the host-side hooks of the thread tests)

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t0 = time.time()
qp = qpgen.make(cfg)
t_gen = time.time() - t0
rng = np.random.default_rng(0)
D = np.exp(rng.uniform(-4, 4, qp.m2))
p = rng.standard_normal(qp.n)
comm = ThreadComm(world)
out, errs = [None] * world, []


def body(rank):
    try:
        s = from_qp(qp, rank=rank, world=world, allreduce=comm.fn(rank), halo=comm.halo(rank))
        plan = s.operator_halo_plan()
        lo, hi = plan["own"]
        Dg = D[s.row0:s.row0 + s.m2]
        q_ar = s.operator_apply(Dg, p)
        pin = np.zeros(qp.n)
        pin[lo:hi] = p[lo:hi]
        t1 = time.time()
        q, pw = s.operator_apply_halo(Dg, pin)
        t_halo = time.time() - t1
        err = float(np.max(np.abs(q[lo:hi] - q_ar[lo:hi])) / np.max(np.abs(q_ar)))
        a, b = plan["p_window"]
        out[rank] = dict(rank=rank, rows=(int(s.row0), int(s.row0 + s.m2)), **plan,
                         rel_err_vs_allreduce_path=err, window_filled=bool(np.array_equal(pw[a:b], p[a:b])),
                         wall_s_host_hooks=t_halo)
        s.close()
    except BaseException as e:  # noqa: BLE001
        errs.append(e)
        comm.bar.abort()


ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
for t in ts:
    t.start()
for t in ts:
    t.join()
if errs:
    raise errs[0]
print(json.dumps({"config": cfg, "world": world, "n": qp.n, "m2": qp.m2, "t_generate_s": t_gen,
                  "allreduce_doubles_per_product": qp.n, "ranks": out}))
