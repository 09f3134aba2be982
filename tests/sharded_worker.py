"""One rank of the multi-PROCESS sharded-mode test (tests/test_gpu_sharded_mp.py).

Each process: torch.distributed (gloo, 127.0.0.1) for the collective, the library's sharded ν-row mode
(qp_b200.h "Sharded mode") on cuda:0 with qp_allreduce_fn backed by that process group (the rank's
stream is synchronised, the buffer copied to the host, all-reduced by gloo, copied back: no kernel of
one process ever waits on the other's).  Writes a JSON result for the test to compare with the oracle.

usage: python tests/sharded_worker.py CASE OUT.json   (RANK / WORLD_SIZE / MASTER_* from the env)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    from cuda.bindings import runtime as rt

    import qpgen
    from paper_2104_12916_b200.binding import from_qp

    case, out = sys.argv[1], sys.argv[2]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    ops = {0: dist.ReduceOp.SUM, 1: dist.ReduceOp.MAX, 2: dist.ReduceOp.MIN}

    def allreduce(buf, count, op, stream):
        (err,) = rt.cudaStreamSynchronize(stream)
        if int(err):
            return int(err)
        host = np.empty(count)
        (err,) = rt.cudaMemcpy(host.ctypes.data, buf, count * 8, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        if int(err):
            return int(err)
        t = torch.from_numpy(host)
        dist.all_reduce(t, op=ops[op])
        # back on the caller's stream, and complete before returning: a plain cudaMemcpy from pageable memory
        # may return before its DMA lands and is not ordered with the library's non-blocking stream
        (err,) = rt.cudaMemcpyAsync(buf, t.numpy().ctypes.data, count * 8, rt.cudaMemcpyKind.cudaMemcpyHostToDevice,
                                    stream)
        if int(err):
            return int(err)
        (err,) = rt.cudaStreamSynchronize(stream)
        return int(err)

    qp = qpgen.make("c0") if case == "c0" else qpgen.scaled_random_qp(700, 130, 900, seed=3)
    s = from_qp(qp, rank=rank, world=world, allreduce=allreduce)
    s.ipm_factor_once("low")
    rng = np.random.default_rng(11)
    D = rng.uniform(0.5, 2.0, qp.m2)
    b = rng.standard_normal(qp.m2)
    lo, hi = s.row0, s.row0 + s.m2
    res = {"rank": rank, "row0": lo, "row1": hi}
    for k in (1, 4):
        x, it, rr, rc = s.pcg_solve(D[lo:hi], b[lo:hi], tol=0.0, maxit=k)
        res[f"x{k}"] = x.tolist()
        res[f"it{k}"] = it
    x, it, rr, rc = s.pcg_solve(D[lo:hi], b[lo:hi], tol=1e-12, maxit=2000)
    res.update(x_tight=x.tolist(), it_tight=it, rr_tight=rr)
    # the x-space operator with sharded rows: every rank's q is the all-reduced H p + Cᵀ(D⁻¹∘(C p))
    pg = np.random.default_rng(12).standard_normal(qp.n)
    res["Gp"] = s.operator_apply(D[lo:hi], pg).tolist()
    if case == "c0":
        r = s.ipm_solve(ipm_tol=1e-10)
        res.update(objective=r["objective"], converged=bool(r["converged"]), n_ipm=r["n_ipm"],
                   x_ipm=r["x"].tolist(), nu_ipm=r["nu"].tolist(), s_ipm=r["s"].tolist(),
                   pcg_iters=r["pcg_iters"])
    json.dump(res, open(out, "w"))
    s.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
