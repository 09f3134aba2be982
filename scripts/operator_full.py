"""The north_star's operator G p = H p + Cᵀ(D⁻¹∘(C p)) (qp_operator_apply) at FULL BASELINE size — C3
(n = 4e6, m2 = 8e6, Zipf rows) and C4 (n = 32e6, m2 = 6.4e7, banded) — where F cannot be factored, timed
with CUDA events over R applications on device-resident vectors.  Algorithmic bytes per application:
12·nnz(H) + 24·nnz(C) (values + column indices, C read twice: rows, then Cᵀ) + 8·(3·m2 + 2·n) (D, the
t write and read, p, q) against MEASURED_PEAKS.json's copy bandwidth.  python scripts/operator_full.py c4 [R]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import qpgen  # noqa: E402
from paper_2104_12916_b200.binding import from_qp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 20
t0 = time.time()
qp = qpgen.make(cfg)
t_gen = time.time() - t0
t0 = time.time()
s = from_qp(qp, vectors_on_device=True)
t_setup = time.time() - t0
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
D = torch.exp(torch.rand(qp.m2, generator=g, device=dev, dtype=torch.float64) * 8 - 4)
p = torch.randn(qp.n, generator=g, device=dev, dtype=torch.float64)
q = torch.empty(qp.n, device=dev, dtype=torch.float64)
for _ in range(3):
    s.operator_apply(D, p, out=q)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(R):
    s.operator_apply(D, p, out=q)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
nnzH, nnzC = qp.H.nnz, qp.C.nnz
bytes_alg = 12.0 * nnzH + 24.0 * nnzC + 8.0 * (3 * qp.m2 + 2 * qp.n)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
gbs = bytes_alg / (ms / 1e3) / 1e9
# spot check against SciPy on sampled rows (the full oracle product is two SpMVs on the host)
qh = q.cpu().numpy()
ph, Dh = p.cpu().numpy(), D.cpu().numpy()
rng = np.random.default_rng(1)
rows = np.sort(rng.choice(qp.n, size=2000, replace=False))
t_full = qp.C @ ph / Dh
ref = qp.H[rows] @ ph + qp.C.T.tocsr()[rows] @ t_full
err = float(np.max(np.abs(qh[rows] - ref)) / np.max(np.abs(ref)))
print(json.dumps({"config": cfg, "n": qp.n, "m2": qp.m2, "nnz_H": int(nnzH), "nnz_C": int(nnzC),
                  "ms_per_apply": ms, "algorithmic_bytes": bytes_alg, "GBps": gbs, "frac_of_measured_copy": gbs / peak,
                  "peak": peak, "sampled_rel_err_vs_scipy": err, "t_generate_s": t_gen, "t_setup_s": t_setup,
                  "kernels": "k_op_t + k_op_q (qp_operator_apply)"}))
