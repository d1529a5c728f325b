"""Diagnostic: the config-4 append chain on the device against the oracle,
block by block (per-block R error, LOO of the device basis)."""
import sys
import warnings

import numpy as np

sys.path.insert(0, ".")
import paper_2507_07788_b200 as cq  # noqa: E402
from oracle import cholqr_oracle as co  # noqa: E402
from paper_2507_07788_b200.workloads import next_block  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 31
reserve = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = 16
rng = np.random.default_rng(4)
q0 = np.linalg.qr(rng.standard_normal((m, p)))[0]
ref = co.rs_chol_qr(q0)
q_ref, r_ref = ref.q, ref.r
res0 = cq.rs_chol_qr(cq.CudaVectorArray.from_numpy(q0))
q_dev, r_dev = res0.q, res0.r
if reserve:
    q_dev.reserve(p * (blocks + 1))
for j in range(blocks):
    a_new = next_block(q_ref, rng, p)
    r_o = co.chol_qr_update(q_ref, r_ref, a_new)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        r_d = cq.chol_qr_update(q_dev, r_dev, cq.CudaVectorArray.from_numpy(a_new))
    k = r_d.q.ncols
    newc = slice(k - p, k)
    err_b = np.max(np.abs(r_d.r[: k - p, newc] - r_o.r[: k - p, newc])) / np.max(np.abs(r_o.r[: k - p, newc]))
    err_d = np.max(np.abs(r_d.r[newc, newc] - r_o.r[newc, newc])) / np.max(np.abs(r_o.r[newc, newc]))
    qd = r_d.q.to_numpy()
    loo = np.linalg.norm(np.eye(k) - qd.T @ qd)
    dq = np.max(np.abs(qd[:, newc] - r_o.q[:, newc]))
    print(f"block {j+1:2d} q={k-p:3d} its d/o {r_d.iterations}/{r_o.iterations} att {r_d.shift_attempts}/{r_o.shift_attempts} "
          f"B err {err_b:.2e} Rjj err {err_d:.2e} newQ diff {dq:.2e} LOO {loo:.2e} oracle LOO {co.loo_fro(r_o.q):.2e}",
          flush=True)
    q_ref, r_ref = r_o.q, r_o.r
    q_dev, r_dev = r_d.q, r_d.r
