import sys, warnings
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2507_07788_b200 as cq
from oracle import cholqr_oracle as co
from paper_2507_07788_b200.matgen import MatrixSpec, generate_host
def _matrix(m, k, cond, seed): return generate_host(MatrixSpec(m, k, cond, seed))[0]
for i, m, k, cond in [(11509, 1200, 1, 2.0), (8229, 18, 3, 2.0)]:
    rng = np.random.default_rng(1000 + i)
    p = int(min(16, max(1, k // 2)))
    q_in = np.linalg.qr(rng.standard_normal((m, k)))[0]
    r_in = np.triu(rng.standard_normal((k, k))) + k * np.eye(k)
    scale = 10.0 ** (-cond / 2)
    a_new = q_in @ rng.standard_normal((k, p)) + scale * _matrix(m, p, min(cond, 8.0), i)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = co.chol_qr_update(q_in, r_in, a_new, co.default_cfg())
        mine = cq.chol_qr_update(cq.CudaVectorArray.from_numpy(q_in), r_in, cq.CudaVectorArray.from_numpy(a_new))
    qd = mine.q.to_numpy()
    print("case", i, "its", mine.iterations, ref.iterations, "att", mine.shift_attempts, ref.shift_attempts)
    print(" err_hist dev", mine.err_history, "\n err_hist ref", getattr(ref, "err_history", None))
    for name, q in (("dev", qd), ("ref", ref.q)):
        g = q.T @ q - np.eye(q.shape[1])
        print(" ", name, "LOO", np.linalg.norm(g), "cross", np.abs(g[:k, k:]).max(), "new diag", np.abs(g[k:, k:]).max(), "basis", np.abs(g[:k,:k]).max())
    print(" R diff", np.abs(mine.r - ref.r).max(), "newQ diff", np.abs(qd[:, k:] - ref.q[:, k:]).max())
