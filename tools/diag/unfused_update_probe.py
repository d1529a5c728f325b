"""Components of the unfused chol_qr_update path (new blocks wider than 16
columns: pn_chol_qr with wide panels) timed one by one at m x q basis, m x p
block: projection lincomb, axpy, TRMM, Gram, cross Gram, column copy.
python tools/diag/unfused_update_probe.py [m] [q] [p]"""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200 import algorithms as alg  # noqa: E402
from paper_2507_07788_b200._engine import Engine, cross_gram_device, gram_device  # noqa: E402
from paper_2507_07788_b200.workloads import device_gaussian  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
q = int(sys.argv[2]) if len(sys.argv) > 2 else 128
p = int(sys.argv[3]) if len(sys.argv) > 3 else 32
sp = cq.VectorSpace(m)
wide = device_gaussian(cq.CudaVectorArray.zeros(sp, 256), 1)
q_in = device_gaussian(cq.CudaVectorArray.zeros(sp, q, capacity=256), 2)
blk = device_gaussian(cq.CudaVectorArray.zeros(sp, p), 3)
bt = 1e-3 * torch.randn((p, q), dtype=torch.float64, device="cuda")
eng = Engine(p, cq.AlgoConfig(), q=q)
eng.gram(blk)
eng.factor(cq._lib.POLICY_PLAIN, m, p)
tmp = cq.CudaVectorArray.zeros(sp, p)


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"m": m, "q": q, "p": p}
out["lincomb_proj_ms"] = t(lambda: alg._lincomb_device(q_in, bt, q, p))
out["lincomb_sub_ms"] = t(lambda: alg._lincomb_device(q_in, bt, q, p, minus_from=blk))
proj = alg._lincomb_device(q_in, bt, q, p)
out["axpy_ms"] = t(lambda: blk.axpy(-1.0, proj))
out["trmm_ms"] = t(lambda: eng.apply(blk, tmp, with_gram=False))
out["trmm_gram_ms"] = t(lambda: eng.apply(blk, tmp, with_gram=True))
out["gram_ms"] = t(lambda: eng.gram(blk))
out["cross_gram_ms"] = t(lambda: cross_gram_device(q_in, blk))
out["copy_cols_ms"] = t(lambda: wide.copy(range(64, 64 + p)))
out["block_copy_ms"] = t(lambda: blk.copy())
fl = 2.0 * m * q * p
out["ideal_proj_or_cross_ms"] = max(fl / 37.2e12, 8.0 * m * (q + p) / 6.54e12) * 1e3
print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in out.items()}))
