"""Per-call trace of the k x k factor inside one algorithm run: policy, status
code, attempts, norm-estimate iterations and phase times (debug profile).

    python tools/factor_trace.py [--m 2000000 --k 256 --cond 15]   (BASELINE config 3 construction)
"""
import argparse, ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2_000_000)
ap.add_argument("--k", type=int, default=256)
ap.add_argument("--cond", type=float, default=15.0)
a = ap.parse_args()
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200 import _engine
from paper_2507_07788_b200.workloads import device_svd_matrix

space = cq.VectorSpace(a.m)
x = device_svd_matrix(lambda t: cq.CudaVectorArray.from_device_colmajor(space, t.T), a.m, a.k, a.cond, 2025,
                      u_from="cholqr2")
orig = _engine.Engine.factor
trace = []


def traced(self, policy, *args, **kw):
    st = orig(self, policy, *args, **kw)
    buf = (ctypes.c_ulonglong * 16)()
    self.cx.lib.cqr_debug_factor_profile(buf)
    t0 = buf[0]
    trace.append({"policy": int(policy), "code": st.code, "attempts": st.retries,
                  "est_iters": int(buf[8]) if buf[8] < 1000 else None,
                  "phases_us": [round((buf[i] - t0) / 1e3, 1) if buf[i] >= t0 else None for i in range(7)]})
    return st


_engine.Engine.factor = traced
res = cq.rs_chol_qr(x)
torch.cuda.synchronize()
trace = []
res = cq.rs_chol_qr(x)
for t in trace:
    print(json.dumps(t))
