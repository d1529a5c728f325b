"""Update pass (iteration mode) at every basis width of config 4's chain, with
the cross-Gram lag off / on (cqr_debug_update_lag) and the 16-row sub-panel
threshold (cqr_debug_update_sr16_from); one JSON line per (q, setting).
python tools/diag/update_lag_sweep.py [--m 8000000] [--qs 160,176,...]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200 import _lib  # noqa: E402
from paper_2507_07788_b200._device import ctx  # noqa: E402
from paper_2507_07788_b200._engine import Engine  # noqa: E402
from paper_2507_07788_b200.workloads import device_gaussian  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=8_000_000)
ap.add_argument("--qs", default=",".join(str(16 * j) for j in range(1, 32)))
ap.add_argument("--settings", default="0:193,0:145,2:145", help="lag:sr16_from pairs")
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
m, p = a.m, 16
lib = ctx().lib
qb = device_gaussian(cq.CudaVectorArray.zeros(cq.VectorSpace(m), p), 3)
for q in [int(v) for v in a.qs.split(",")]:
    q_in = device_gaussian(cq.CudaVectorArray.zeros(cq.VectorSpace(m), q, capacity=512), 2)
    eng = Engine(p, cq.AlgoConfig(), q=q)
    g = torch.randn((p, p), dtype=torch.float64, device="cuda")
    eng.G.copy_(g @ g.T + p * torch.eye(p, dtype=torch.float64, device="cuda"))
    assert eng.factor(_lib.POLICY_PLAIN, m, p).code == _lib.FACTORED
    eng.Bt.copy_(1e-3 * torch.randn_like(eng.Bt))
    for st in a.settings.split(","):
        lag, sr16 = (int(v) for v in st.split(":"))
        lib.cqr_debug_update_lag(lag)
        lib.cqr_debug_update_sr16_from(sr16)
        eng.update_pass(q_in, qb, initial=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            eng.update_pass(q_in, qb, initial=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        flops = 4.0 * m * q * p + 2.0 * m * p * (p + 1)
        print(json.dumps({"q": q, "lag": lag, "sr16_from": sr16, "ms": round(ms, 4), "tfs": round(flops / ms / 1e9, 2)}),
              flush=True)
    del q_in, eng
