"""K5 streaming residual (cqr_resid_gram) on m x k device arrays: event-timed
sweeps, and the algorithmic rates (bytes: Q and A read once; flops: TRMM
k(k+1) + SYRK k(k+1) per row).  --reps 1 for an ncu capture."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200.metrics import residual_gram  # noqa: E402
from paper_2507_07788_b200.workloads import device_gaussian  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=32_000_000)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
sp = cq.VectorSpace(a.m)
x = device_gaussian(cq.CudaVectorArray.zeros(sp, a.k), 1)
q = device_gaussian(cq.CudaVectorArray.zeros(sp, a.k), 2)
r = np.triu(np.random.default_rng(0).standard_normal((a.k, a.k)))
residual_gram(x, q, r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    residual_gram(x, q, r)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
byts = 2 * a.m * a.k * 8
fl = 2 * a.m * a.k * (a.k + 1)
print(json.dumps({"m": a.m, "k": a.k, "ms_per_call": ms, "GB_s": byts / ms / 1e6, "TF_s": fl / ms / 1e9}))
