"""Host time of one s_chol_qr3 call on the native fixed schedule (config 1
shape), segment by segment, plus a cProfile of back-to-back calls.
python tools/diag/host_native.py [--m 200000] [--k 64]"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200 import _engine as en  # noqa: E402
from paper_2507_07788_b200 import algorithms as al  # noqa: E402
from paper_2507_07788_b200.workloads import device_svd_matrix  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=200_000)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--calls", type=int, default=200)
args = ap.parse_args()
m, k = args.m, args.k
a = device_svd_matrix(lambda x: cq.CudaVectorArray.from_device_colmajor(cq.VectorSpace(m), x.T), m, k, 12.0, 2025)
for _ in range(20):
    cq.s_chol_qr3(a)
torch.cuda.synchronize()

T = {}


def wrap(obj, name):
    fn = getattr(obj, name)

    def w(*a_, **kw):
        t = time.perf_counter_ns()
        try:
            return fn(*a_, **kw)
        finally:
            T[name] = T.get(name, 0) + time.perf_counter_ns() - t
    setattr(obj, name, w)
    return fn


orig = {n: wrap(en.Engine, n) for n in ("__init__", "run_fixed", "collect", "r_host", "fixed_ok")}
orig_fresh = wrap(al, "_fresh_like")
N = args.calls
t0 = time.perf_counter_ns()
for _ in range(N):
    cq.s_chol_qr3(a)
torch.cuda.synchronize()
tot = time.perf_counter_ns() - t0
for n, fn in orig.items():
    setattr(en.Engine, n, fn)
al._fresh_like = orig_fresh
print(f"wall per call {tot / N / 1e3:.1f} us")
for kk, v in sorted(T.items(), key=lambda x: -x[1]):
    print(f"  {kk:15s} {v / N / 1e3:8.1f} us")

# wall of back-to-back calls with the GPU side removed from the critical path
# is not measurable here; cProfile shows where the host time goes
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    cq.s_chol_qr3(a)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
