"""Where one chol_qr_update call spends its time at config 4's shape
(m = 8M, basis q, block 16): event-timed kernels vs wall clock, and a cProfile.
    python tools/update_overhead.py [--q 256]"""
import argparse, cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--q", type=int, default=256)
a = ap.parse_args()
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200 import _device
from paper_2507_07788_b200.workloads import device_gaussian

m, p = 8_000_000, 16
space = cq.VectorSpace(m)
g = device_gaussian(cq.CudaVectorArray.zeros(space, a.q), 5)
q0 = cq.rs_chol_qr(g)
qb, rb = q0.q, q0.r
c = np.random.default_rng(1).standard_normal((a.q, p))
blk = qb.lincomb(c)
noise = device_gaussian(cq.CudaVectorArray.zeros(space, p), 7)
blk.axpy(1e-8, noise)
for _ in range(2):
    cq.chol_qr_update(qb, rb, blk)
torch.cuda.synchronize()
cx = _device.ctx()
cx.timer = _device.KernelTimer()
t0 = time.perf_counter()
res = cq.chol_qr_update(qb, rb, blk)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
s = cx.timer.summary()
cx.timer = None
print({"wall_ms": round(wall, 3), "iterations": res.iterations,
       "kernels_ms": {n: round(sum(v["ms"]), 3) for n, v in s.items()}})
pr = cProfile.Profile()
pr.enable()
res = cq.chol_qr_update(qb, rb, blk)
torch.cuda.synchronize()
pr.disable()
out = io.StringIO()
pstats.Stats(pr, stream=out).sort_stats("tottime").print_stats(14)
print(out.getvalue()[:3000])
