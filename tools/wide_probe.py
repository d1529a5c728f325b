"""Timing of the generic wide paths (k > 256): rs_chol_qr / chol_qr2 at
m x k and the per-kernel split.   python tools/wide_probe.py --m 500000 --k 512"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=500_000)
ap.add_argument("--k", type=int, default=512)
a = ap.parse_args()
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200 import _device
from paper_2507_07788_b200.workloads import device_gaussian

x = device_gaussian(cq.CudaVectorArray.zeros(cq.VectorSpace(a.m), a.k), 3)
cq.chol_qr2(x)
torch.cuda.synchronize()
cx = _device.ctx()
cx.timer = _device.KernelTimer()
t0 = time.perf_counter()
res = cq.chol_qr2(x)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
s = cx.timer.summary()
cx.timer = None
print(json.dumps({"m": a.m, "k": a.k, "chol_qr2_ms": round(wall, 3),
                  "kernels_ms": {n: [round(v, 3) for v in d["ms"]] for n, d in s.items()},
                  "loo": cq.loss_of_orthogonality(res.q, norm="frobenius")}))
