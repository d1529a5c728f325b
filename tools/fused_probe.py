"""Fused vs two-kernel TRMM + Gram at one shape: python tools/fused_probe.py --m M --k K
(cqr_set_fused modes: 0 = TRMM then Gram, 2 = default, 1 = every fused kernel)"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=32_000_000)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200 import _lib
from paper_2507_07788_b200._device import ctx
from paper_2507_07788_b200._engine import Engine
from paper_2507_07788_b200.workloads import device_gaussian

x = device_gaussian(cq.CudaVectorArray.zeros(cq.VectorSpace(a.m), a.k), 1)
q = cq.CudaVectorArray.zeros(cq.VectorSpace(a.m), a.k)
eng = Engine(a.k, cq.AlgoConfig())
eng.gram(x)
assert eng.factor(_lib.POLICY_PLAIN, a.m, a.k).code == _lib.FACTORED
out = {"m": a.m, "k": a.k}
for fused in (0, 1, 0, 1):
    ctx().lib.cqr_set_fused(fused)   # 1: every fused kernel (k <= 64: the default one)
    eng.apply(x, q, with_gram=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        eng.apply(x, q, with_gram=True)
    e1.record()
    torch.cuda.synchronize()
    out.setdefault("fused_ms" if fused else "unfused_ms", []).append(round(e0.elapsed_time(e1) / a.reps, 3))
ctx().lib.cqr_set_fused(2)
print(json.dumps(out))
