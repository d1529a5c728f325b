"""Self-Gram schedules at one shape (cqr_set_gram_pairs modes: 1 = default,
2 = block-row pairs, 0 = tiles): python tools/gram_probe.py --m M --k K"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=32_000_000)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--modes", default="1,2")
a = ap.parse_args()
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200._device import ctx
from paper_2507_07788_b200._engine import Engine
from paper_2507_07788_b200.workloads import device_gaussian

x = device_gaussian(cq.CudaVectorArray.zeros(cq.VectorSpace(a.m), a.k), 1)
eng = Engine(a.k, cq.AlgoConfig())
out = {"m": a.m, "k": a.k}
for mode in [int(v) for v in a.modes.split(",")] * 2:
    ctx().lib.cqr_set_gram_pairs(mode)
    eng.gram(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        eng.gram(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    out.setdefault(f"mode{mode}_ms", []).append(round(ms, 3))
    out[f"mode{mode}_tfs"] = round(a.m * a.k * (a.k + 1) / ms / 1e9, 2)
ctx().lib.cqr_set_gram_pairs(1)
print(json.dumps(out))
