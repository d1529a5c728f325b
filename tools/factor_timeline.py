"""Kernel timeline of back-to-back k x k factor calls (torch.profiler):
per-kernel durations and the gaps between them.
    python tools/factor_timeline.py --k 64 --policy plain"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--policy", default="plain")
ap.add_argument("--n", type=int, default=8)
a = ap.parse_args()
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200 import _lib
from paper_2507_07788_b200._engine import Engine

k = a.k
eng = Engine(k, cq.AlgoConfig())
g = torch.randn((k, k), dtype=torch.float64, device="cuda")
eng.G.copy_(g @ g.T + k * torch.eye(k, dtype=torch.float64, device="cuda"))
pol = {"plain": _lib.POLICY_PLAIN, "recompute": _lib.POLICY_RECOMPUTE, "shift_once": _lib.POLICY_SHIFT_ONCE}[a.policy]
for _ in range(3):
    eng.collect([eng.factor_async(pol, 10**6, k)])
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.n):
        h = eng.factor_async(pol, 10**6, k)
        eng.collect([h])
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
rows = []
for i, e in enumerate(ev[:12]):
    gap = e.time_range.start - ev[i - 1].time_range.end if i else 0.0
    rows.append((e.name[:40], round(e.time_range.end - e.time_range.start, 1), round(gap, 1)))
import ctypes
buf = (ctypes.c_ulonglong * 16)()
eng.cx.lib.cqr_debug_factor_profile(buf)
phases = [round((buf[i] - buf[0]) / 1e3, 2) if buf[i] >= buf[0] else None for i in range(7)]
print(json.dumps({"k": k, "policy": a.policy, "phases_us(last call: 0 start,1 X formed,2 copied in,3 factored,"
                  "4 stored,6 end)": phases, "first_kernels_us_gap": rows[:4]}))
