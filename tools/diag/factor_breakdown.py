"""Per-kernel durations and inter-kernel gaps of back-to-back factor calls
(torch.profiler / CUPTI), for several k and policies; q > 0 = update policy
with a q x k cross Gram (the config-4 shape)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200 import _lib  # noqa: E402
from paper_2507_07788_b200._engine import Engine  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

POL = {"plain": _lib.POLICY_PLAIN, "recompute": _lib.POLICY_RECOMPUTE, "shift_once": _lib.POLICY_SHIFT_ONCE,
       "update": _lib.POLICY_UPDATE}


def run(k, policy, q=0, n=6):
    eng = Engine(k, cq.AlgoConfig(), q=q)
    g = torch.randn((k, k), dtype=torch.float64, device="cuda")
    spd = g @ g.T + k * torch.eye(k, dtype=torch.float64, device="cuda")
    if q:
        eng.Bt.copy_(1e-3 * torch.randn_like(eng.Bt))
    kw = dict(update_b=True) if policy == "update" else {}
    for _ in range(3):
        eng.G.copy_(spd)
        eng.collect([eng.factor_async(POL[policy], 10**6, k, **kw)])
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(n):
            eng.G.copy_(spd)
            eng.collect([eng.factor_async(POL[policy], 10**6, k, **kw)])
        torch.cuda.synchronize()
    ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                key=lambda e: e.time_range.start)
    per = {}
    prev_end = None
    for e in ev:
        name = e.name.split("(")[0].replace("void ", "")[:40]
        d = e.time_range.end - e.time_range.start
        gap = (e.time_range.start - prev_end) if prev_end is not None else 0.0
        prev_end = e.time_range.end
        s = per.setdefault(name, [0.0, 0.0, 0])
        s[0] += d
        s[1] += gap
        s[2] += 1
    buf = (ctypes.c_ulonglong * 16)()
    eng.cx.lib.cqr_debug_factor_profile(buf)
    phases = [round((buf[i] - buf[0]) / 1e3, 2) if buf[i] >= buf[0] else None for i in range(7)]
    steps = max(int(buf[11]), 1)
    phases.append({"steps": int(buf[11]), "panel_cyc": buf[9] // steps, "update_cyc": buf[10] // steps,
                   "diag_cyc": buf[12] // steps})
    out = {n_: {"mean_us": round(v[0] / v[2], 2), "gap_before_us": round(v[1] / v[2], 2)} for n_, v in per.items()}
    # host-visible time per call
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(n):
        eng.G.copy_(spd)
        eng.collect([eng.factor_async(POL[policy], 10**6, k, **kw)])
    t1.record()
    torch.cuda.synchronize()
    print(json.dumps({"k": k, "q": q, "policy": policy, "call_us": round(t0.elapsed_time(t1) * 1e3 / n, 1),
                      "kernels": out, "phases_us": phases}), flush=True)


import sys as _s
CASES = [(16, "update", 256), (16, "update", 496), (64, "plain", 0), (64, "shift_once", 0),
         (128, "plain", 0), (256, "plain", 0), (256, "recompute", 0)]
if len(_s.argv) > 1 and _s.argv[1] == "steps":
    CASES = [(64, "plain", 0), (128, "plain", 0), (256, "plain", 0)]
import paper_2507_07788_b200._device as _d  # noqa: E402
for banded in (0, 1):
    _d.ctx().lib.cqr_debug_factor_banded(banded)
    print(json.dumps({"banded": banded}))
    for k, pol, q in CASES:
        run(k, pol, q)
