"""Is the k x k stage slower after a tall pass because its code (and data)
were evicted from L2?  Factor-kernel durations (torch.profiler / CUPTI) for
back-to-back calls (warm), and for calls each preceded by a 512 MB write
(L2 flushed: the instruction fetches of the ~1 MB factor kernel go to HBM).
python tools/diag/factor_cold.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200 import _lib  # noqa: E402
from paper_2507_07788_b200._engine import Engine  # noqa: E402

POL = {"plain": _lib.POLICY_PLAIN, "shift_once": _lib.POLICY_SHIFT_ONCE}
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def run(k, policy, cold, n=8):
    eng = Engine(k, cq.AlgoConfig())
    g = torch.randn((k, k), dtype=torch.float64, device="cuda")
    spd = g @ g.T + k * torch.eye(k, dtype=torch.float64, device="cuda")
    for _ in range(3):
        eng.G.copy_(spd)
        eng.collect([eng.factor_async(POL[policy], 10**6, k)])
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(n):
            if cold:
                flush.fill_(1)
            eng.G.copy_(spd)
            eng.collect([eng.factor_async(POL[policy], 10**6, k)])
        torch.cuda.synchronize()
    per = {}
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA:
            continue
        name = e.name.split("(")[0].replace("void ", "")[:40]
        per.setdefault(name, []).append(e.time_range.end - e.time_range.start)
    return {nm: round(sum(v) / len(v), 2) for nm, v in per.items() if "cqr" in nm}


for k in (16, 64, 128, 256):
    for pol in ("plain", "shift_once"):
        print(json.dumps({"k": k, "policy": pol, "warm": run(k, pol, False), "l2_flushed": run(k, pol, True)}),
              flush=True)
