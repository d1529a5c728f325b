"""Config 4 at reduced rows: per chol_qr_update call, the CUDA-event time
(what bench.py sums) against the GPU time of the kernels inside it, from a
torch.profiler trace of one chain (31 calls, 16 -> 512 columns).
python tools/diag/update_gaps.py [--m 8000000]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200.workloads import device_gaussian  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=8_000_000)
args = ap.parse_args()
m, p, nblk = args.m, 16, 31
space = cq.VectorSpace(m)
g0 = device_gaussian(cq.CudaVectorArray.zeros(space, p), 2025)
base = cq.rs_chol_qr(g0)
q0 = cq.CudaVectorArray.zeros(space, 0, capacity=p * (nblk + 1))
q0.append(base.q)


def chain(prof_marks):
    hgen = np.random.default_rng(2025)
    q, r = q0.copy(), base.r
    q.reserve(p * (nblk + 1))
    ev = []
    for j in range(nblk):
        c = hgen.standard_normal((q.ncols, p))
        a = q.lincomb(c)
        noise = cq.CudaVectorArray.zeros(space, p)
        device_gaussian(noise, int(hgen.integers(1 << 30)))
        a.axpy(1e-8, noise)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        with torch.profiler.record_function(f"upd{j}"):
            res = cq.chol_qr_update(q, r, a)
        e1.record()
        torch.cuda.synchronize()
        ev.append((e0, e1, res.iterations))
        q, r = res.q, res.r
    return ev


chain(None)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    ev = chain(True)
tot_ev = sum(a.elapsed_time(b) for a, b, _ in ev)
# kernels inside each call: GPU events between the call's CPU range start and the next call
cpu_ranges = sorted([e for e in prof.events() if e.name.startswith("upd") and e.device_type == torch.autograd.DeviceType.CPU],
                    key=lambda e: e.time_range.start)
gpu = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
per = {}
calls = []
for i, cr in enumerate(cpu_ranges):
    lo = cr.time_range.start
    hi = cpu_ranges[i + 1].time_range.start if i + 1 < len(cpu_ranges) else float("inf")
    ks = [g for g in gpu if lo <= g.time_range.start < hi and not g.name.startswith("upd")]
    # keep the call's own kernels: from its first libcqr launch to the last before the next call's block generation
    busy = sum(g.time_range.end - g.time_range.start for g in ks if "cqr::" in g.name or "Memcpy" in g.name)
    for g in ks:
        nm = g.name.split("(")[0].replace("void ", "")[:30]
        per.setdefault(nm, 0.0)
        per[nm] += g.time_range.end - g.time_range.start
    calls.append({"j": i, "event_ms": round(ev[i][0].elapsed_time(ev[i][1]), 3), "busy_ms": round(busy / 1e3, 3),
                  "iters": ev[i][2]})
print(json.dumps({"m": m, "event_total_ms": round(tot_ev, 2),
                  "busy_total_ms": round(sum(c["busy_ms"] for c in calls), 2),
                  "kernels_ms": {k: round(v / 1e3, 2) for k, v in sorted(per.items(), key=lambda x: -x[1])},
                  "calls": calls}, indent=0))

# one call's GPU timeline (the 21st): kernels and the idle gaps between them
cr = cpu_ranges[20]
lo = cr.time_range.start
hi = cpu_ranges[21].time_range.start
ks = [g for g in gpu if lo <= g.time_range.start < hi]
t0 = ks[0].time_range.start
prev_end = None
for g in ks:
    gap = (g.time_range.start - prev_end) if prev_end is not None else 0.0
    print(f"{(g.time_range.start - t0) / 1e3:9.3f} ms  +{gap:8.1f} us idle  {(g.time_range.end - g.time_range.start):9.1f} us  {g.name[:60]}")
    prev_end = g.time_range.end
print("cpu range of call 21:", round((cr.time_range.end - cr.time_range.start) / 1e3, 3), "ms")
