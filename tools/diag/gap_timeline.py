"""GPU busy time and idle gaps of back-to-back calls (torch.profiler / CUPTI):
per call, the sum of kernel durations, the idle time between kernels (and
before which kernel it falls), and the wall time.  Config 1 by default:
python tools/diag/gap_timeline.py [--config 1] [--calls 20]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200.workloads import device_svd_matrix  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--calls", type=int, default=20)
ap.add_argument("--m", type=int, default=200_000)
ap.add_argument("--k", type=int, default=64)
args = ap.parse_args()
m, k = args.m, args.k
a = device_svd_matrix(lambda x: cq.CudaVectorArray.from_device_colmajor(cq.VectorSpace(m), x.T), m, k, 12.0, 2025)
for _ in range(10):
    cq.s_chol_qr3(a)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(args.calls):
    cq.s_chol_qr3(a)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / args.calls * 1e6
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(args.calls):
        cq.s_chol_qr3(a)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
busy = sum(e.time_range.end - e.time_range.start for e in ev)
durs = {}
for i, e in enumerate(ev):
    nm = e.name.split("(")[0].replace("void ", "")[:36]
    durs.setdefault((i % max(1, len(ev) // args.calls), nm), []).append(e.time_range.end - e.time_range.start)
gaps = {}
prev = None
for e in ev:
    if prev is not None:
        gap = e.time_range.start - prev.time_range.end
        nm = e.name.split("(")[0].replace("void ", "")[:36]
        gaps.setdefault(nm, []).append(gap)
    prev = e
span = ev[-1].time_range.end - ev[0].time_range.start
print(json.dumps({"m": m, "k": k, "wall_us_per_call": round(wall, 1),
                  "gpu_busy_us_per_call": round(busy / args.calls, 1),
                  "gpu_span_us_per_call": round(span / args.calls, 1),
                  "kernels_per_call": len(ev) / args.calls,
                  "kernel_us_in_call_order": [[nm, round(sum(v) / len(v), 1)] for (i, nm), v in
                                              sorted(durs.items())],
                  "idle_before_us_per_call": {n: round(sum(v) / args.calls, 1) for n, v in
                                              sorted(gaps.items(), key=lambda x: -sum(x[1]))}}, indent=1))
