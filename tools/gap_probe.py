"""GPU idle time inside one rs_chol_qr call at config 3's construction: a
torch.profiler kernel timeline of one timed call, the gaps between
consecutive kernels, and where the largest ones sit.

    python tools/gap_probe.py [--m 2000000] [--k 256] [--cond 15]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200.workloads import device_svd_matrix  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=2_000_000)
    ap.add_argument("--k", type=int, default=256)
    ap.add_argument("--cond", type=float, default=15.0)
    ap.add_argument("--algo", default="rs_chol_qr")
    a = ap.parse_args()
    space = cq.VectorSpace(a.m)

    def from_global(x_full):
        return cq.CudaVectorArray.from_device_colmajor(space, x_full.T)

    x = device_svd_matrix(from_global, a.m, a.k, a.cond, 20250, u_from="cholqr2")
    algo = getattr(cq, a.algo)
    for _ in range(3):
        algo(x)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(4):
            algo(x)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    # calls 2-4 (back to back, as in bench.py's timed loop)
    n_per = len(ev) // 4
    ev = ev[n_per:]
    busy = sum(e.time_range.end - e.time_range.start for e in ev)
    span = ev[-1].time_range.end - ev[0].time_range.start
    gl = []
    for i in range(len(ev) - 1):
        g = ev[i + 1].time_range.start - ev[i].time_range.end
        gl.append((g, ev[i].name[:40], ev[i + 1].name[:40]))
    gl.sort(reverse=True)
    out = {"kernels": len(ev), "span_us": span, "busy_us": busy, "idle_us": span - busy,
           "largest_gaps_us": [(round(g, 1), x, y) for g, x, y in gl[:12]],
           "sum_gaps_under_10us": round(sum(g for g, _, _ in gl if g < 10), 1)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
