"""Strong-scaling model from measured per-GPU work.

With one GPU per gpurun call, the N-GPU step is measured as the 1-GPU call on
m/N rows -- the work one rank does -- and the modelled N-GPU step adds one
k x k exchange per pass: an NCCL all-gather of the per-rank partials over
NVLink (~25 us at 512 KB per rank; an assumption, stated in the output) plus
the in-order device sum (cqr_sum_ranks, measured here on N partials).  The pass count of the full-size problem is used (a smaller
matrix of the same construction can take fewer passes).

    python tools/scaling_model.py --config 3 [--allreduce-us 25]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS = {1: 200_000, 2: 4_000_000, 3: 2_000_000, 5: 128_000_000}


def bench(config, rows):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(config), "--rows", str(rows),
                          "--steps", "5", "--warmup", "3", "--no-e2e", "--no-cpu"],
                         cwd=ROOT, capture_output=True, text=True, check=True)
    return json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])


def sum_ranks_us(n, elems, reps=50):
    """CUDA-event time of one in-order device sum of n partials (cqr_sum_ranks)."""
    sys.path.insert(0, ROOT)
    import torch

    from paper_2507_07788_b200._device import ctx

    cx = ctx()
    parts = torch.randn(n * elems, dtype=torch.float64, device=cx.device)
    out = torch.empty(elems, dtype=torch.float64, device=cx.device)
    cx.lib.cqr_sum_ranks(parts.data_ptr(), n, elems, out.data_ptr(), cx.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        cx.lib.cqr_sum_ranks(parts.data_ptr(), n, elems, out.data_ptr(), cx.stream)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3, choices=sorted(ROWS))
    ap.add_argument("--allreduce-us", type=float, default=25.0, help="assumed all-gather latency per pass (us)")
    a = ap.parse_args()
    m = ROWS[a.config]
    full = bench(a.config, m)
    passes = len(full["config"].get("shift_attempts") or []) or full["config"].get("passes", 2)
    t1 = full["ms_per_step"]
    k = full["config"]["cols"]
    rows = {"config": a.config, "rows": m, "t1_ms": t1, "allgather_us_assumed": a.allreduce_us, "n": {}}
    for n in (2, 4, 8):
        sum_us = sum_ranks_us(n, k * k)
        d = bench(a.config, m // n)
        kt = d["kernels"]
        # per-pass kernel means, scaled to the full-size pass structure
        per_gpu = 0.0
        for name, v in kt.items():
            per_gpu += v["mean_ms"] * full["kernels"][name]["launches_per_step"]
        gaps = max(0.0, t1 - sum(v["mean_ms"] * v["launches_per_step"] for v in full["kernels"].values()))
        tn = per_gpu + gaps + (passes + 1) * (a.allreduce_us + sum_us) * 1e-3
        rows["n"][n] = {"per_gpu_ms": round(tn, 3), "efficiency": round(t1 / (n * tn), 3),
                        "factor_ms_per_gpu": round(kt["factor"]["mean_ms"] * full["kernels"]["factor"]["launches_per_step"], 3),
                        "sum_ranks_us": round(sum_us, 2)}
    print(json.dumps(rows))


if __name__ == "__main__":
    main()
