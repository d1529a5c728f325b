"""Strong-scaling model from measured per-GPU work.

With one GPU per gpurun call, the N-GPU step is measured as the 1-GPU call on
m/N rows -- the work one rank does -- and the modelled N-GPU step adds one
k x k allreduce per pass (NVLink, ~25 us for 512 KB; an assumption, stated in
the output).  The pass count of the full-size problem is used (a smaller
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3, choices=sorted(ROWS))
    ap.add_argument("--allreduce-us", type=float, default=25.0)
    a = ap.parse_args()
    m = ROWS[a.config]
    full = bench(a.config, m)
    passes = len(full["config"].get("shift_attempts") or []) or full["config"].get("passes", 2)
    t1 = full["ms_per_step"]
    rows = {"config": a.config, "rows": m, "t1_ms": t1, "allreduce_us_assumed": a.allreduce_us, "n": {}}
    for n in (2, 4, 8):
        d = bench(a.config, m // n)
        kt = d["kernels"]
        # per-pass kernel means, scaled to the full-size pass structure
        per_gpu = 0.0
        for name, v in kt.items():
            per_gpu += v["mean_ms"] * full["kernels"][name]["launches_per_step"]
        gaps = max(0.0, t1 - sum(v["mean_ms"] * v["launches_per_step"] for v in full["kernels"].values()))
        tn = per_gpu + gaps + (passes + 1) * a.allreduce_us * 1e-3
        rows["n"][n] = {"per_gpu_ms": round(tn, 3), "efficiency": round(t1 / (n * tn), 3)}
    print(json.dumps(rows))


if __name__ == "__main__":
    main()
