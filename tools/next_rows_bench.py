"""Measurement of the SURVEY §8(f) "next" rows on the device: `is_chol_qr` and
`pn_chol_qr` (r = 2 .. 16 panels) on BASELINE config 3's matrix (2,000,000 x 256,
kappa 1e15; seeded, built in HBM), CUDA events, with the work model of each
run's own pass structure and the CPU oracle timed on a bounded row sample.
One JSON line per case (profiles/r02d_next_rows.jsonl).

    python tools/next_rows_bench.py [--m 2000000] [--k 256] [--cond 15] [--cpu-rows 200000]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

FP64_PEAK = 37.2e12   # measured DMMA peak (profiles/r01_fp64_peak.json)
HBM_PEAK = 6.54e12    # MEASURED_PEAKS.json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=2_000_000)
    ap.add_argument("--k", type=int, default=256)
    ap.add_argument("--cond", type=float, default=15.0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--panels", default="2,4,8,16")
    ap.add_argument("--cpu-rows", type=int, default=200_000)
    a = ap.parse_args()
    import paper_2507_07788_b200 as cq
    from paper_2507_07788_b200._device import ctx
    from paper_2507_07788_b200.algorithms import panel_widths
    from paper_2507_07788_b200.workloads import device_svd_matrix, host_svd_matrix

    cx = ctx()
    m, k = a.m, a.k
    space = cq.VectorSpace(m)
    x = device_svd_matrix(lambda full: cq.CudaVectorArray.from_device_colmajor(space, full.T), m, k, a.cond, 2025,
                          u_from="cholqr2")
    torch.cuda.synchronize()

    def timed(fn):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = fn()
            res = None
            res = fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n0 = cx.launches
            e0.record()
            for _ in range(a.steps):
                res = None
                res = fn()
            e1.record()
            torch.cuda.synchronize()
        return res, e0.elapsed_time(e1) / a.steps, (cx.launches - n0) // a.steps

    def quality(res):
        return {"loo_fro": cq.loss_of_orthogonality(res.q, norm="frobenius"),
                "rrr_fro": cq.reconstruction_residual(x, res.q, res.r, norm="frobenius")}

    def cpu(fn_name, *args):
        from oracle import cholqr_oracle as co   # the checker / CPU baseline, as bench.py's cpu_baseline leg

        xs = host_svd_matrix(a.cpu_rows, k, a.cond, 2025, u_from="cholqr2")
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            t0 = time.perf_counter()
            r = getattr(co, fn_name)(xs, *args)
            sec = time.perf_counter() - t0
        return {"value": a.cpu_rows * k / sec, "unit": "rows*cols/s", "cores": os.cpu_count(), "kind": "port",
                "sample": f"oracle {fn_name} on {a.cpu_rows} x {k} rows of the same construction",
                "iterations": r.iterations}

    # ---- is_chol_qr: x passes of TRMM + Gram after the first Gram
    res, ms, launches = timed(lambda: cq.is_chol_qr(x))
    flops = (2 * res.iterations + 1) * m * k * (k + 1.0)
    nbytes = (1 + 3 * res.iterations) * m * k * 8.0        # k > 64: TRMM (read, write) then Gram (read)
    bound = max(flops / FP64_PEAK, nbytes / HBM_PEAK) * 1e3
    print(json.dumps({"algo": "is_chol_qr", "rows": m, "cols": k, "log10_cond": a.cond, "ms": ms,
                      "value": m * k / (ms * 1e-3), "unit": "rows*cols/s", "passes": res.iterations,
                      "shift_attempts": list(res.shift_attempts), "bound_ms": bound, "frac": bound / ms,
                      "gpu_launches": launches, "quality": quality(res), "cpu_baseline": cpu("is_chol_qr")}), flush=True)
    res = None

    # ---- pn_chol_qr: the first panel is rs_chol_qr, every later one a chol_qr_update
    for r_panels in [int(v) for v in a.panels.split(",")]:
        res, ms, launches = timed(lambda: cq.pn_chol_qr(x, r_panels))
        widths = panel_widths(k, r_panels)
        flops = nbytes = 0.0
        q = 0
        for w, prof in zip(widths, res.panel_profiles):
            its = prof.outer                     # iterations of this panel
            # initial pass: Bt = Q_in^T A, G = A^T A; per iteration: projection, TRMM, cross Gram, Gram
            flops += m * (2.0 * q * w + w * (w + 1.0)) + its * m * (4.0 * q * w + 2.0 * w * (w + 1.0))
            nbytes += 8.0 * m * ((q + w) + its * (q + 2.0 * w))
            q += w
        bound = max(flops / FP64_PEAK, nbytes / HBM_PEAK) * 1e3
        print(json.dumps({"algo": "pn_chol_qr", "r_panels": r_panels, "panel_width": widths[0], "rows": m, "cols": k,
                          "log10_cond": a.cond, "ms": ms, "value": m * k / (ms * 1e-3), "unit": "rows*cols/s",
                          "iterations": res.iterations, "per_panel_iterations": [p.outer for p in res.panel_profiles],
                          "shifted_iterations": int(sum(1 for v in res.shift_attempts if v)),
                          "bound_ms": bound, "frac": bound / ms, "gpu_launches": launches,
                          "fused_update_pass": bool(widths[0] <= 16), "quality": quality(res),
                          "cpu_baseline": cpu("pn_chol_qr", r_panels)}), flush=True)
        res = None


if __name__ == "__main__":
    main()
