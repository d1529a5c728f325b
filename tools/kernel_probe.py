"""Time the individual libcqr kernels on one shape (CUDA events), for ncu
captures and quick per-kernel measurements.

    python tools/kernel_probe.py --m 2000000 --k 256 [--reps 5] [--only gram|apply|factor]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=2_000_000)
    ap.add_argument("--k", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="all")
    ap.add_argument("--shifted", action="store_true", help="factor a rank-deficient Gram (shift path)")
    a = ap.parse_args()
    import paper_2507_07788_b200 as cq
    from paper_2507_07788_b200 import _lib
    from paper_2507_07788_b200._engine import Engine

    m, k = a.m, a.k
    from paper_2507_07788_b200.workloads import device_gaussian

    x = device_gaussian(cq.CudaVectorArray.zeros(cq.VectorSpace(m), k), 1)
    q = cq.CudaVectorArray.zeros(cq.VectorSpace(m), k)
    eng = Engine(k, cq.AlgoConfig())
    eng.gram(x)
    st = eng.factor(_lib.POLICY_PLAIN, m, k)
    assert st.code == _lib.FACTORED, st.code
    out = {"m": m, "k": k}

    def timeit(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    flops = m * k * (k + 1)
    if a.only in ("all", "gram"):
        ms = timeit(lambda: eng.gram(x), a.reps)
        out["gram_ms"] = ms
        out["gram_tfs"] = flops / ms / 1e9
    if a.only in ("all", "apply"):
        ms = timeit(lambda: eng.apply(x, q, with_gram=True), a.reps)
        out["apply_gram_ms"] = ms
        out["apply_gram_tfs"] = 2 * flops / ms / 1e9
        ms = timeit(lambda: eng.apply(x, q, with_gram=False), a.reps)
        out["trmm_ms"] = ms
        out["trmm_tfs"] = flops / ms / 1e9
    if a.only in ("all", "factor"):
        for kk in (64, 128, 256):
            e2 = Engine(kk, cq.AlgoConfig())
            g = torch.randn((kk, kk), dtype=torch.float64, device="cuda")
            spd = g @ g.T + kk * torch.eye(kk, dtype=torch.float64, device="cuda")
            if a.shifted:
                v = torch.randn((kk, kk // 2), dtype=torch.float64, device="cuda")
                spd = v @ v.T
            e2.G.copy_(spd)
            pol = _lib.POLICY_RECOMPUTE
            ms = timeit(lambda: e2.factor(pol, 10**6, kk), a.reps)
            out[f"factor_k{kk}_ms"] = ms
            import ctypes
            buf = (ctypes.c_ulonglong * 16)()
            e2.cx.lib.cqr_debug_factor_profile(buf)
            t0 = buf[0]
            out[f"factor_k{kk}_phases_us"] = [round((buf[i] - t0) / 1e3, 1) if buf[i] >= t0 else None for i in range(7)]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
