"""Time the individual libcqr kernels on one shape (CUDA events), for ncu
captures and quick per-kernel measurements.

    python tools/kernel_probe.py --m 2000000 --k 256 [--reps 5] [--only gram|apply|factor]
    python tools/kernel_probe.py --only update --m 8000000 --q 256 --k 16   (update pass, basis q, block k)
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
    ap.add_argument("--q", type=int, default=256, help="basis width for --only update")
    ap.add_argument("--fk", default="64,128,256", help="widths for --only factor")
    ap.add_argument("--tma", type=int, default=1, help="update: TMA tensor staging of narrow sub-panels (0/1)")
    ap.add_argument("--initial", action="store_true", help="update: time the initial pass (Bt = Q_in^T Q, G = Q^T Q)")
    ap.add_argument("--cap", type=int, default=0, help="update: column capacity of the basis (config 4's chain: 512)")
    a = ap.parse_args()
    import paper_2507_07788_b200 as cq
    from paper_2507_07788_b200 import _lib
    from paper_2507_07788_b200._engine import Engine

    m, k = a.m, a.k
    from paper_2507_07788_b200.workloads import device_gaussian

    if a.only == "update":
        from paper_2507_07788_b200._device import ctx

        ctx().lib.cqr_debug_update_tma(a.tma)
        q_in = device_gaussian(cq.CudaVectorArray.zeros(cq.VectorSpace(m), a.q, capacity=a.cap or None), 2)
        qb = device_gaussian(cq.CudaVectorArray.zeros(cq.VectorSpace(m), k), 3)
        eng = Engine(k, cq.AlgoConfig(), q=a.q)
        g = torch.randn((k, k), dtype=torch.float64, device="cuda")
        eng.G.copy_(g @ g.T + k * torch.eye(k, dtype=torch.float64, device="cuda"))
        st = eng.factor(_lib.POLICY_PLAIN, m, k)
        assert st.code == _lib.FACTORED, st.code
        eng.Bt.copy_(1e-3 * torch.randn_like(eng.Bt))

        def run():
            eng.update_pass(q_in, qb, initial=a.initial)

        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        flops = 4.0 * m * a.q * k + 2.0 * m * k * (k + 1)
        if a.initial:
            flops = 2.0 * m * a.q * k + 1.0 * m * k * (k + 1)
        print(json.dumps({"m": m, "q": a.q, "p": k, "initial": a.initial, "cap": a.cap, "update_ms": ms, "update_tfs": flops / ms / 1e9,
                          "qin_gbs": m * a.q * 8 / ms / 1e6}))
        return

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
        for kk in [int(v) for v in a.fk.split(",")]:
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
            # back to back on the stream (no host sync per call), as inside a pass loop
            def burst():
                hs = [e2.factor_async(pol, 10**6, kk) for _ in range(e2.nslots)]
                e2.collect(hs)
            out[f"factor_k{kk}_stream_ms"] = timeit(burst, max(1, a.reps // e2.nslots)) / e2.nslots
            import ctypes
            buf = (ctypes.c_ulonglong * 16)()
            e2.cx.lib.cqr_debug_factor_profile(buf)
            t0 = buf[0]
            out[f"factor_k{kk}_phases_us"] = [round((buf[i] - t0) / 1e3, 1) if buf[i] >= t0 else None for i in range(7)]
            out[f"factor_k{kk}_est_iters"] = int(buf[8]) if buf[8] < 1000 else None
            out[f"factor_k{kk}_finish_cycles"] = {"racc": int(buf[13]), "diag_inv": int(buf[14]),
                                                   "backsub_end": int(buf[15])}
            if buf[11]:
                out[f"factor_k{kk}_step_cycles"] = {"steps": int(buf[11]), "solve": int(buf[9] // buf[11]),
                                                    "update": int(buf[10] // buf[11]),
                                                    "diag_warp0": int(buf[12] // buf[11])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
