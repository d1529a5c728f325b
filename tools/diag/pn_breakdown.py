"""pn_chol_qr on config 3's matrix: summed kernel times by kind (KernelTimer) against the
call's event / wall time.  python tools/diag/pn_breakdown.py [4,8,16] [verbose]"""
import sys, json, warnings
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200 import _device
from paper_2507_07788_b200._device import ctx
from paper_2507_07788_b200.workloads import device_svd_matrix
cx = ctx()
m, k = 2_000_000, 256
PANELS = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [4, 8, 16]
VERBOSE = len(sys.argv) > 2
space = cq.VectorSpace(m)
x = device_svd_matrix(lambda full: cq.CudaVectorArray.from_device_colmajor(space, full.T), m, k, 15.0, 2025, u_from="cholqr2")
for r in PANELS:
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cq.pn_chol_qr(x, r)
        torch.cuda.synchronize()
        cx.timer = _device.KernelTimer()
        res = cq.pn_chol_qr(x, r)
        torch.cuda.synchronize()
        kt = cx.timer.summary()
        cx.timer = None
    print(r, {n: (len(v["ms"]), round(sum(v["ms"]), 3)) for n, v in kt.items()})
    if VERBOSE:
        for n, v in kt.items():
            print(n, [(w, round(t, 3)) for w, t in zip(v["work"], v["ms"])][:40])
# wall/event time of one pn_chol_qr call against the summed kernel time
import time
for r in PANELS:
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        res = cq.pn_chol_qr(x, r)
        e1.record()
        torch.cuda.synchronize()
        print("r", r, "event ms", e0.elapsed_time(e1), "wall ms", (time.perf_counter() - t0) * 1e3)
