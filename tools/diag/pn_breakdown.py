import sys, json, warnings
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200 import _device
from paper_2507_07788_b200._device import ctx
from paper_2507_07788_b200.workloads import device_svd_matrix
cx = ctx()
m, k = 2_000_000, 256
space = cq.VectorSpace(m)
x = device_svd_matrix(lambda full: cq.CudaVectorArray.from_device_colmajor(space, full.T), m, k, 15.0, 2025, u_from="cholqr2")
for r in (4, 8):
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
    if r == 8:
        for n, v in kt.items():
            print(n, [(w, round(t, 3)) for w, t in zip(v["work"], v["ms"])][:40])
