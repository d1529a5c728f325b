"""Timeline of bench.py's streamed e2e schedule (config 3): per call, when its
H2D, compute and D2H start and end (CUDA events, ms from the first H2D)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200 import _device  # noqa: E402
from paper_2507_07788_b200.workloads import device_svd_matrix  # noqa: E402

m, k = 2_000_000, 256
cx = _device.ctx()
space = cq.VectorSpace(m)
a = device_svd_matrix(lambda x: cq.CudaVectorArray.from_device_colmajor(space, x.T), m, k, 15.0, 2025, u_from="cholqr2")
host = torch.empty((k, m), dtype=torch.float64, pin_memory=True)
host.copy_(a.to_device_colmajor())
qhost = torch.empty((k, m), dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize()
comp = torch.cuda.current_stream()
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
dev_in = [torch.empty((k, m), dtype=torch.float64, device="cuda") for _ in range(2)]
ev_in = [torch.cuda.Event() for _ in range(2)]


def E():
    return torch.cuda.Event(enable_timing=True)


def run(n):
    marks = []
    held = []
    freed = torch.cuda.Event()
    freed.record(comp)
    t0 = E()
    with torch.cuda.stream(s_in):
        t0.record(s_in)
        dev_in[0].copy_(host, non_blocking=True)
        ev_in[0].record(s_in)
        h_end0 = E()
        h_end0.record(s_in)
    h_ends = [h_end0]
    host_t = []
    for i in range(n):
        b = i & 1
        comp.wait_event(ev_in[b])
        if i + 1 < n:
            with torch.cuda.stream(s_in):
                s_in.wait_event(freed)
                hs = E()
                hs.record(s_in)
                dev_in[b ^ 1].copy_(host, non_blocking=True)
                ev_in[b ^ 1].record(s_in)
                he = E()
                he.record(s_in)
                h_ends.append(he)
        cs = E()
        cs.record(comp)
        arr = cq.CudaVectorArray.from_device_colmajor(space, dev_in[b])
        freed = torch.cuda.Event()
        freed.record(comp)
        th = time.perf_counter()
        r = cq.rs_chol_qr(arr)
        host_t.append(time.perf_counter() - th)
        ce = E()
        ce.record(comp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ce)
            ds = E()
            ds.record(s_out)
            qdev = r.q.to_device_colmajor()
            qhost.copy_(qdev, non_blocking=True)
            de = E()
            de.record(s_out)
        held.append((r, qdev))
        marks.append((cs, ce, ds, de))
    torch.cuda.synchronize()
    for i, (cs, ce, ds, de) in enumerate(marks):
        print(f"call {i}: H2D end {t0.elapsed_time(h_ends[i]):7.1f}  compute {t0.elapsed_time(cs):7.1f}-{t0.elapsed_time(ce):7.1f}"
              f"  D2H {t0.elapsed_time(ds):7.1f}-{t0.elapsed_time(de):7.1f}  host call {host_t[i]*1e3:6.1f} ms")
    print("total", t0.elapsed_time(marks[-1][3]), "per call", t0.elapsed_time(marks[-1][3]) / n)


run(3)
run(6)
