"""Host cost of the pieces of a pooled Engine() and of one Gram launch (us)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200 import _engine as en
from paper_2507_07788_b200._device import ctx, _raw_stream
from paper_2507_07788_b200.workloads import device_svd_matrix
m, k = 200_000, 64
a = device_svd_matrix(lambda x: cq.CudaVectorArray.from_device_colmajor(cq.VectorSpace(m), x.T), m, k, 12.0, 2025)
cfg = cq.AlgoConfig()
for _ in range(20):
    e = en.Engine(k, cfg); e.gram(a); del e
torch.cuda.synchronize()
cx = ctx()
def bench(name, fn, n=2000):
    fn(); t = time.perf_counter_ns()
    for _ in range(n): fn()
    print(f"{name:34s} {(time.perf_counter_ns() - t) / n / 1e3:7.2f} us")
bench("torch.cuda.current_stream(dev)", lambda: torch.cuda.current_stream(cx.device))
bench("raw stream", lambda: _raw_stream(cx.device.index))
ev = torch.cuda.Event(); ev.record()
s = torch.cuda.current_stream(cx.device)
bench("stream.wait_event", lambda: s.wait_event(ev))
e = en.Engine(k, cfg)
bench("Racc.copy_(racc0)", lambda: e.Racc.copy_(e._racc0))
bench("stat_all[0]", lambda: e.stat_all[0])
bench("stat_host_all.numpy()", lambda: e.stat_host_all.numpy())
bench("Event()+record", lambda: torch.cuda.Event().record(s))
def mk():
    x = en.Engine(k, cfg); del x
bench("Engine() + del (pooled)", mk, n=500)
bench("eng.gram(a)", lambda: e.gram(a), n=500)
bench("a.ptr(); a.ld; a.m_local", lambda: (a.ptr(), a.ld, a.m_local))
bench("cqr_gram_workspace_bytes", lambda: cx.lib.cqr_gram_workspace_bytes(a.m_local, k, k, 1))
torch.cuda.synchronize()
