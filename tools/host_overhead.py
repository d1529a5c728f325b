"""Host-side cost of one small call (config 1 shape): Engine construction and a
cProfile of s_chol_qr3.   python tools/host_overhead.py"""
import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200._engine import Engine
from paper_2507_07788_b200.workloads import device_gaussian

a = device_gaussian(cq.CudaVectorArray.zeros(cq.VectorSpace(200_000), 64), 1)
for _ in range(3):
    cq.s_chol_qr3(a)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    Engine(64, cq.AlgoConfig())
torch.cuda.synchronize()
print("Engine() us", (time.perf_counter() - t0) / 20 * 1e6)
t0 = time.perf_counter()
for _ in range(20):
    cq.s_chol_qr3(a)
torch.cuda.synchronize()
print("s_chol_qr3 us", (time.perf_counter() - t0) / 20 * 1e6)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    cq.s_chol_qr3(a)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18)
print(s.getvalue()[:4000])
