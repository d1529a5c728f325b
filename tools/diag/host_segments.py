import os, sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200 import algorithms as al, _engine as en, _lib
from paper_2507_07788_b200.workloads import device_svd_matrix
m, k = 200_000, 64
a = device_svd_matrix(lambda x: cq.CudaVectorArray.from_device_colmajor(cq.VectorSpace(m), x.T), m, k, 12.0, 2025)
for _ in range(20): cq.s_chol_qr3(a)
torch.cuda.synchronize()
T = {}
def tick(name, t0):
    t = time.perf_counter_ns(); T[name] = T.get(name, 0) + (t - t0); return t
N = 200
for _ in range(N):
    t = time.perf_counter_ns()
    cfg = al.AlgoConfig(); aa = al._device_array(a); t = tick('setup', t)
    eng = en.Engine(k, cfg); t = tick('engine', t)
    eng.gram(aa); t = tick('gram', t)
    hs = [eng.factor_async(_lib.POLICY_SHIFT_ONCE, m, k)]; t = tick('factor1', t)
    q = al._fresh_like(aa, k); t = tick('fresh', t)
    eng.apply(aa, q, with_gram=True); t = tick('apply1', t)
    hs.append(eng.factor_async(_lib.POLICY_PLAIN, m, k)); t = tick('factor2', t)
    q = al._apply_gram_into(eng, q, fresh_ok=False); t = tick('apply2', t)
    hs.append(eng.factor_async(_lib.POLICY_PLAIN, m, k)); t = tick('factor3', t)
    al._apply_last(eng, q); t = tick('apply3', t)
    eng.r_prefetch(); t = tick('r_prefetch', t)
    sts = eng.collect(hs); t = tick('collect(wait)', t)
    r = eng.r_host(); t = tick('r_host', t)
    res = al.QRResult(q=q, r=r, iterations=3, shifts_applied=[sts[0].shifts[0]], pivot_margins=[s.min_pivot_rel for s in sts]); t = tick('result', t)
    del eng; t = tick('del_engine', t)
for kk, v in T.items(): print(f"{kk:15s} {v / N / 1e3:8.1f} us")
