"""Host-side cost of one s_chol_qr3 call at config 1 (cProfile, cumulative)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200.workloads import device_svd_matrix  # noqa: E402

m, k = 200_000, 64
a = device_svd_matrix(lambda x: cq.CudaVectorArray.from_device_colmajor(cq.VectorSpace(m), x.T), m, k, 12.0, 2025)
for _ in range(10):
    cq.s_chol_qr3(a)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    cq.s_chol_qr3(a)
torch.cuda.synchronize()
print("wall us per call", (time.perf_counter() - t0) / n * 1e6)
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    cq.s_chol_qr3(a)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
