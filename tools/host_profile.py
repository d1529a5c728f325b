"""Host-side profile of one small algorithm call (config 1 shape): where the
time goes outside the kernels.  python tools/host_profile.py"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2507_07788_b200 as cq
from paper_2507_07788_b200.workloads import device_svd_matrix


def main():
    m, k = 200_000, 64
    a = device_svd_matrix(lambda x: cq.CudaVectorArray.from_device_colmajor(cq.VectorSpace(m), x.T), m, k, 12.0, 2025)
    for _ in range(5):
        cq.s_chol_qr3(a)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        cq.s_chol_qr3(a)
    torch.cuda.synchronize()
    print("wall ms per call", (time.perf_counter() - t0) / 20 * 1e3)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(20):
        cq.s_chol_qr3(a)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
