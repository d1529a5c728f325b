import sys
sys.path.insert(0, ".")
import torch
import paper_2507_07788_b200 as cq
from paper_2507_07788_b200 import _lib
from paper_2507_07788_b200._engine import Engine
from paper_2507_07788_b200.workloads import device_gaussian
m, q, init, cap = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3] == "1", int(sys.argv[4])
k = 16
q_in = device_gaussian(cq.CudaVectorArray.zeros(cq.VectorSpace(m), q, capacity=cap or None), 2)
qb = device_gaussian(cq.CudaVectorArray.zeros(cq.VectorSpace(m), k), 3)
eng = Engine(k, cq.AlgoConfig(), q=q)
g = torch.randn((k, k), dtype=torch.float64, device="cuda")
eng.G.copy_(g @ g.T + k * torch.eye(k, dtype=torch.float64, device="cuda"))
assert eng.factor(_lib.POLICY_PLAIN, m, k).code == _lib.FACTORED
eng.update_pass(q_in, qb, initial=init)
torch.cuda.synchronize()
print(m, q, init, cap, "ok")
