"""A few back-to-back factor calls of one shape (for ncu captures):
python tools/diag/factor_one.py K POLICY KIND [CLUSTER]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200._device import ctx  # noqa: E402
from paper_2507_07788_b200._engine import Engine  # noqa: E402
from tools.diag.cluster_ab import POL, gramian  # noqa: E402

k, pol, kind = int(sys.argv[1]), sys.argv[2], sys.argv[3]
cl = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cx = ctx()
cx.lib.cqr_debug_factor_cluster(cl)
eng = Engine(k, cq.AlgoConfig())
g = torch.from_numpy(gramian(k, kind, 1)).to(cx.device)
for _ in range(4):
    eng.G.copy_(g)
    st = eng.factor(POL[pol], 10 ** 6, k)
torch.cuda.synchronize()
print("code", st.code)
