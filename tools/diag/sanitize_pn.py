"""compute-sanitizer target: pn_chol_qr whose last panel is narrower
than 16 columns inside a basis with capacity - k < 16, i.e. the update pass's
TMA box reaches past the block's last column.  Run as
    compute-sanitizer --tool memcheck python tools/diag/sanitize_pn.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2507_07788_b200 as cq  # noqa: E402

rng = np.random.default_rng(0)
for n, r in ((100, 8), (90, 7), (45, 4)):
    a = cq.CudaVectorArray.from_numpy(rng.standard_normal((5000, n)))
    res = cq.pn_chol_qr(a, r)
    print(n, r, res.success, res.iterations, cq.loss_of_orthogonality(res.q, norm="frobenius"))
