"""Diagnostic: dump the device's per-pass Gramians of one golden rs case and
replay the oracle's Cholesky on them."""
import sys
import warnings

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import parity as P  # noqa: E402
import paper_2507_07788_b200 as cq  # noqa: E402
from oracle import cholqr_oracle as co  # noqa: E402
from oracle import matgen_oracle as mg  # noqa: E402

m, n, x, s = 300, 10, 16.0, 1
blk = mg.generate(m, n, x, s)
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    res, tr = P.traced(cq.rs_chol_qr, cq.CudaVectorArray.from_numpy(blk))
print("device attempts", res.shift_attempts, "margins", res.decision_margins, "errs", res.err_history)
gs = []
for i, e in enumerate(tr[: res.iterations + 1]):
    g, _ = P._device_x(e)
    raw = e["G"].cpu().numpy()
    gs.append(raw)
    try:
        r = co.cholesky_upper(g)
        print(i, "oracle plain ok, margin", co._margin(g, r))
    except co.OracleBreakdown as exc:
        print(i, "oracle breakdown at", exc.pivot_index, exc.pivot_value, "diag", np.diag(g)[:4], "asym", np.max(np.abs(raw - raw.T)))
np.savez("gpurun_out/diag_replay.npz", *gs)
