"""Per-band timeline of the band-cluster factor (group 0, last attempt):
globaltimer stamps per band relative to band 0's start (us), plus the
single-CTA phase counters of band 0 (per-step cycles) and the power
iteration count of the last estimate."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200._device import ctx  # noqa: E402
from paper_2507_07788_b200._engine import Engine  # noqa: E402
from tools.diag.cluster_ab import POL, gramian  # noqa: E402

EV = ["start", "loaded", "upstream_in", "updated", "factored", "published", "agreed"]


def timeline(k, policy, kind):
    cx = ctx()
    cx.lib.cqr_debug_factor_cluster(1)
    eng = Engine(k, cq.AlgoConfig())
    g = torch.from_numpy(gramian(k, kind, 1)).to(cx.device)
    for _ in range(3):
        eng.G.copy_(g)
        st = eng.factor(POL[policy], 10 ** 6, k)
    buf = (ctypes.c_ulonglong * 64)()
    cx.lib.cqr_debug_factor_cluster_profile(buf)
    fp = (ctypes.c_ulonglong * 16)()
    cx.lib.cqr_debug_factor_profile(fp)
    C = (k + 31) // 32
    t0 = buf[0]
    bands = []
    for r in range(C):
        row = {}
        for e, name in enumerate(EV):
            v = buf[8 * r + e]
            row[name] = round((v - t0) / 1e3, 2) if v >= t0 and v - t0 < 10 ** 7 else None
        bands.append(row)
    steps = max(int(fp[11]), 1)
    # kernel-level phases (rank 0 of group 0): start, X/err done, attempt start (band 0), status write
    kphase = {"xerr_us": round((fp[1] - fp[0]) / 1e3, 2), "to_attempt_us": round((buf[0] - fp[0]) / 1e3, 2),
              "attempt_us": round((buf[8 * 0 + 6] - buf[0]) / 1e3, 2),
              "tail_us": round((fp[6] - buf[6]) / 1e3, 2) if fp[6] > buf[6] else None}
    print(json.dumps({"k": k, "policy": policy, "kind": kind, "code": st.code, "est_iters": int(fp[8]),
                      "band0_steps": int(fp[11]), "panel_cyc": fp[9] // steps, "update_cyc": fp[10] // steps,
                      "diag_cyc": fp[12] // steps, "finish_cyc": {"racc": fp[13], "inv_diag": fp[14], "rinv": fp[15]},
                      "kphase": kphase, "bands": bands}), flush=True)


if __name__ == "__main__" and len(sys.argv) == 1:
    for k, pol, kind in ((256, "plain", "spd"), (256, "shift_once", "illcond"), (192, "plain", "spd"),
                         (160, "plain", "spd")):
        timeline(k, pol, kind)


def steps(k, policy, kind, cta):
    """clock64 stamps of the first 4 blocked steps of CTA `cta` (cycles from each step's start)."""
    cx = ctx()
    cx.lib.cqr_debug_factor_cluster(1)
    cx.lib.cqr_debug_factor_step_profile(cta, None)
    eng = Engine(k, cq.AlgoConfig())
    g = torch.from_numpy(gramian(k, kind, 1)).to(cx.device)
    for _ in range(3):
        eng.G.copy_(g)
        eng.factor(POL[policy], 10 ** 6, k)
    out = (ctypes.c_longlong * 32)()
    cx.lib.cqr_debug_factor_step_profile(cta, ctypes.cast(out, ctypes.c_void_p))
    cx.lib.cqr_debug_factor_step_profile(-1, None)
    names = ["start", "w0_solved", "w0_updated", "w0_diag", "wk_panel", "wk_update", "barrier", "diag_load"]
    for P in range(4):
        row = [out[8 * P + i] for i in range(8)]
        rec = {n: row[i] - row[0] for i, n in enumerate(names[:7])}
        rec["diag_load"] = row[7]
        print(json.dumps({"k": k, "cta": cta, "step": P, **rec}))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "steps":
    for cta in (0, 4, 7):
        steps(256, "plain", "spd", cta)
