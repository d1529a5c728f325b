"""A/B of the k x k stage: the band-cluster path (128 < k <= 256, one CTA per
32-row band) against the single-CTA path, on the same Gramians.

Part 1 compares the outcome of every policy (status fields, shifts, Rk, R^-1
tiles, Racc) for several k, including plain breakdowns that go through the
speculative RECOMPUTE launch.  Part 2 times back-to-back calls (CUDA events)
and the kernels of one call (torch.profiler).  One JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_07788_b200 as cq  # noqa: E402
from paper_2507_07788_b200 import _lib  # noqa: E402
from paper_2507_07788_b200._device import ctx  # noqa: E402
from paper_2507_07788_b200._engine import Engine  # noqa: E402

POL = {"plain": _lib.POLICY_PLAIN, "recompute": _lib.POLICY_RECOMPUTE, "shift_once": _lib.POLICY_SHIFT_ONCE,
       "update": _lib.POLICY_UPDATE, "fixed": _lib.POLICY_FIXED_SHIFT, "estimate": _lib.POLICY_ESTIMATE}
FIELDS = ("code", "retries", "n_shifts", "pivot_index", "est_calls", "est_flag", "escalations", "singular_index")


def gramian(k, kind, seed):
    rng = np.random.default_rng(seed)
    if kind == "spd":
        a = rng.standard_normal((4 * k, k))
        return a.T @ a
    q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    if kind == "illcond":           # kappa(G) = 1e30: the plain attempt breaks down late
        lam = np.logspace(0, -30, k)
    elif kind == "indef":           # one negative eigenvalue: breakdown at a rounding-level pivot
        lam = np.logspace(0, -8, k)
        lam[-1] = -1e-9
    elif kind == "zerocol":
        a = rng.standard_normal((4 * k, k))
        a[:, k // 2] = 0.0
        return a.T @ a
    else:
        raise ValueError(kind)
    g = (q * lam) @ q.T
    return 0.5 * (g + g.T)


CLUSTER_ON = int(os.environ.get("CQR_CLUSTER_MODE", "1"))


def one(k, policy, kind, seed, cluster, q=0):
    cx = ctx()
    cx.lib.cqr_debug_factor_cluster(CLUSTER_ON if cluster else 0)
    eng = Engine(k, cq.AlgoConfig(), q=q)
    g = torch.from_numpy(gramian(k, kind, seed)).to(cx.device)
    eng.G.copy_(g)
    if q:
        eng.Bt.copy_(1e-3 * torch.randn(eng.Bt.shape, dtype=torch.float64, generator=torch.Generator().manual_seed(seed)).to(cx.device))
    kw = dict(update_b=True) if policy == "update" else {}
    if policy == "fixed":
        kw["fixed_shift"] = 1e-10
    st = eng.factor(POL[policy], 10 ** 6, k, **kw)
    torch.cuda.synchronize()
    return st, eng.Rk[:, :k].clone(), eng.Rinv.clone(), eng.Racc[:, :k].clone()


def compare(k, policy, kind, seed, q=0):
    a = one(k, policy, kind, seed, 1, q)
    b = one(k, policy, kind, seed, 0, q)
    sa, sb = a[0], b[0]
    rec = {"k": k, "policy": policy, "kind": kind, "seed": seed,
           "fields_equal": all(getattr(sa, f) == getattr(sb, f) for f in FIELDS),
           "cluster": {f: getattr(sa, f) for f in FIELDS}, "single": {f: getattr(sb, f) for f in FIELDS},
           "shifts_rel": max([abs(x / y - 1) for x, y in zip(sa.shifts, sb.shifts)] or [0.0]),
           "n_shifts": (len(sa.shifts), len(sb.shifts)),
           "margin": (sa.plain_margin, sb.plain_margin)}
    if sa.code == 0 and sb.code == 0:
        scale = float(b[1].abs().max())
        rec["rk_rel"] = float((a[1] - b[1]).abs().max()) / scale
        rec["rk_bitwise"] = bool(torch.equal(a[1], b[1]))
        rec["rinv_rel"] = float((a[2] - b[2]).abs().max()) / float(b[2].abs().max())
        rec["racc_rel"] = float((a[3] - b[3]).abs().max()) / float(b[3].abs().max())
        rec["lower_zero"] = bool(torch.all(torch.tril(a[1], -1) == 0))
    rec["ok"] = rec["fields_equal"] and rec.get("rk_rel", 0.0) < 1e-12 and rec["shifts_rel"] < 1e-9
    print(json.dumps(rec), flush=True)
    return rec["ok"]


def timing(k, policy, kind, n=20):
    from torch.profiler import ProfilerActivity, profile
    out = {"k": k, "policy": policy, "kind": kind}
    for cluster in (0, 1):
        cx = ctx()
        cx.lib.cqr_debug_factor_cluster(CLUSTER_ON if cluster else 0)
        eng = Engine(k, cq.AlgoConfig())
        g = torch.from_numpy(gramian(k, kind, 1)).to(cx.device)
        for _ in range(3):
            eng.G.copy_(g)
            eng.factor(POL[policy], 10 ** 6, k)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record()
        hs = []
        for _ in range(n):
            eng.G.copy_(g)
            hs.append(eng.factor_async(POL[policy], 10 ** 6, k))
            if len(hs) == 4:
                eng.collect(hs)
                hs = []
        t1.record()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(4):
                eng.G.copy_(g)
                eng.factor(POL[policy], 10 ** 6, k)
            torch.cuda.synchronize()
        per = {}
        for e in prof.events():
            if e.device_type != torch.autograd.DeviceType.CUDA:
                continue
            nm = e.name.split("(")[0].replace("void ", "")[:32]
            per.setdefault(nm, []).append(e.time_range.end - e.time_range.start)
        out["cluster" if cluster else "single"] = {
            "call_us": round(t0.elapsed_time(t1) * 1e3 / n, 1),
            "kernels_us": {nm: round(float(np.mean(v)), 1) for nm, v in per.items()}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    bad = 0
    KS = (72, 96, 100, 128) if CLUSTER_ON == 2 else (129, 136, 160, 200, 224, 255, 256)
    for k in KS:
        for policy, kind in (("plain", "spd"), ("plain", "illcond"), ("plain", "zerocol"), ("recompute", "spd"),
                             ("recompute", "illcond"), ("recompute", "indef"), ("shift_once", "illcond"),
                             ("fixed", "illcond"), ("estimate", "spd")):
            for seed in (1, 2):
                bad += not compare(k, policy, kind, seed)
    for k in ((96, 128) if CLUSTER_ON == 2 else (160, 256)):
        bad += not compare(k, "update", "illcond", 3, q=24)
        bad += not compare(k, "update", "spd", 3, q=24)
    TIMING = (((128, "plain", "spd"), (128, "recompute", "illcond"), (96, "plain", "spd"), (128, "shift_once", "illcond"),
               (72, "plain", "spd")) if CLUSTER_ON == 2 else
              ((256, "plain", "spd"), (256, "recompute", "spd"), (256, "recompute", "illcond"),
               (256, "shift_once", "illcond"), (192, "plain", "spd"), (160, "recompute", "illcond")))
    for k, policy, kind in TIMING:
        timing(k, policy, kind)
    ctx().lib.cqr_debug_factor_cluster(1)
    print(json.dumps({"mismatches": bad}))
