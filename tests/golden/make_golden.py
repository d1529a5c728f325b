"""Generate golden vectors from the reference implementation itself.

Run in the build container (where `/root/reference` exists):

    python tests/golden/make_golden.py

It imports the UNMODIFIED reference package from `/root/reference/pkg/src`
and records, for small seeded inputs taken from the reference's own test
suite (`pkg/tests/*.py`), the inputs and the reference's outputs (R, shift
decisions, iteration counts, orthogonality/residual metrics, exception
fields).  The fixtures are committed; the GPU box never reads the reference.
"""

from __future__ import annotations

import json
import math
import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import cholqr  # noqa: E402  (the reference)
    return cholqr


def _block(c, m, n, x, seed):
    a, _ = c.generate(c.MatrixSpec(m, n, float(x), seed=seed))
    return c.to_dense_block(a)


def _metrics(c, a_block, res):
    a = c.DenseVectorArray.from_numpy(a_block)
    return (
        c.loss_of_orthogonality(res.q, norm="frobenius"),
        c.reconstruction_residual(a, res.q, res.r, norm="frobenius"),
    )


def main():
    c = _ref()
    cases = []
    arrays = {}

    def add(name, algo, inp, res=None, exc=None, extra=None, cfg=None, spec=None):
        rec = {"name": name, "algo": algo, "cfg": cfg or {}}
        if spec is None:
            arrays[f"{name}__in"] = inp
        else:
            # rebuilt from the (pinned) matgen restatement: [m, n, log10_cond, seed, zero_cols]
            rec["spec"] = spec
        if exc is not None:
            rec["exception"] = type(exc).__name__
            for f in ("pivot_index", "pivot_value", "attempts", "last_shift"):
                if hasattr(exc, f):
                    v = getattr(exc, f)
                    rec[f] = float(v) if isinstance(v, float) else v
        if res is not None:
            arrays[f"{name}__r"] = np.asarray(res.r)
            rec.update(
                iterations=res.iterations,
                shifts=[float(s) for s in res.shifts_applied],
                attempts=list(res.shift_attempts),
                success=bool(res.success),
                orth_error=None if res.orth_error is None else float(res.orth_error),
            )
        if extra:
            rec.update(extra)
        cases.append(rec)

    # --- single-input routines (test_algorithms.py, test_acceptance.py:92-131)
    ladder = [(300, 10, x, s) for x in range(0, 21, 2) for s in (0, 1)]
    for (m, n, x, s) in ladder:
        blk = _block(c, m, n, x, s)
        a = c.DenseVectorArray.from_numpy(blk)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = c.rs_chol_qr(a)
        loo, rrr = _metrics(c, blk, res)
        sp = [m, n, x, s, []]
        add(f"rs_{m}x{n}_c{x}_s{s}", "rs_chol_qr", blk, res, extra={"loo": loo, "rrr": rrr}, spec=sp)
        if x <= 14:
            try:
                res = c.is_chol_qr(a)
                loo, rrr = _metrics(c, blk, res)
                add(f"is_{m}x{n}_c{x}_s{s}", "is_chol_qr", blk, res, extra={"loo": loo, "rrr": rrr}, spec=sp)
            except c.CholeskyBreakdown as e:
                add(f"is_{m}x{n}_c{x}_s{s}", "is_chol_qr", blk, exc=e, spec=sp)
            try:
                res = c.s_chol_qr3(a)
                loo, rrr = _metrics(c, blk, res)
                add(f"s3_{m}x{n}_c{x}_s{s}", "s_chol_qr3", blk, res, extra={"loo": loo, "rrr": rrr}, spec=sp)
            except c.CholeskyBreakdown as e:
                add(f"s3_{m}x{n}_c{x}_s{s}", "s_chol_qr3", blk, exc=e, spec=sp)
        for algo, fn in (("chol_qr", c.chol_qr), ("chol_qr2", c.chol_qr2)):
            try:
                res = fn(a)
                loo, rrr = _metrics(c, blk, res)
                add(f"{algo}_{m}x{n}_c{x}_s{s}", algo, blk, res, extra={"loo": loo, "rrr": rrr}, spec=sp)
            except c.CholeskyBreakdown as e:
                add(f"{algo}_{m}x{n}_c{x}_s{s}", algo, blk, exc=e, spec=sp)

    # larger well/ill-conditioned shapes with k a multiple of the GPU tiles
    for (m, n, x, s) in [(2000, 64, 12, 0), (3000, 128, 8, 1), (1500, 33, 15, 2), (4000, 96, 16, 3)]:
        blk = _block(c, m, n, x, s)
        a = c.DenseVectorArray.from_numpy(blk)
        res = c.rs_chol_qr(a)
        loo, rrr = _metrics(c, blk, res)
        sp = [m, n, x, s, []]
        add(f"rs_{m}x{n}_c{x}_s{s}", "rs_chol_qr", blk, res, extra={"loo": loo, "rrr": rrr}, spec=sp)
        try:
            res = c.s_chol_qr3(a)
            loo, rrr = _metrics(c, blk, res)
            add(f"s3_{m}x{n}_c{x}_s{s}", "s_chol_qr3", blk, res, extra={"loo": loo, "rrr": rrr}, spec=sp)
        except c.CholeskyBreakdown as e:
            add(f"s3_{m}x{n}_c{x}_s{s}", "s_chol_qr3", blk, exc=e, spec=sp)

    # zero column: every iteration retries once, capped (test_algorithms.py:153-164)
    blk = _block(c, 150, 6, 1.0, 4)
    blk[:, 2] = 0.0
    res = c.rs_chol_qr(c.DenseVectorArray.from_numpy(blk), c.AlgoConfig(max_iter=4))
    add("rs_zero_col_cap4", "rs_chol_qr", blk, res, cfg={"max_iter": 4}, spec=[150, 6, 1.0, 4, [2]])
    blk = _block(c, 80, 6, 2.0, 1)
    blk[:, 3] = 0.0
    res = c.rs_chol_qr(c.DenseVectorArray.from_numpy(blk))
    add("rs_zero_col_default", "rs_chol_qr", blk, res, spec=[80, 6, 2.0, 1, [3]])
    # scaled orthogonal columns (test_acceptance.py:356-368)
    q0 = np.linalg.qr(np.random.default_rng(7).normal(size=(200, 12)))[0]
    res = c.rs_chol_qr(c.DenseVectorArray.from_numpy(2.0 * q0))
    add("rs_scaled_orth", "rs_chol_qr", 2.0 * q0, res)
    # single column
    blk = _block(c, 50, 1, 0.0, 0)
    res = c.rs_chol_qr(c.DenseVectorArray.from_numpy(blk))
    add("rs_single_col", "rs_chol_qr", blk, res, spec=[50, 1, 0.0, 0, []])
    # tol_policy roundoff runs to the cap (test_algorithms.py:180-192)
    blk = _block(c, 200, 8, 2.0, 5)
    res = c.rs_chol_qr(c.DenseVectorArray.from_numpy(blk), c.AlgoConfig(tol_policy="roundoff"))
    add("rs_roundoff_policy", "rs_chol_qr", blk, res, cfg={"tol_policy": "roundoff"}, spec=[200, 8, 2.0, 5, []])

    # --- update path (test_update_panel.py)
    def upd(name, qin, rin, anew, cfg=None, cfgd=None):
        a_in = c.DenseVectorArray.from_numpy(qin) if qin.shape[1] else c.DenseVectorArray.zeros(
            c.VectorSpace(anew.shape[0]), 0)
        arrays[f"{name}__qin"] = qin
        arrays[f"{name}__rin"] = rin
        try:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                res = c.chol_qr_update(a_in, rin, c.DenseVectorArray.from_numpy(anew), cfg)
            loo = c.loss_of_orthogonality(res.q, norm="frobenius")
            add(name, "chol_qr_update", anew, res, cfg=cfgd, extra={"loo": loo})
        except (c.ShiftAttemptLimitError, c.CholeskyBreakdown) as e:
            add(name, "chol_qr_update", anew, exc=e, cfg=cfgd)

    base = c.rs_chol_qr(c.generate(c.MatrixSpec(400, 6, 2.0, seed=0))[0])
    inc = _block(c, 400, 4, 3.0, 2)
    upd("upd_extend", c.to_dense_block(base.q), base.r, inc)
    base = c.rs_chol_qr(c.generate(c.MatrixSpec(2000, 5, 2.0, seed=0))[0])
    upd("upd_duplicate", c.to_dense_block(base.q), base.r, c.to_dense_block(base.q)[:, [0]].copy())
    blk = _block(c, 300, 7, 6.0, 1)
    upd("upd_empty", np.zeros((300, 0)), np.zeros((0, 0)), blk)
    blk = _block(c, 300, 4, 1.0, 3)
    blk[:, 1] = 0.0
    upd("upd_width_existing", np.zeros((300, 0)), np.zeros((0, 0)), blk,
        c.AlgoConfig(max_iter=1, update_shift_width="existing"),
        {"max_iter": 1, "update_shift_width": "existing"})
    upd("upd_width_incoming", np.zeros((300, 0)), np.zeros((0, 0)), blk,
        c.AlgoConfig(max_iter=1, update_shift_width="incoming"),
        {"max_iter": 1, "update_shift_width": "incoming"})
    upd("upd_shift_limit", 2.0 * np.eye(4, 1), 2.0 * np.eye(1), np.eye(4, 1),
        c.AlgoConfig(max_shift_attempts=5), {"max_shift_attempts": 5})
    nanblk = _block(c, 100, 3, 1.0, 7)
    nanblk[0, 1] = np.nan
    upd("upd_nan", np.zeros((100, 0)), np.zeros((0, 0)), nanblk,
        c.AlgoConfig(max_shift_attempts=3), {"max_shift_attempts": 3})
    # a multi-block append chain in the config-4 style (scaled): basis of 16,
    # blocks Q_prev C + 1e-8 G
    rng = np.random.default_rng(44)
    m = 1000
    q0 = np.linalg.qr(rng.standard_normal((m, 16)))[0]
    res = c.rs_chol_qr(c.DenseVectorArray.from_numpy(q0))
    qcur, rcur = c.to_dense_block(res.q), res.r
    for j in range(1, 4):
        anew = qcur @ rng.standard_normal((qcur.shape[1], 16)) + 1e-8 * rng.standard_normal((m, 16))
        name = f"upd_chain{j}"
        upd(name, qcur, rcur, anew)
        r = c.chol_qr_update(c.DenseVectorArray.from_numpy(qcur), rcur, c.DenseVectorArray.from_numpy(anew))
        qcur, rcur = c.to_dense_block(r.q), r.r

    # --- panel scheme (test_update_panel.py:115-162): Alg. 3 as a fold of the update
    def pn(name, blk, r_panels, cfg=None, cfgd=None, spec=None):
        rec_extra = {"r_panels": r_panels}
        try:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                res = c.pn_chol_qr(c.DenseVectorArray.from_numpy(blk), r_panels, cfg)
            loo, rrr = _metrics(c, blk, res)
            rec_extra.update(loo=loo, rrr=rrr,
                             panel_profiles=[None if p is None else [p.outer, list(p.shift_attempts)]
                                             for p in res.panel_profiles])
            add(name, "pn_chol_qr", blk, res, cfg=cfgd, extra=rec_extra, spec=spec)
        except (c.ShiftAttemptLimitError, c.CholeskyBreakdown) as e:
            rec_extra["panel_index"] = getattr(e, "panel_index", None)
            add(name, "pn_chol_qr", blk, exc=e, cfg=cfgd, extra=rec_extra, spec=spec)

    for rp in (1, 2, 3, 5, 10):
        pn(f"pn_500x10_c10_s5_r{rp}", _block(c, 500, 10, 10.0, 5), rp, spec=[500, 10, 10.0, 5, []])
    for rp in (2, 4):
        pn(f"pn_2000x64_c12_s0_r{rp}", _block(c, 2000, 64, 12.0, 0), rp, spec=[2000, 64, 12.0, 0, []])
    blk = _block(c, 300, 8, 2.0, 6)
    blk[:, 1] = 0.0
    pn("pn_capped_panel", blk, 2, c.AlgoConfig(max_iter=3, update_shift_width="incoming"),
       {"max_iter": 3, "update_shift_width": "incoming"}, spec=[300, 8, 2.0, 6, [1]])
    blk = _block(c, 100, 6, 1.0, 7)
    blk[0, 4] = np.nan
    pn("pn_nan_panel", blk, 2, c.AlgoConfig(max_shift_attempts=3), {"max_shift_attempts": 3})

    # --- k x k kernels (test_kernels.py)
    kern = {}
    kern["chol_4252"] = c.cholesky(np.array([[4.0, 2.0], [2.0, 5.0]])).tolist()
    try:
        c.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    except c.CholeskyBreakdown as e:
        kern["chol_1221"] = [e.pivot_index, e.pivot_value]
    kern["shift_300_10_1"] = c.compute_shift(300, 10, 1.0)
    kern["shift_clamp"] = c.compute_shift(300, 10, 0.0)
    g = np.random.default_rng(1).normal(size=(8, 8))
    spd = g @ g.T + 8 * np.eye(8)
    arrays["kern_spd8"] = spd
    arrays["kern_spd8_chol"] = c.cholesky(spd)
    arrays["kern_spd8_inv"] = c.tri_inverse(c.cholesky(spd))
    kern["spd8_est"] = c.spectral_norm_estimate(spd)
    # matgen pin
    arrays["matgen_300_10_c6_s0"] = _block(c, 300, 10, 6.0, 0)
    arrays["matgen_50_1_c0_s0"] = _block(c, 50, 1, 0.0, 0)

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump({"cases": cases, "kernels": kern,
                   "numpy": np.__version__}, fh, indent=1, sort_keys=True,
                  default=lambda v: None if (isinstance(v, float) and math.isnan(v)) else v)
    print(f"{len(cases)} cases, {len(arrays)} arrays")


if __name__ == "__main__":
    main()
