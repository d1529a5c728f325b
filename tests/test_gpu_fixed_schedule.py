"""Native fixed schedules (cqr_fixed_schedule): chol_qr, chol_qr2 and
s_chol_qr3 enqueued by one libcqr call and replayed as CUDA graphs must give
bitwise the results of the per-kernel launches (same kernels, same arguments,
same order), raise the same errors, and reuse one graph per plan.  GPU only.

Reference schedules: /root/reference/pkg/src/cholqr/algorithms.py:201-244."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cq():
    import paper_2507_07788_b200 as cq

    return cq


def _mode(mode):
    from paper_2507_07788_b200 import _engine

    old = _engine.NATIVE_SCHEDULE
    _engine.NATIVE_SCHEDULE = mode
    return old


def _run(algo, a, mode):
    cq = _cq()
    old = _mode(mode)
    try:
        res = getattr(cq, algo)(a)
        return res, res.q.to_numpy()
    finally:
        _mode(old)


def _matrix(m, k, kappa_exp, seed):
    from paper_2507_07788_b200.workloads import host_svd_matrix

    return host_svd_matrix(m, k, kappa_exp, seed=seed)


@pytest.mark.parametrize("algo", ["chol_qr", "chol_qr2", "s_chol_qr3"])
@pytest.mark.parametrize("m,k", [(5003, 16), (40000, 64), (20011, 100), (30000, 128), (12000, 200), (20000, 256)])
def test_native_graph_bitwise_equals_per_kernel_launches(algo, m, k):
    cq = _cq()
    x = _matrix(m, k, 6.0 if algo != "s_chol_qr3" else 12.0, seed=k)
    a = cq.CudaVectorArray.from_numpy(x)
    ref, qref = _run(algo, a, 0)
    for mode in (1, 2, 2):   # native enqueue, graph capture, graph replay
        res, q = _run(algo, a, mode)
        assert np.array_equal(q, qref), (algo, m, k, mode)
        assert np.array_equal(res.r, ref.r), (algo, m, k, mode)
        assert res.iterations == ref.iterations
        assert list(res.shifts_applied) == list(ref.shifts_applied)
        assert res.pivot_margins == ref.pivot_margins


def test_graph_cached_once_per_plan_and_replayed_on_other_streams():
    import torch

    cq = _cq()
    lib = cq._lib.load()
    x = _matrix(30000, 64, 12.0, seed=5)
    a = cq.CudaVectorArray.from_numpy(x)
    first, q0 = _run("s_chol_qr3", a, 2)
    n0 = lib.cqr_fixed_graphs()
    outs = []
    keep = []
    for _ in range(6):
        res, q = _run("s_chol_qr3", a, 2)
        keep.append(res)   # live results: the allocator hands out new Q buffers (new plans)
        outs.append(q)
    n1 = lib.cqr_fixed_graphs()
    assert n1 - n0 <= 6
    del keep
    res, q = _run("s_chol_qr3", a, 2)
    n2 = lib.cqr_fixed_graphs()
    for _ in range(4):   # same buffers again: pure replays, no new capture
        res, q = _run("s_chol_qr3", a, 2)
        outs.append(q)
    assert lib.cqr_fixed_graphs() == n2
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        res, q = _run("s_chol_qr3", a, 2)
        outs.append(q)
    torch.cuda.synchronize()
    for q in outs:
        assert np.array_equal(q, q0)
    assert np.array_equal(res.r, first.r)


@pytest.mark.parametrize("algo", ["chol_qr", "chol_qr2"])
def test_native_breakdown_raises_like_per_kernel_path(algo):
    """A zero column breaks down in pass 1: the native path raises
    the same CholeskyBreakdown (pivot index, value) as the per-kernel path."""
    cq = _cq()
    rng = np.random.default_rng(3)
    x = rng.standard_normal((4000, 32))
    x[:, 7] = 0.0   # zero column: an exactly zero pivot
    a = cq.CudaVectorArray.from_numpy(x)
    errs = []
    for mode in (0, 2, 2):
        old = _mode(mode)
        try:
            with pytest.raises(cq.CholeskyBreakdown) as ei:
                getattr(cq, algo)(a)
            errs.append((ei.value.pivot_index, ei.value.pivot_value, str(ei.value)))
        finally:
            _mode(old)
    assert errs[0] == errs[1] == errs[2]


def test_native_ledger_charges_match():
    cq = _cq()
    x = _matrix(20000, 64, 12.0, seed=9)
    a = cq.CudaVectorArray.from_numpy(x)
    led = []
    for mode in (0, 2):
        old = _mode(mode)
        try:
            ledger = cq.FlopLedger()
            cq.s_chol_qr3(a, ledger=ledger)
            led.append(dict(ledger.counts) if hasattr(ledger, "counts") else repr(ledger))
        finally:
            _mode(old)
    assert led[0] == led[1]
