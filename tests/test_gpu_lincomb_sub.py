"""Skinny general products on the device (GPU only): `cqr_lincomb_sub`
(Y = Yin - X C, the update iteration's projection and axpy in one pass,
reference algorithms.py:442-444) against lincomb followed by axpy, bit for
bit, and the narrow-tile instances of the row-panel GEMM (<= 16 and <= 32
output columns) against the full-tile instance on a zero-padded C."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _arrays(m, k, n, seed):
    import torch

    import paper_2507_07788_b200 as cq
    from paper_2507_07788_b200._device import ctx

    rng = np.random.default_rng(seed)
    x = rng.standard_normal((m, k))
    c = rng.standard_normal((k, n))
    y = rng.standard_normal((m, n))
    cdev = torch.from_numpy(np.ascontiguousarray(c.T)).to(ctx().device)   # column-major k x n as torch (n, k)
    return cq, x, c, y, cdev


@pytest.mark.parametrize("k,n", [(16, 16), (40, 5), (128, 32), (224, 32), (64, 48), (128, 64), (130, 100), (256, 128),
                                 (33, 17)])
def test_lincomb_sub_equals_lincomb_then_axpy_bitwise(k, n):
    from paper_2507_07788_b200.algorithms import _lincomb_device

    m = 5003                      # ragged: not a multiple of the 64-row tile
    cq, x, c, y, cdev = _arrays(m, k, n, seed=k + n)
    xa = cq.CudaVectorArray.from_numpy(x)
    ya = cq.CudaVectorArray.from_numpy(y)
    proj = _lincomb_device(xa, cdev, k, n)
    want = ya.copy()
    want.axpy(-1.0, proj)
    got = _lincomb_device(xa, cdev, k, n, minus_from=ya)
    np.testing.assert_array_equal(got.to_numpy(), want.to_numpy())
    np.testing.assert_array_equal(ya.to_numpy(), y)          # the source block is untouched
    ref = y - x @ c
    assert np.max(np.abs(got.to_numpy() - ref)) <= 1e-13 * max(1.0, np.abs(ref).max()) * k


@pytest.mark.parametrize("k,n", [(128, 32), (96, 24), (200, 16), (64, 9), (32, 1)])
def test_narrow_tiles_equal_full_tile_bitwise(k, n):
    """n <= 32 runs the 2-block (n <= 16: 1-block) instance; the same product
    with C zero-padded to 40 columns runs the full-tile instance."""
    from paper_2507_07788_b200.algorithms import _lincomb_device
    import torch

    m = 3001
    cq, x, c, _, cdev = _arrays(m, k, n, seed=7 * k + n)
    xa = cq.CudaVectorArray.from_numpy(x)
    narrow = _lincomb_device(xa, cdev, k, n).to_numpy()
    cpad = torch.zeros((40, k), dtype=torch.float64, device=cdev.device)
    cpad[:n] = cdev
    wide = _lincomb_device(xa, cpad, k, 40).to_numpy()
    np.testing.assert_array_equal(narrow, wide[:, :n])
    assert np.all(wide[:, n:] == 0.0)


def test_lincomb_sub_in_place_alias():
    """Y may alias Yin (cqr.h): each element is read, then written, by one thread."""
    from paper_2507_07788_b200 import _lib
    from paper_2507_07788_b200._device import ctx
    from paper_2507_07788_b200.varray import coeff_tiles

    m, k, n = 4000, 96, 32
    cq, x, c, y, cdev = _arrays(m, k, n, seed=3)
    xa = cq.CudaVectorArray.from_numpy(x)
    ya = cq.CudaVectorArray.from_numpy(y)
    want = ya.copy()
    from paper_2507_07788_b200.algorithms import _lincomb_device

    want = _lincomb_device(xa, cdev, k, n, minus_from=ya).to_numpy()
    cx = ctx()
    tiles = coeff_tiles(cdev, k, n, k)
    _lib.check(cx.lib.cqr_lincomb_sub(xa.ptr(), xa.ld, xa.m_local, k, tiles.data_ptr(), n, ya.ptr(), ya.ld, ya.ptr(),
                                      ya.ld, cx.stream), "lincomb_sub")
    np.testing.assert_array_equal(ya.to_numpy(), want)


@pytest.mark.parametrize("ka,kb", [(8, 32), (64, 32), (100, 24), (224, 32), (130, 1), (64, 16), (96, 33), (40, 64)])
def test_skinny_cross_gram_matches_numpy(ka, kb):
    """A^T B with a right operand of at most 32 columns takes the warp-pair k
    split of the cross-Gram kernel (wider ones the 2 x 2 sub-tile map): both
    against NumPy, and deterministic run to run."""
    import paper_2507_07788_b200 as cq
    from paper_2507_07788_b200._engine import cross_gram_host

    m = 7001                      # ragged: not a multiple of the 32-row stage
    rng = np.random.default_rng(ka * 100 + kb)
    a = rng.standard_normal((m, ka))
    b = rng.standard_normal((m, kb))
    aa, bb = cq.CudaVectorArray.from_numpy(a), cq.CudaVectorArray.from_numpy(b)
    g1 = cross_gram_host(aa, bb)
    g2 = cross_gram_host(aa, bb)
    np.testing.assert_array_equal(g1, g2)
    ref = a.T @ b
    assert g1.shape == ref.shape
    assert np.max(np.abs(g1 - ref)) <= 1e-13 * m
