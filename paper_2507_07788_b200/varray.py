"""Device-resident tall arrays behind the reference's columns-only interface.

`CudaVectorArray` is the B200 backend of the reference's `VectorArray` ABC
(reference varray.py:47-100): the same members (`space`, `ncols`, `copy`,
`append`, `gramian`, `lincomb`, `axpy`, `remove_columns`, `zeros`,
`from_numpy`, `_iter_columns`, `to_numpy`), the same ownership rules
(copy / lincomb / from_numpy allocate independent storage, append copies its
source, axpy mutates in place, gramian returns a host ndarray) and the same
exceptions (ValueError on space/shape, TypeError on backend mixing,
IndexError on bad column indices).

HBM layout: one fp64 buffer per array, column-major like the reference's
Fortran block (reference varray.py:107): column j of the local row shard is
contiguous, leading dimension ld = round_up(m_local, 16) with zero padding
rows, so every column starts 128-byte aligned for the bulk-copy engine.
Column capacity may exceed ncols, so appends (the update path) do not
reallocate.  Under torch.distributed each rank holds rows
[r m / P, (r+1) m / P) of every array; `space.dim` is always the GLOBAL m.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import ctx, round_up


@dataclass(frozen=True)
class VectorSpace:
    """R^dim, the common habitat of an array's columns (reference varray.py:24-32)."""

    dim: int

    def __post_init__(self):
        if self.dim < 1:
            raise ValueError("space dimension must be >= 1")


def _as_index_list(indices, ncols, who):
    idx = [int(i) for i in indices]
    seen = set()
    for i in idx:
        if not 0 <= i < ncols:
            raise IndexError(f"{who}: column index {i} out of range for {ncols} columns")
        if i in seen:
            raise ValueError(f"{who}: duplicate column index {i}")
        seen.add(i)
    return idx


def upload_coeffs(c, rows_pad=None):
    """Host k x n coefficients -> device buffer with zero-padded rows
    (ld = round_up(k, 32)), the layout libcqr expects for C / R^-1."""
    c = np.asarray(c, dtype=float)
    k, n = c.shape
    ld = rows_pad or max(round_up(k, 32), 32)
    host = np.zeros((n, ld))
    host[:, :k] = c.T
    return torch.from_numpy(host).to(ctx().device, non_blocking=False), ld


class CudaVectorArray:
    """Tall fp64 array on the local B200, columns-only interface."""

    def __init__(self, space, buf, ncols):
        self.space = space
        self._buf = buf          # (capacity, ld) float64, row j = column j
        self._k = int(ncols)

    # ------------------------------------------------------------ construction
    @staticmethod
    def _local_rows(space):
        lo, hi = ctx().row_range(space.dim)
        return lo, hi

    @classmethod
    def _alloc(cls, space, cap, zero=True):
        lo, hi = cls._local_rows(space)
        ld = max(round_up(hi - lo, 16), 16)
        fn = torch.zeros if zero else torch.empty
        return fn((max(cap, 0), ld), dtype=torch.float64, device=ctx().device)

    @classmethod
    def zeros(cls, space, k, capacity=None):
        if k < 0:
            raise ValueError("column count must be >= 0")
        cap = max(k, capacity or 0)
        return cls(space, cls._alloc(space, cap), k)

    @classmethod
    def from_numpy(cls, block, capacity=None):
        block = np.asarray(block, dtype=float)
        if block.ndim != 2:
            raise ValueError("need a 2-d block of column vectors")
        space = VectorSpace(block.shape[0])
        k = block.shape[1]
        out = cls.zeros(space, k, capacity)
        if k:
            lo, hi = cls._local_rows(space)
            local = block[lo:hi]
            out._buf[:k, : hi - lo].copy_(torch.from_numpy(np.ascontiguousarray(local.T)))
        return out

    @classmethod
    def from_array(cls, a):
        """Upload any reference-style VectorArray (anything with
        `_iter_columns`, or `to_numpy`) to the device backend."""
        if isinstance(a, cls):
            return a
        if hasattr(a, "to_numpy"):
            return cls.from_numpy(a.to_numpy())
        cols = list(a._iter_columns())
        block = np.column_stack(cols) if cols else np.zeros((a.space.dim, 0))
        return cls.from_numpy(block)

    # ------------------------------------------------------------ views
    @property
    def ncols(self):
        return self._k

    @property
    def ld(self):
        return self._buf.shape[1]

    @property
    def m_local(self):
        lo, hi = self._local_rows(self.space)
        return hi - lo

    @property
    def capacity(self):
        return self._buf.shape[0]

    def ptr(self, col=0):
        return self._buf.data_ptr() + 8 * col * self.ld

    def device_view(self):
        """(ncols, m_local) torch view of the local shard (row j = column j)."""
        return self._buf[: self._k, : self.m_local]

    def __len__(self):
        return self._k

    def __repr__(self):
        return f"{type(self).__name__}(dim={self.space.dim}, ncols={self._k})"

    def _check_space(self, other):
        if self.space != other.space:
            raise ValueError(f"space mismatch: dim {self.space.dim} vs {other.space.dim}")
        if type(self) is not type(other):
            raise TypeError(f"backend mismatch: {type(self).__name__} vs {type(other).__name__}")

    # ------------------------------------------------------------ interface
    def copy(self, indices=None):
        if indices is None:
            out = CudaVectorArray(self.space, self._alloc(self.space, self._k, zero=False), self._k)
            out._buf.copy_(self._buf[: self._k])
            return out
        idx = _as_index_list(indices, self._k, "copy")
        out = CudaVectorArray(self.space, self._alloc(self.space, len(idx), zero=False), len(idx))
        if idx:
            out._buf.copy_(self._buf[torch.tensor(idx, device=self._buf.device)])
        return out

    def reserve(self, capacity):
        """Grow the column capacity (keeps contents)."""
        if capacity <= self.capacity:
            return
        buf = self._alloc(self.space, capacity)
        buf[: self._k].copy_(self._buf[: self._k])
        self._buf = buf

    def append(self, other):
        self._check_space(other)
        need = self._k + other._k
        if need > self.capacity:
            self.reserve(max(need, 2 * self.capacity))
        self._buf[self._k: need].copy_(other._buf[: other._k])
        self._k = need

    def gramian(self, other=None):
        from . import _engine

        if other is None:
            return _engine.gram_host(self)
        self._check_space(other)
        return _engine.cross_gram_host(self, other)

    def lincomb(self, coeffs):
        coeffs = np.asarray(coeffs, dtype=float)
        if coeffs.ndim != 2 or coeffs.shape[0] != self._k:
            raise ValueError(
                f"coefficient matrix needs {self._k} rows, got shape {coeffs.shape}"
            )
        n = coeffs.shape[1]
        out = CudaVectorArray(self.space, self._alloc(self.space, n, zero=self._k == 0), n)
        if n and self._k:
            c, ldc = upload_coeffs(coeffs)
            cx = ctx()
            _lib.check(cx.lib.cqr_lincomb(self.ptr(), self.ld, self.m_local, self._k, c.data_ptr(), ldc, n, 0,
                                          out.ptr(), out.ld, cx.stream), "lincomb")
            cx.launches += 1
        return out

    def axpy(self, alpha, other):
        self._check_space(other)
        if other._k != self._k:
            raise ValueError(f"column count mismatch: {self._k} vs {other._k}")
        if self._k:
            cx = ctx()
            _lib.check(cx.lib.cqr_axpy(self.ptr(), self.ld, float(alpha), other.ptr(), other.ld, self.m_local,
                                       self._k, cx.stream), "axpy")
            cx.launches += 1

    def remove_columns(self, indices):
        idx = set(_as_index_list(indices, self._k, "remove_columns"))
        keep = [j for j in range(self._k) if j not in idx]
        buf = self._alloc(self.space, max(len(keep), 0), zero=False)
        if keep:
            buf.copy_(self._buf[torch.tensor(keep, device=self._buf.device)])
        self._buf = buf
        self._k = len(keep)

    def to_numpy(self):
        """Copy of the full m x k block (Fortran order), gathered over ranks."""
        local = self.device_view().cpu().numpy().T
        full = ctx().allgather_rows(local, self.space.dim)
        return np.asfortranarray(full)

    def _iter_columns(self):
        block = self.to_numpy()
        for j in range(self._k):
            yield block[:, j]
