"""Device-resident tall arrays behind the reference's columns-only interface.

`CudaVectorArray` is the B200 backend of the reference's `VectorArray` ABC
(reference varray.py:47-100): the same members (`space`, `ncols`, `copy`,
`append`, `gramian`, `lincomb`, `axpy`, `remove_columns`, `zeros`,
`from_numpy`, `_iter_columns`, `to_numpy`), the same ownership rules
(copy / lincomb / from_numpy allocate independent storage, append copies its
source, axpy mutates in place, gramian returns a host ndarray) and the same
exceptions (ValueError on space/shape, TypeError on backend mixing,
IndexError on bad column indices).

HBM layout (include/cqr.h): the local row shard is stored row-quad
interleaved -- a (m_pad/4, capacity, 4) fp64 tensor, element (r, c) at
[r // 4, c, r % 4] -- instead of the reference's Fortran block
(varray.py:107).  The interface never exposes rows, so the layout is free:
a 32-row panel is one contiguous run (one bulk copy per pipeline stage) and
the DMMA fragment loads are bank-conflict free.  m_pad = round_up(m, 16),
padding rows are zero.  Column capacity may exceed ncols, so appends (the
update path) do not reallocate.  Under torch.distributed each rank holds
rows [r m / P, (r+1) m / P) of every array; `space.dim` is the GLOBAL m.
Host <-> device transfers go through column-major staging converted by the
libcqr pack / unpack kernels, in row chunks.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import ctx, round_up

_CHUNK_ROWS = 1 << 22   # rows per host-transfer chunk (multiple of 16)


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


def coeff_tiles(c_dev, k, n, ld):
    """Column-major k x n device coefficients (leading dimension ld) -> the
    tiled operand layout of libcqr (cqr_pack_coeffs)."""
    cx = ctx()
    out = torch.empty(max(cx.lib.cqr_coeff_doubles(k, n), 1), dtype=torch.float64, device=cx.device)
    if k and n:
        _lib.check(cx.lib.cqr_pack_coeffs(c_dev.data_ptr(), ld, k, n, out.data_ptr(), cx.stream), "pack_coeffs")
        cx.launches += 1
    return out


def upload_coeffs(c):
    """Host k x n coefficients -> device coefficient tiles."""
    c = np.asarray(c, dtype=float)
    k, n = c.shape
    dev = torch.from_numpy(np.ascontiguousarray(c.T)).to(ctx().device)   # (n, k): column-major k x n
    return coeff_tiles(dev, k, n, max(k, 1))


class _Storage:
    """A device buffer possibly shared by several arrays (zero-copy append:
    the augmented basis of an update is a view that extends its input's
    buffer).  `claimed` = columns in use by the widest view; mutation of a
    shared buffer detaches (copy on write) so every array keeps the
    reference's value semantics."""

    __slots__ = ("claimed", "views", "__weakref__")

    def __init__(self, claimed):
        self.claimed = claimed
        self.views = 0

    def release(self):
        self.views -= 1


class _ColumnBlock:
    """Columns [c0, c0 + n) of an array's buffer as a kernel operand (QI:
    column c starts at 4 c doubles, ld = the buffer's capacity).  No ownership:
    used to let a kernel write straight into free capacity that a later
    `_claim_tail` turns into columns."""

    def __init__(self, arr, c0, n):
        self._arr = arr
        self._c0 = c0
        self.ncols = n
        self.space = arr.space

    def ptr(self):
        return self._arr._buf.data_ptr() + 8 * 4 * self._c0

    @property
    def ld(self):
        return self._arr.capacity

    @property
    def m_local(self):
        return self._arr.m_local


class CudaVectorArray:
    """Tall fp64 array on the local B200, columns-only interface."""

    def __init__(self, space, buf, ncols, storage=None):
        self.space = space
        self._buf = buf          # (m_pad/4, capacity, 4) float64
        self._k = int(ncols)
        self._attach(storage or _Storage(self._k))

    def _attach(self, storage):
        self._st = storage
        storage.views += 1
        if self._k > storage.claimed:
            storage.claimed = self._k
        self._fin = weakref.finalize(self, storage.release)

    def _detach(self):
        """Copy on write: give this array a private buffer before mutating."""
        if self._st.views <= 1:
            return
        old = CudaVectorArray(self.space, self._buf, self._k, self._st)
        buf = self._alloc(self.space, max(self._k, 1))
        self._fin()
        self._buf = buf
        self._attach(_Storage(self._k))
        self._gather(old, j0=0, n=self._k)

    # ------------------------------------------------------------ construction
    @staticmethod
    def _local_rows(space):
        return ctx().row_range(space.dim)

    @classmethod
    def _alloc(cls, space, cap, zero=True):
        lo, hi = cls._local_rows(space)
        nq = max(round_up(hi - lo, 16), 16) // 4
        fn = torch.zeros if zero else torch.empty
        return fn((nq, max(cap, 0), 4), dtype=torch.float64, device=ctx().device)

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
            for r0 in range(0, hi - lo, _CHUNK_ROWS):
                r1 = min(hi - lo, r0 + _CHUNK_ROWS)
                stage = torch.from_numpy(np.ascontiguousarray(local[r0:r1].T)).to(out._buf.device, non_blocking=True)
                out._load_rows(stage, r0)
        return out

    @classmethod
    def from_device_colmajor(cls, space, t, capacity=None):
        """Build from a device (k, m_local) tensor (column-major local shard)."""
        k = t.shape[0]
        out = cls.zeros(space, k, capacity)
        if k:
            out._load_rows(t.contiguous(), 0)
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

    def _load_rows(self, stage, r0):
        """Pack a device column-major (k, rows) block into local rows r0.."""
        cx = ctx()
        k, rows = stage.shape
        dst = self._buf.data_ptr() + 8 * (r0 // 4) * 4 * self.capacity
        _lib.check(cx.lib.cqr_pack_tall(stage.data_ptr(), rows, rows, k, dst, self.capacity, cx.stream), "pack")
        cx.launches += 1

    # ------------------------------------------------------------ views
    @property
    def ncols(self):
        return self._k

    @property
    def ld(self):
        """Column capacity (the QI layout's ldk)."""
        return self._buf.shape[1]

    capacity = ld

    @property
    def m_local(self):
        lo, hi = self._local_rows(self.space)
        return hi - lo

    def ptr(self):
        return self._buf.data_ptr()

    def to_device_colmajor(self):
        """Device (k, m_local) column-major copy of the local shard."""
        cx = ctx()
        m = self.m_local
        out = torch.empty((self._k, m), dtype=torch.float64, device=cx.device)
        if self._k and m:
            _lib.check(cx.lib.cqr_unpack_tall(self.ptr(), self.ld, m, self._k, out.data_ptr(), m, cx.stream),
                       "unpack")
            cx.launches += 1
        return out

    def __len__(self):
        return self._k

    def __repr__(self):
        return f"{type(self).__name__}(dim={self.space.dim}, ncols={self._k})"

    def _check_space(self, other):
        if self.space != other.space:
            raise ValueError(f"space mismatch: dim {self.space.dim} vs {other.space.dim}")
        if type(self) is not type(other):
            raise TypeError(f"backend mismatch: {type(self).__name__} vs {type(other).__name__}")

    def _gather(self, src, idx=None, j0=0, n=None, dcol0=0):
        cx = ctx()
        n = len(idx) if idx is not None else n
        if not n:
            return
        idx_dev = torch.tensor(idx, dtype=torch.int32, device=cx.device) if idx is not None else None
        _lib.check(cx.lib.cqr_gather_cols(src.ptr(), src.ld, idx_dev.data_ptr() if idx_dev is not None else None,
                                          j0, self.ptr(), self.ld, dcol0, n, self.m_local, cx.stream), "gather")
        cx.launches += 1

    # ------------------------------------------------------------ interface
    def copy(self, indices=None):
        if indices is None:
            out = CudaVectorArray(self.space, self._alloc(self.space, self._k, zero=False), self._k)
            out._gather(self, j0=0, n=self._k)
            return out
        idx = _as_index_list(indices, self._k, "copy")
        out = CudaVectorArray(self.space, self._alloc(self.space, len(idx), zero=False), len(idx))
        out._gather(self, idx=idx)
        return out

    def reserve(self, capacity):
        """Grow the column capacity (keeps contents; detaches from shared storage)."""
        if capacity <= self.capacity and self._st.views <= 1:
            return
        old = CudaVectorArray(self.space, self._buf, self._k, self._st)
        buf = self._alloc(self.space, max(capacity, self._k))
        self._fin()
        self._buf = buf
        self._attach(_Storage(self._k))
        self._gather(old, j0=0, n=self._k)

    def _tail_free(self, n):
        return self._k + n <= self.capacity and self._st.claimed == self._k

    def append(self, other):
        self._check_space(other)
        need = self._k + other._k
        if not self._tail_free(other._k):
            self.reserve(max(need, 2 * self.capacity))
        self._gather(other, j0=0, n=other._k, dcol0=self._k)
        self._k = need
        self._st.claimed = max(self._st.claimed, need)

    def _tail_block(self, n):
        """The n free columns after this array's own (requires _tail_free(n))."""
        return _ColumnBlock(self, self._k, n)

    def _claim_tail(self, n):
        """This array plus the n tail columns (already written) as a new array
        sharing the buffer: extended() without the copy."""
        return CudaVectorArray(self.space, self._buf, self._k + n, self._st)

    def extended(self, other):
        """q_in.copy() + append(other) as a new array (reference
        algorithms.py:453-454).  When this array owns free capacity after its
        columns, the result shares the buffer (no O(m k) copy); both arrays
        keep value semantics through copy on write."""
        self._check_space(other)
        if not self._tail_free(other._k):
            out = self.copy()
            out.reserve(self._k + other._k)
            out.append(other)
            return out
        self._gather(other, j0=0, n=other._k, dcol0=self._k)
        return CudaVectorArray(self.space, self._buf, self._k + other._k, self._st)

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
            c = upload_coeffs(coeffs)
            cx = ctx()
            _lib.check(cx.lib.cqr_lincomb(self.ptr(), self.ld, self.m_local, self._k, c.data_ptr(), n, 0,
                                          out.ptr(), out.ld, cx.stream), "lincomb")
            cx.launches += 1
        return out

    def axpy(self, alpha, other):
        self._check_space(other)
        if other._k != self._k:
            raise ValueError(f"column count mismatch: {self._k} vs {other._k}")
        if self._k:
            self._detach()
            cx = ctx()
            _lib.check(cx.lib.cqr_axpy(self.ptr(), self.ld, float(alpha), other.ptr(), other.ld, self.m_local,
                                       self._k, cx.stream), "axpy")
            cx.launches += 1

    def remove_columns(self, indices):
        idx = set(_as_index_list(indices, self._k, "remove_columns"))
        keep = [j for j in range(self._k) if j not in idx]
        out = CudaVectorArray(self.space, self._alloc(self.space, len(keep), zero=False), len(keep))
        out._gather(self, idx=keep)
        self._fin()
        self._buf, self._k = out._buf, out._k
        self._attach(_Storage(self._k))

    def to_numpy(self):
        """Copy of the full m x k block (Fortran order), gathered over ranks."""
        local = self.to_device_colmajor().cpu().numpy().T
        full = ctx().allgather_rows(local, self.space.dim)
        return np.asfortranarray(full)

    def _iter_columns(self):
        block = self.to_numpy()
        for j in range(self._k):
            yield block[:, j]
