"""Row-sharding plumbing of the data-parallel path.

Rank r of P owns rows [r m / P, (r+1) m / P) of every tall array.  Tall
kernels run on local rows; the one exchange per pass is a sum of the k x k
Gram (or the q x p cross Gram) over ranks, after which every rank runs the
k x k stage redundantly on bit-identical data.  These helpers are pure
host logic (torch.distributed, any backend) so they are exercised by the
gloo tests on CPU as well as by the NCCL runs on the GPU.
"""

from __future__ import annotations

import torch


def row_range(m, rank, world):
    """Rows [lo, hi) of a global row count m owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return m * rank // world, m * (rank + 1) // world


def _world(group=None):
    d = torch.distributed
    if d.is_available() and d.is_initialized():
        return d.get_world_size(group)
    return 1


def reduce_ranks_(flat, group=None):
    """Sum a small per-rank partial over ranks in place, deterministically.

    The partials are all-gathered (pure data movement, so NCCL's choice of
    ring / tree / NVLS cannot change a bit) and added in rank order --
    ((p0 + p1) + p2) + ... -- on the device by libcqr's `cqr_sum_ranks`, or by
    the same in-order loop for CPU tensors (the gloo tests).  Every rank
    therefore holds the same bits, two runs give the same bits, and
    bit-symmetric Gram partials give a bit-symmetric Gram with no mirroring
    pass.  One collective per call: an update pass packs Bt and G into one
    buffer."""
    world = _world(group)
    if world == 1:
        return flat
    src = flat.reshape(-1)
    assert src.is_contiguous() and src.data_ptr() == flat.data_ptr(), "reduce_ranks_ needs a contiguous tensor"
    n = src.numel()
    if flat.is_cuda and torch.distributed.get_backend(group) == "gloo":
        # gloo moves host memory: stage the partial through the host (the
        # 1-GPU test harness runs its ranks on one device with gloo; NCCL
        # gathers device buffers directly)
        host = torch.empty(world * n, dtype=flat.dtype)
        torch.distributed.all_gather_into_tensor(host, src.cpu(), group=group)
        parts = host.to(flat.device)
    else:
        parts = torch.empty(world * n, dtype=flat.dtype, device=flat.device)
        torch.distributed.all_gather_into_tensor(parts, src, group=group)
    if flat.is_cuda:
        from . import _lib
        from ._device import ctx

        cx = ctx()
        _lib.check(cx.lib.cqr_sum_ranks(parts.data_ptr(), world, n, src.data_ptr(), cx.stream), "sum_ranks")
        cx.launches += 1
    else:
        acc = parts[:n].clone()
        for r in range(1, world):
            acc += parts[r * n:(r + 1) * n]
        src.copy_(acc)
    return flat


def symmetrize_lower_(g):
    """Mirror the lower triangle onto the upper (exact)."""
    low = torch.tril(g)
    g.copy_(low + torch.tril(g, -1).T)
    return g


def allreduce_gram_(g, group=None, symmetric=True):
    """Sum a k x k Gram over ranks in place with torch.distributed.all_reduce
    (kept for comparisons: its summation order is the collective's own, so
    the lower triangle is mirrored afterwards).  The product path uses
    reduce_ranks_."""
    if _world(group) > 1:
        torch.distributed.all_reduce(g, group=group)
        if symmetric:
            symmetrize_lower_(g)
    return g
