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


def symmetrize_lower_(g):
    """Mirror the lower triangle onto the upper (exact)."""
    low = torch.tril(g)
    g.copy_(low + torch.tril(g, -1).T)
    return g


def allreduce_gram_(g, group=None, symmetric=True):
    """Sum a k x k Gram over ranks in place.  A ring reduction may add the two
    mirror elements of a symmetric matrix in different orders, so the lower
    triangle is mirrored afterwards: every rank sees the same bit-symmetric
    matrix (the factor kernel reads only the lower triangle anyway)."""
    if torch.distributed.is_available() and torch.distributed.is_initialized() and \
            torch.distributed.get_world_size(group) > 1:
        torch.distributed.all_reduce(g, group=group)
        if symmetric:
            symmetrize_lower_(g)
    return g
