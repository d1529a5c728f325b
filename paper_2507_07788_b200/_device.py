"""Per-process device context: CUDA device, stream, workspaces, row sharding.

PyTorch is plumbing here: device allocations (caching allocator), the
stream handle passed to libcqr, pinned host staging and torch.distributed
(NCCL) for the one collective of a pass.  One process drives one GPU; under
torch.distributed each rank owns a contiguous block of rows of every tall
array.
"""

from __future__ import annotations

import os

import torch

from . import _lib

_ctx = None

if hasattr(torch._C, "_cuda_getCurrentRawStream"):
    def _raw_stream(index):
        return torch._C._cuda_getCurrentRawStream(index)
else:   # pragma: no cover
    def _raw_stream(index):
        return torch.cuda.current_stream(index).cuda_stream


def round_up(a, b):
    return (a + b - 1) // b * b


class DeviceContext:
    def __init__(self):
        if not torch.cuda.is_available():
            raise RuntimeError(
                "paper_2507_07788_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
        self.lib = _lib.load()
        if "CQR_FACTOR_CLUSTER" in os.environ:   # diagnostics: k x k stage schedule (cqr_debug_factor_cluster)
            self.lib.cqr_debug_factor_cluster(int(os.environ["CQR_FACTOR_CLUSTER"]))
        if "CQR_UPDATE_NARROW_TEAMS" in os.environ:   # diagnostics: narrow update pass schedule
            self.lib.cqr_debug_update_narrow_teams(int(os.environ["CQR_UPDATE_NARROW_TEAMS"]))
        if "CQR_UPDATE_SR16_FROM" in os.environ:   # diagnostics: sub-panel height switch of the update pass
            self.lib.cqr_debug_update_sr16_from(int(os.environ["CQR_UPDATE_SR16_FROM"]))
        if "CQR_UPDATE_DIRECT" in os.environ:   # diagnostics: initial passes read the staged block in place
            self.lib.cqr_debug_update_direct(int(os.environ["CQR_UPDATE_DIRECT"]))
        if "CQR_UPDATE_LAG" in os.environ:   # diagnostics: cross-Gram lag of the update pass
            self.lib.cqr_debug_update_lag(int(os.environ["CQR_UPDATE_LAG"]))
        if torch.distributed.is_available() and torch.distributed.is_initialized():
            self.rank = torch.distributed.get_rank()
            self.world = torch.distributed.get_world_size()
            local = int(os.environ.get("LOCAL_RANK", self.rank % max(torch.cuda.device_count(), 1)))
        else:
            self.rank, self.world, local = 0, 1, torch.cuda.current_device()
        self.device = torch.device("cuda", local)
        torch.cuda.set_device(self.device)
        self._ws = torch.empty(0, dtype=torch.uint8, device=self.device)
        self._ws2 = torch.empty(0, dtype=torch.uint8, device=self.device)
        self._pinned = {}   # shape -> free pinned host buffers (status slots; cudaHostAlloc is slow)
        self._streams = {}   # raw cudaStream_t -> torch Stream (torch_stream)
        self.engine_pool = {}   # (k, q, status capacity) -> [(Engine buffers, release event)]
        self.launches = 0   # libcqr kernel launches issued (bench bookkeeping)
        self.timer = None   # optional KernelTimer (bench): CUDA events per libcqr call
        # optional list (tests): every factor call appends the k x k inputs it
        # reads -- (policy, m_global, width, G copy, Bt copy or None) -- so a
        # checker can replay the decision stage on the device's own Gramians
        self.trace = None

    # ---------------------------------------------------------------- plumbing
    def torch_stream(self):
        """torch's current stream as a Stream object, cached by raw handle
        (torch.cuda.current_stream() builds a new object per query, ~8 us)."""
        raw = _raw_stream(self.device.index)
        s = self._streams.get(raw)
        if s is None:
            s = self._streams[raw] = torch.cuda.current_stream(self.device)
        return s

    @property
    def stream(self):
        """Handle of torch's current stream on this device (the raw query: building
        a torch Stream object per launch cost ~5 us of host time)."""
        return _raw_stream(self.device.index)

    def acquire_pinned(self, shape):
        """A pinned uint8 host buffer of `shape` from the free list (or a new one)."""
        free = self._pinned.setdefault(tuple(shape), [])
        return free.pop() if free else torch.empty(shape, dtype=torch.uint8, pin_memory=True)

    def release_pinned(self, buf):
        self._pinned.setdefault(tuple(buf.shape), []).append(buf)

    def workspace(self, nbytes, which=0):
        """Reusable device scratch (grown on demand)."""
        buf = self._ws if which == 0 else self._ws2
        if buf.numel() < nbytes:
            buf = torch.empty(round_up(max(nbytes, 1 << 20), 1 << 20), dtype=torch.uint8, device=self.device)
            if which == 0:
                self._ws = buf
            else:
                self._ws2 = buf
        return buf

    def row_range(self, m):
        """Rows [lo, hi) of a global row count m owned by this rank."""
        from .dist import row_range

        return row_range(m, self.rank, self.world)

    def reduce_ranks_(self, t):
        """Sum a small device tensor over ranks in a fixed order (all-gather +
        in-order device sum, dist.reduce_ranks_); no-op on one rank."""
        if self.world == 1:
            return t
        from .dist import reduce_ranks_

        return reduce_ranks_(t)

    def allgather_rows(self, local, m):
        """Concatenate per-rank row blocks (host numpy, m_local x k) to m x k."""
        if self.world == 1:
            return local
        import numpy as np

        t = torch.from_numpy(np.ascontiguousarray(local)).to(self.device)
        sizes = [self_hi - self_lo for (self_lo, self_hi) in
                 (((m * r) // self.world, (m * (r + 1)) // self.world) for r in range(self.world))]
        mx = max(sizes)
        pad = torch.zeros((mx, t.shape[1]), dtype=t.dtype, device=self.device)
        pad[: t.shape[0]] = t
        out = [torch.empty_like(pad) for _ in range(self.world)]
        torch.distributed.all_gather(out, pad)
        return np.concatenate([o[:s].cpu().numpy() for o, s in zip(out, sizes)], axis=0)


class KernelTimer:
    """CUDA events around each libcqr call on the launching stream, by name.
    Used by bench.py to time the dominant kernel inside the timed region."""

    def __init__(self):
        self.events = []   # (name, start, end, work)

    def start(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def stop(self, name, start, work=None, gate=None):
        """`gate`: the device status slot a gated launch depended on; a copy of
        its code is kept so launches the device skipped are left out."""
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        code = gate[:4].clone() if gate is not None else None
        self.events.append((name, start, e, work, code))

    def summary(self):
        torch.cuda.synchronize()
        out = {}
        for name, s, e, work, code in self.events:
            if code is not None and int(code.view(torch.int32).item()) != 0:
                continue   # gated off on the device (the pass after convergence)
            d = out.setdefault(name, {"ms": [], "work": []})
            d["ms"].append(s.elapsed_time(e))
            d["work"].append(work)
        return out


def ctx():
    """The process-wide device context (created on first use)."""
    global _ctx
    if _ctx is None:
        _ctx = DeviceContext()
    return _ctx


def reset():
    """Forget the context (after torch.distributed is (re)initialized)."""
    global _ctx
    _ctx = None
