"""Device pass engine: the tall passes and the k x k stage of one algorithm
run, with the one collective (Gram allreduce) and the one status read per
pass.  `algorithms.py` drives it with the reference's control flow.

Per run the engine owns, on the device:
  G      k x k Gram of the current pass (allreduced over ranks)
  Rk/Rinv/Racc  ldr x k (ldr = round_up(k, 32), zero padded) factors
  B, Bt  q x p blocks of the update path
  stat   status record + shift list (one D2H copy per pass)
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib
from ._device import ctx, round_up

STATUS_BYTES = 96   # sizeof(cqr_factor_status) rounded to 16

# Fixed schedules (chol_qr, chol_qr2, s_chol_qr3) enqueue natively through
# cqr_fixed_schedule, replayed as a CUDA graph: CQR_NATIVE_SCHEDULE=0 keeps the
# per-kernel Python launches, =1 the native enqueue without a graph, =2 (default)
# the native enqueue captured as a graph.
NATIVE_SCHEDULE = int(os.environ.get("CQR_NATIVE_SCHEDULE", "2"))


def _gram_ws(m_local, ka, kb, self_):
    cx = ctx()
    return cx.workspace(cx.lib.cqr_gram_workspace_bytes(m_local, ka, kb, 1 if self_ else 0))


def gram_device(arr, out=None):
    """G = X^T X (allreduced, bit-symmetric) as a k x k device tensor."""
    cx = ctx()
    k = arr.ncols
    g = out if out is not None else torch.empty((k, k), dtype=torch.float64, device=cx.device)
    ws = _gram_ws(arr.m_local, k, k, True)
    t0 = cx.timer.start() if cx.timer else None
    # G is column-major k x k: torch (k, k) row-major of G^T == G (symmetric)
    _lib.check(cx.lib.cqr_gram(arr.ptr(), arr.ld, arr.m_local, k, g.data_ptr(), k, ws.data_ptr(), ws.numel(),
                               cx.stream), "gram")
    if t0 is not None:
        cx.timer.stop("gram", t0, (arr.m_local, k))
    cx.launches += 2
    cx.reduce_ranks_(g)
    return g


def gram_host(arr):
    if arr.ncols == 0:
        return np.zeros((0, 0))
    return gram_device(arr).cpu().numpy()


def cross_gram_device(left, right, out=None):
    """G = L^T R (ka x kb) as a column-major device buffer: torch (kb, ka)."""
    cx = ctx()
    ka, kb = left.ncols, right.ncols
    g = out if out is not None else torch.empty((kb, ka), dtype=torch.float64, device=cx.device)
    if ka and kb:
        ws = _gram_ws(left.m_local, ka, kb, False)
        _lib.check(cx.lib.cqr_cross_gram(left.ptr(), left.ld, ka, right.ptr(), right.ld, kb, left.m_local,
                                         g.data_ptr(), ka, ws.data_ptr(), ws.numel(), cx.stream), "cross_gram")
        cx.launches += 2
        cx.reduce_ranks_(g)
    else:
        g.zero_()
    return g


def cross_gram_host(left, right):
    g = cross_gram_device(left, right)
    return g.cpu().numpy().T.copy()


# cqr_factor_status as a NumPy record (include/cqr.h; offsets checked against
# the ctypes struct in tests/test_abi_cpu.py)
_STATUS_DTYPE = np.dtype({
    "names": [n for n, _ in _lib.FactorStatus._fields_],
    "formats": [np.int32 if t is ctypes.c_int32 else np.float64 for _, t in _lib.FactorStatus._fields_],
    "offsets": [getattr(_lib.FactorStatus, n).offset for n, _ in _lib.FactorStatus._fields_],
    "itemsize": ctypes.sizeof(_lib.FactorStatus)})


_LAUNCHES = {}


def _fixed_launches(lib, k, n):
    """Kernels one cqr_fixed_schedule run launches: Gram (2), per pass the
    k x k stage (2) and the TRMM (+ Gram), R's download (1)."""
    key = (k, n)
    v = _LAUNCHES.get(key)
    if v is None:
        v = _LAUNCHES[key] = 2 + 2 * n + lib.cqr_apply_gram_launches(k) * (n - 1) + 1 + 1
    return v


class PassStatus:
    """Host copy of one cqr_factor_status plus the shifts it appended."""

    __slots__ = tuple(n for n, _ in _lib.FactorStatus._fields_) + ("shifts",)

    def __init__(self, raw):
        """raw: the slot's pinned bytes (uint8 NumPy view): status record, then shifts."""
        rec = raw[:_STATUS_DTYPE.itemsize].view(_STATUS_DTYPE)[0].item()
        for name, v in zip(_STATUS_DTYPE.names, rec):
            object.__setattr__(self, name, v)
        n = max(self.n_shifts, 0)
        self.shifts = raw[STATUS_BYTES:STATUS_BYTES + 8 * n].view(np.float64).tolist()


class Engine:
    """Buffers and launches for one algorithm run on width-k blocks."""

    def __init__(self, k, cfg, q=0, defer_reset=False):
        cx = ctx()
        self.cx = cx
        self.k = k
        self.q = q
        self.cfg = cfg
        self.cap = cfg.max_shift_attempts + 1
        # status slots: fixed-schedule algorithms enqueue several factor calls and
        # read their statuses once at the end (factor_async / collect)
        self.nslots = 4
        self._next_slot = 0
        self._stat_ev = [None] * self.nslots   # event after each slot's status write
        self._r_pending = None
        self._br_pending = None
        self._key = (k, q, self.cap)
        # Buffers come from the context's pool when an earlier run of the same
        # shape released them: a call then starts with one reset copy instead of
        # seven allocations and three fill kernels (short calls, config 1, are
        # host bound between calls).  Kernels never write the zero padding of
        # Rk / Rinv, so only Racc (and the update blocks) need resetting.
        # the stream this run enqueues on (a call runs on one stream; torch's
        # current_stream() costs ~8 us of host time per query)
        self._stream = cx.torch_stream()
        free = cx.engine_pool.get(self._key)
        reused = bool(free)
        if reused:
            bufs, ev = free.pop()
            self._stream.wait_event(ev)   # released on another stream
            (self.G, self.Rk, self.Rinv, self.Racc, self._racc0, self.stat_all, self.stat_host_all, self.fws,
             self.B, self.Bt, self._xch, self._fcfg, self._slot_ev, self._fx) = bufs
            if not defer_reset:   # else the caller resets (reset_racc, or the native schedule)
                self.Racc.copy_(self._racc0)
            if q:
                self.B.zero_()
                self.Bt.zero_()
        else:
            dev = cx.device
            self.ldr = max(round_up(k, 32), 32)
            # the exchange buffer of one pass: [Bt (q x p) | G (p x p)] for updates,
            # G alone otherwise -- one cross-rank reduction per pass
            self._xch = torch.empty(k * q + k * k, dtype=torch.float64, device=dev)
            self.G = self._xch[k * q:].view(k, k)
            self.Rk = torch.zeros((k, self.ldr), dtype=torch.float64, device=dev)
            self.Rinv = torch.zeros(max(cx.lib.cqr_coeff_doubles(k, k), 1), dtype=torch.float64, device=dev)  # tiles
            self._racc0 = torch.eye(k, self.ldr, dtype=torch.float64, device=dev)   # [I | 0]
            self.Racc = self._racc0.clone()
            nbytes = STATUS_BYTES + 8 * self.cap
            self.stat_all = torch.empty((self.nslots, nbytes), dtype=torch.uint8, device=dev)
            self.stat_host_all = cx.acquire_pinned((self.nslots, nbytes))
            self.fws = torch.empty(cx.lib.cqr_factor_workspace_bytes(k), dtype=torch.uint8, device=dev)
            if q:
                self.B = torch.zeros((k, q), dtype=torch.float64, device=dev)     # (p, q): column-major q x p
                self.Bt = self._xch[: k * q].view(k, q)
                self.Bt.zero_()
            else:
                self.B = self.Bt = None
        self.ldr = self.Rk.shape[1]
        self.stat, self.stat_host = self.stat_all[0], self.stat_host_all[0]
        self._stat_np = self.stat_host_all.numpy()   # (nslots, bytes) view of the pinned slots
        # per-slot launch config (static fields set once; the kernel writes the status
        # and shifts straight into the slot's pinned host buffer, no D2H copy) and
        # per-slot completion events, reused across the run's factor calls
        # (kept with the pooled buffers: the pinned slots they point at go with them)
        if not reused:
            self._fcfg = []
            for slot in range(self.nslots):
                hp = self.stat_host_all[slot].data_ptr()
                self._fcfg.append(_lib.FactorConfig(accumulate=1, status_mirror=hp, shifts_mirror=hp + STATUS_BYTES))
            self._slot_ev = [torch.cuda.Event() for _ in range(self.nslots)]
            self._fx = None   # native fixed-schedule state (run_fixed), built on first use
        for fc in self._fcfg:
            fc.unit_roundoff = cfg.unit_roundoff
            fc.shift_escalation = cfg.shift_escalation
            fc.max_shift_attempts = cfg.max_shift_attempts

    def __del__(self):
        try:
            if self._r_pending is not None:
                self._r_pending[2].synchronize()
                if self._r_pending[0] is not None:
                    self.cx.release_pinned(self._r_pending[0])
            if self._br_pending is not None:
                if self._br_pending[2] is not None:
                    self._br_pending[2].synchronize()
                self.cx.release_pinned(self._br_pending[0])
                self.cx.release_pinned(self._br_pending[1])
            ev = torch.cuda.Event()
            ev.record(self._stream)
            free = self.cx.engine_pool.setdefault(self._key, [])
            if len(free) < 2:
                free.append(((self.G, self.Rk, self.Rinv, self.Racc, self._racc0, self.stat_all, self.stat_host_all,
                              self.fws, self.B, self.Bt, self._xch, self._fcfg, self._slot_ev, self._fx), ev))
            else:
                self.cx.release_pinned(self.stat_host_all)
                if self._fx is not None:
                    self.cx.release_pinned(self._fx[3])
        except Exception:   # interpreter shutdown
            pass

    # ------------------------------------------------------------ k x k stage
    def factor(self, policy, m_global, width, *, tol=0.0, check_tol=False, stop=False, update_b=False,
               fixed_shift=0.0, est_tol=1e-2, est_max_iter=100):
        """Run the k x k stage and return its status (one host sync)."""
        h = self.factor_async(policy, m_global, width, tol=tol, check_tol=check_tol, stop=stop, update_b=update_b,
                              fixed_shift=fixed_shift, est_tol=est_tol, est_max_iter=est_max_iter)
        return self.collect([h])[0]

    def gate(self, handle):
        """Device address of the status code of an enqueued factor call: the
        gate of the launches that must only run if that call factored."""
        return self.stat_all[handle].data_ptr()

    def collect(self, handles):
        """Statuses of enqueued factor calls, in order: waits only for their own
        status copies, so later enqueued work keeps the GPU busy meanwhile."""
        for h in handles:
            ev = self._stat_ev[h]
            if ev is None:
                self._stream.synchronize()
            else:
                ev.synchronize()
        stat = self._stat_np
        return [PassStatus(stat[h].copy()) for h in handles]

    def factor_async(self, policy, m_global, width, *, tol=0.0, check_tol=False, stop=False, update_b=False,
                     fixed_shift=0.0, gate=None, gate_slot=None, est_tol=1e-2, est_max_iter=100):
        """Enqueue the k x k stage; its status lands in a pinned host slot
        (returned handle) without a sync.  Up to `nslots` calls may be pending."""
        cx = self.cx
        slot = self._next_slot
        self._next_slot = (slot + 1) % self.nslots
        cfg = self.cfg
        if cx.trace is not None:
            # stream-ordered copies: exactly what this launch will read
            cx.trace.append(dict(policy=policy, m_global=m_global, width=width, tol=tol, check_tol=check_tol,
                                 stop=stop, fixed_shift=fixed_shift, G=self.G.clone(),
                                 Bt=self.Bt.clone() if (self.Bt is not None and self.q) else None))
        fc = self._fcfg[slot]
        fc.policy = policy
        fc.shift_width = width
        fc.m_global = m_global
        fc.check_tol = 1 if check_tol else 0
        fc.tol = tol
        fc.stop = 1 if stop else 0
        fc.update_b = 1 if update_b else 0
        fc.est_max_iter = est_max_iter
        fc.est_tol = est_tol
        fc.fixed_shift = fixed_shift
        fc.gate = gate
        bt = self.Bt.data_ptr() if self.Bt is not None else None
        b = self.B.data_ptr() if self.B is not None else None
        base = self.stat_all[slot].data_ptr()
        t0 = cx.timer.start() if cx.timer else None
        _lib.check(cx.lib.cqr_factor(ctypes.byref(fc), self.k, self.G.data_ptr(), self.k, bt, max(self.q, 1),
                                     self.q, self.Rk.data_ptr(), self.Rinv.data_ptr(), self.ldr,
                                     self.Racc.data_ptr(), b, max(self.q, 1), base + STATUS_BYTES, base,
                                     self.fws.data_ptr(), self.fws.numel(), cx.stream), "factor")
        if t0 is not None:
            cx.timer.stop("factor", t0, (self.k,),
                          gate=self.stat_all[gate_slot] if gate_slot is not None else None)
        cx.launches += 2
        ev = self._slot_ev[slot]
        ev.record(self._stream)
        self._stat_ev[slot] = ev
        return slot

    def reset_racc(self):
        self.Racc.copy_(self._racc0)

    def fixed_ok(self):
        """The native fixed-schedule enqueue applies: one rank (no cross-rank
        sum between a Gram and its factor call) and no per-launch timer or
        decision trace attached."""
        cx = self.cx
        return NATIVE_SCHEDULE > 0 and cx.world == 1 and cx.trace is None and cx.timer is None

    def _fixed_state(self):
        """The cqr_fixed_plan of this engine's buffers with every static field
        set, its dst / lddst arrays, the pinned R buffer it downloads into and
        a NumPy view of R there (kept with the pooled buffers: per call only
        the shape, the tall operands and the workspace are written)."""
        if self._fx is None:
            k = self.k
            plan = _lib.FixedPlan()
            plan.k = k
            plan.G = self.G.data_ptr()
            plan.Rk = self.Rk.data_ptr()
            plan.Rinv = self.Rinv.data_ptr()
            plan.Racc = self.Racc.data_ptr()
            plan.Racc0 = self._racc0.data_ptr()
            plan.ldr = self.ldr
            plan.fws = self.fws.data_ptr()
            plan.fws_bytes = self.fws.numel()
            for i in range(3):
                plan.fcfg[i] = ctypes.pointer(self._fcfg[i])
                plan.status[i] = self.stat_all[i].data_ptr()
            rbuf = self.cx.acquire_pinned((self.Racc.numel() * 8,))
            plan.R_host = rbuf.data_ptr()
            rview = rbuf.numpy().view(np.float64).reshape(self.Racc.shape)[:, :k]
            self._fx = (plan, plan.dst, plan.lddst, rbuf, rview, {})
        return self._fx

    def run_fixed(self, policies, m_global, width, src, dsts):
        """Enqueue a whole fixed schedule with one libcqr call
        (cqr_fixed_schedule): Racc reset, Gram(src), then per pass i the k x k
        stage (policies[i], status slot i) and dsts[i] = src_i R_i^-1 with the
        next Gram (plain TRMM on the last pass), then R's download.  Returns
        the status handles (slots 0..len-1) for collect()."""
        cx = self.cx
        k = self.k
        n = len(policies)
        assert 1 <= n <= 3 and len(dsts) == n and self._next_slot == 0
        plan, dst, lddst, _rbuf, rview, wsz = self._fixed_state()
        m = src.m_local
        plan.passes = n
        plan.m = m
        plan.X = src.ptr()
        plan.ldx = src.ld
        for i, d in enumerate(dsts):
            dst[i] = d.ptr()
            lddst[i] = d.ld
            fc = self._fcfg[i]
            fc.policy = policies[i]
            fc.shift_width = width
            fc.m_global = m_global
            fc.check_tol = 0
            fc.tol = 0.0
            fc.stop = 0
            fc.update_b = 0
            fc.est_max_iter = 100
            fc.est_tol = 1e-2
            fc.fixed_shift = 0.0
            fc.gate = None
        need = wsz.get(m)
        if need is None:
            need = wsz[m] = max(cx.lib.cqr_gram_workspace_bytes(m, k, k, 1), cx.lib.cqr_apply_gram_workspace_bytes(m, k))
        ws = cx.workspace(need)
        plan.ws = ws.data_ptr()
        plan.ws_bytes = ws.numel()
        plan.use_graph = 1 if NATIVE_SCHEDULE >= 2 else 0
        _lib.check(cx.lib.cqr_fixed_schedule(ctypes.byref(plan), cx.stream), "fixed_schedule")
        ev = self._slot_ev[0]
        ev.record(self._stream)
        cx.launches += _fixed_launches(cx.lib, k, n)
        for i in range(n):
            self._stat_ev[i] = ev
        self._next_slot = n % self.nslots
        self._r_pending = (None, rview, ev)   # R lands in the engine's own pinned buffer
        return list(range(n))

    # ------------------------------------------------------------ tall passes
    def gram(self, arr):
        gram_device(arr, self.G)

    def apply(self, src, dst, with_gram=True, gate=None, gate_slot=None):
        """dst = src R^-1 (TRMM); with_gram also forms G = dst^T dst.  With a
        gate (Engine.gate of a factor call) the device skips it unless that
        call factored."""
        cx = self.cx
        t0 = cx.timer.start() if cx.timer else None
        if with_gram:
            ws = cx.workspace(cx.lib.cqr_apply_gram_workspace_bytes(src.m_local, self.k))
            _lib.check(cx.lib.cqr_apply_gram_gated(src.ptr(), src.ld, src.m_local, self.k, self.Rinv.data_ptr(),
                                                   dst.ptr(), dst.ld, self.G.data_ptr(), self.k,
                                                   ws.data_ptr(), ws.numel(), gate, cx.stream), "apply_gram")
            cx.launches += cx.lib.cqr_apply_gram_launches(self.k)
            if t0 is not None:
                cx.timer.stop("apply_gram", t0, (src.m_local, self.k),
                              gate=self.stat_all[gate_slot] if gate_slot is not None else None)
            cx.reduce_ranks_(self.G)
        else:
            assert gate is None, "gated TRMM without Gram is not needed by any schedule"
            _lib.check(cx.lib.cqr_lincomb(src.ptr(), src.ld, src.m_local, self.k, self.Rinv.data_ptr(),
                                          self.k, 1, dst.ptr(), dst.ld, cx.stream), "apply")
            if t0 is not None:
                cx.timer.stop("apply", t0, (src.m_local, self.k))
            cx.launches += 1

    def update_pass(self, q_in, qb, initial, out=None, gate=None, gate_slot=None):
        """Fused block-update pass (cqr_update_pass_to): Bt, G from Q_in and the
        block; in iteration mode the block is first replaced by
        (Q - Q_in Bt) R^-1, in place or written to `out`."""
        cx = self.cx
        dst = qb if out is None else out
        ws = cx.workspace(cx.lib.cqr_update_workspace_bytes(qb.m_local, q_in.ncols, self.k), which=1)
        t0 = cx.timer.start() if cx.timer else None
        _lib.check(cx.lib.cqr_update_pass_gated(q_in.ptr(), q_in.ld, q_in.ncols, qb.ptr(), qb.ld, dst.ptr(),
                                                dst.ld, self.k, qb.m_local, self.Bt.data_ptr(), q_in.ncols,
                                                self.Rinv.data_ptr(), 1 if initial else 0, self.Bt.data_ptr(),
                                                self.G.data_ptr(), self.k, ws.data_ptr(), ws.numel(), gate,
                                                cx.stream),
                   "update_pass")
        if t0 is not None:
            cx.timer.stop("update_pass", t0, (qb.m_local, q_in.ncols, self.k, 1 if initial else 0),
                          gate=self.stat_all[gate_slot] if gate_slot is not None else None)
        cx.launches += 2
        # one collective per pass: Bt and G are adjacent in one buffer
        cx.reduce_ranks_(self._xch)

    def in_place_ok(self):
        """TRMM may overwrite its input (one 64-wide column tile per row tile)."""
        return self.k <= 64

    def in_place_gram_ok(self):
        """apply_gram may overwrite its input (fused kernel, or k <= 64)."""
        return self.k <= 64 or self.cx.lib.cqr_apply_gram_inplace_ok(self.k) == 1

    def _store_host(self, t, buf):
        """Enqueue t (contiguous device fp64) -> the pinned buffer `buf` as a
        kernel's mapped stores (cqr_store_to_host), not a copy-engine
        transfer: it must not queue behind a caller's bulk D2H copy of Q on
        another stream (the streamed e2e loader)."""
        _lib.check(self.cx.lib.cqr_store_to_host(t.data_ptr(), t.numel(), buf.data_ptr(), self.cx.stream),
                   "store_to_host")
        self.cx.launches += 1

    def _to_host(self, t):
        """A column-major device matrix as a row-major numpy array, through a
        pooled pinned buffer (a pageable copy costs several times more)."""
        t = t.contiguous()
        buf = self.cx.acquire_pinned((t.numel() * 8,))
        try:
            view = buf.view(torch.float64)[: t.numel()].view(t.shape)
            self._store_host(t, buf)
            self._stream.synchronize()
            return view.numpy().T.copy()
        finally:
            self.cx.release_pinned(buf)

    def r_prefetch(self):
        """Enqueue the download of R now (after the last launch of a fixed
        schedule), so it runs right behind the last kernel while the host reads
        the statuses; r_host() then only waits for it."""
        t = self.Racc[:, : self.k]
        if not t.is_contiguous():
            t = t.contiguous()
        buf = self.cx.acquire_pinned((t.numel() * 8,))
        view = buf.view(torch.float64)[: t.numel()].view(t.shape)
        self._store_host(t, buf)
        ev = torch.cuda.Event()
        ev.record(self._stream)
        self._r_pending = (buf, view, ev)

    def r_host(self):
        if self._r_pending is not None:
            buf, view, ev = self._r_pending
            self._r_pending = None
            ev.synchronize()
            if buf is None:   # run_fixed: a NumPy view of the engine's own buffer
                return view.T.copy()
            out = view.numpy().T.copy()
            self.cx.release_pinned(buf)
            return out
        return self._to_host(self.Racc[:, : self.k])

    def br_prefetch(self):
        """Enqueue the downloads of B and R (whole Racc buffer) into one pair of
        pinned buffers, reused on every call: the update loop enqueues them
        behind every newly enqueued pass (passes after convergence are gated
        no-ops, so the last downloads hold the final B and R), and br_host() then
        waits once instead of two synchronous round trips after the loop."""
        if self._br_pending is None:
            bb = self.cx.acquire_pinned((self.B.numel() * 8,))
            rb = self.cx.acquire_pinned((self.Racc.numel() * 8,))
            self._br_pending = [bb, rb, None]
        bb, rb, _ = self._br_pending
        self._store_host(self.B, bb)
        self._store_host(self.Racc, rb)
        ev = torch.cuda.Event()
        ev.record(self._stream)
        self._br_pending[2] = ev

    def br_host(self):
        """(B, R) as row-major numpy arrays, from the last br_prefetch."""
        bb, rb, ev = self._br_pending
        self._br_pending = None
        ev.synchronize()
        b = bb.view(torch.float64)[: self.B.numel()].view(self.B.shape).numpy().T.copy()
        r = rb.view(torch.float64)[: self.Racc.numel()].view(self.Racc.shape).numpy()[:, : self.k].T.copy()
        self.cx.release_pinned(bb)
        self.cx.release_pinned(rb)
        return b, r

    def b_host(self):
        return self._to_host(self.B)
