"""Benchmark of the shifted Cholesky QR hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Default workload: BASELINE.json config 3 (the metric is quoted on shifted
CholeskyQR3; config 3 is the largest shifted-CholQR3 configuration that fits
one GPU): `rs_chol_qr` ("shifted CholeskyQR3 with the paper's improved
shift") on X = U diag(sigma) V^T, 2,000,000 x 256, sigma 1 -> 1e-15.  One
step = one full `rs_chol_qr` call on the input resident in HBM (all passes,
k x k stages, status reads).  Rows are sharded evenly over ranks (strong
scaling: the global matrix is fixed).  value = global rows*cols / step time.

e2e: the same call through the public API from pinned HOST memory (H2D of the
rank's rows, the run, D2H of Q and R inside the timed region), K calls
streamed the way a loader feeds them (call i+1's H2D and call i-1's D2H on copy
streams overlap call i); the one-call-at-a-time number is reported beside it
(`e2e.serial`).
roofline: the dominant kernel (fused TRMM + Gram pass) timed with CUDA events
on the launching stream inside the timed region; achieved = algorithmic fp64
flops per launch (k(k+1) per row for the TRMM by the triangular R^-1 plus
k(k+1) per row for the symmetric Gram) / mean launch time, against the FP64
peak measured on this pool's B200s (profiles/r01_fp64_peak.json, DMMA).
cpu_baseline: the CPU oracle (NumPy restatement of the reference, `oracle/`)
on a bounded row sample of the same construction, all host cores.

CQR_BENCH_ONE_GPU_RANKS=1 (tests only): under torchrun every rank runs on
cuda:0 with gloo instead of NCCL, to exercise the N > 1 code path on a
one-GPU box; its timings mean nothing.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
FP64_PEAK_TFS = 37.2          # measured DMMA peak, profiles/r01_fp64_peak.json
FP64_PEAK_SRC = "measured DMMA.8x8x4 microbenchmark (profiles/r01_fp64_peak.json)"


def _hbm_peak_gbs():
    """The driver-measured copy bandwidth (MEASURED_PEAKS.json), else the
    profiling recipe's fallback for B200."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6550.0
# DRAM traffic of one dominant-kernel launch from `ncu --set full` captures at
# the bench's exact per-launch shape (tools/profile_round.sh); per config: the
# captures summed, and the (rows, cols) they were taken at.
NCU_SUMMARY = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_ncu_summary.json")
TRAFFIC_CAPTURES = {
    3: (("trmm_k256.ncu-rep", "gram_k256.ncu-rep"), (2_000_000, 256)),
    # config 5's pass is one fused launch; captured at 32M rows (the 128M-row
    # launch is 4x the same streaming sweep), scaled per row
    5: (("fused_k64.ncu-rep",), (32_000_000, 64)),
}


def _traffic(config, rows, cols):
    """Measured DRAM bytes per launch (read + write) of the dominant pass, or
    None when no capture matches (same width; rows scaled for streaming sweeps
    captured at a smaller row count)."""
    caps, shape = TRAFFIC_CAPTURES.get(config, ((), None))
    if not caps or shape[1] != cols or rows <= 0 or not os.path.exists(NCU_SUMMARY):
        return None
    with open(NCU_SUMMARY) as fh:
        by = {d["capture"]: d for d in json.load(fh)}
    if not all(c in by for c in caps):
        return None
    return sum(by[c]["dram_read_bytes"] + by[c]["dram_write_bytes"] for c in caps) * rows / shape[0]


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--rows", type=int, default=None, help="override global rows (testing)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    return p.parse_args()


ARGS = _args()
if ARGS.impl == "reference":
    # reference CLI pins BLAS threads before NumPy loads (cli.py:179-199)
    n = str(os.cpu_count() or 1)
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "CHOLQR_THREADS"):
        os.environ.setdefault(v, n)

import numpy as np  # noqa: E402

sys.path.insert(0, ROOT)

CFG = {
    1: dict(workload="s_chol_qr3 200000x64 kappa=1e12 (BASELINE config 1)", m=200_000, k=64, algo="s_chol_qr3",
            cond=12.0, cpu_rows=200_000),
    2: dict(workload="chol_qr2 4000000x128 N(0,1) (BASELINE config 2)", m=4_000_000, k=128, algo="chol_qr2",
            cond=None, cpu_rows=1_000_000),
    # cpu_rows: the bounded CPU sample; 1M rows of config 3 take the same 5
    # passes [1, 1, 1, 0, 0] as the 2M-row workload (200k rows take 4)
    3: dict(workload="rs_chol_qr 2000000x256 kappa=1e15 (BASELINE config 3)", m=2_000_000, k=256,
            algo="rs_chol_qr", cond=15.0, cpu_rows=1_000_000),
    4: dict(workload="chol_qr_update chain 8000000 x (16 + 31 x 16), A_j = Q_prev C_j + 1e-8 G_j "
                     "(BASELINE config 4)", m=8_000_000, k=512, p=16, blocks=31, algo="chol_qr_update",
            cond=None, cpu_rows=200_000),
    5: dict(workload="chol_qr2 128000000x64 N(0,1) (BASELINE config 5)", m=128_000_000, k=64, algo="chol_qr2",
            cond=None, cpu_rows=4_000_000),
}
SEED = 2025


def _metric():
    if ARGS.config == 4:
        return "block-append update rows*cols/s (cols = 512)"
    return "shifted CholQR3 rows*cols/s" if ARGS.config in (1, 3) else "CholQR2 rows*cols/s"


# ---------------------------------------------------------------------------- CPU legs
def _cpu_update_chain(rows, blocks, p=16, seed=SEED):
    """Oracle block-append chain on `rows` rows; returns the seconds spent in
    chol_qr_update calls (block generation excluded, as on the GPU)."""
    from oracle import cholqr_oracle as co
    from paper_2507_07788_b200.workloads import next_block

    rng = np.random.default_rng(seed)
    q0 = np.linalg.qr(rng.standard_normal((rows, p)))[0]
    res = co.rs_chol_qr(q0)
    q, r = res.q, res.r
    spent = 0.0
    for _ in range(blocks):
        a = next_block(q, rng, p)
        t0 = time.perf_counter()
        res = co.chol_qr_update(q, r, a)
        spent += time.perf_counter() - t0
        q, r = res.q, res.r
    return spent


def _cpu_run(cfg, rows, reps):
    """Time the oracle (reference restatement) on `rows` rows of the config's
    construction; returns (seconds per call, sample description)."""
    from oracle import cholqr_oracle as co
    from paper_2507_07788_b200.workloads import host_config

    if ARGS.config == 4:
        sec = _cpu_update_chain(rows, cfg["blocks"])
        return sec, f"31 chol_qr_update calls on {rows} rows (16 -> 512 columns), block generation excluded"

    x = host_config(ARGS.config, m=rows, seed=SEED)
    fn = {"s_chol_qr3": co.s_chol_qr3, "chol_qr2": co.chol_qr2, "rs_chol_qr": co.rs_chol_qr}[cfg["algo"]]
    fn(x)  # warm-up (cli.py:463)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        res = fn(x)
        times.append(time.perf_counter() - t0)
    passes = res.iterations
    return float(np.median(times)), f"{cfg['algo']} on {rows}x{cfg['k']} rows of the same construction " \
                                    f"({passes} passes), median of {reps}"


def run_reference():
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CFG[ARGS.config]
    rows = ARGS.rows or cfg["cpu_rows"]
    from oracle import cholqr_oracle as co  # noqa: F401
    from paper_2507_07788_b200.workloads import host_config

    if ARGS.config == 4:
        _cpu_update_chain(rows, 2)
        dt = sum(_cpu_update_chain(rows, cfg["blocks"]) for _ in range(ARGS.steps)) / ARGS.steps
    else:
        x = host_config(ARGS.config, m=rows, seed=SEED)
        fn = {"s_chol_qr3": co.s_chol_qr3, "chol_qr2": co.chol_qr2, "rs_chol_qr": co.rs_chol_qr}[cfg["algo"]]
        # NumPy / OpenBLAS need one warm-up call (thread pool, page faults); more
        # would only lengthen the run (each call is a bounded ~10-20 s sample)
        for _ in range(min(ARGS.warmup, 1)):
            fn(x)
        t0 = time.perf_counter()
        for _ in range(ARGS.steps):
            fn(x)
        dt = (time.perf_counter() - t0) / ARGS.steps
    value = rows * cfg["k"] / dt
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": _metric(), "value": value, "unit": "rows*cols/s",
        "n_gpus": ARGS.gpus, "steps": ARGS.steps, "warmup": ARGS.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded)",
        "config": {"workload": cfg["workload"], "rows_sampled": rows, "cols": cfg["k"]},
        "cpu_baseline": {"value": value, "unit": "rows*cols/s", "cores": cores, "kind": "port",
                         "sample": f"oracle {cfg['algo']} on {rows}x{cfg['k']} (bounded row sample of the "
                                   f"workload), {cores} BLAS threads"},
        "e2e": {"value": value, "unit": "rows*cols/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, idx):
        self.idx = idx
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([s.strip() for s in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = sorted(float(r[1]) for r in self.rows)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for n, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.rows[0][2]), "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------- GPU arm
def run_ours():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # plumbing check of the N > 1 path on a one-GPU box (tests only): every rank
    # on cuda:0 with gloo's host-staged allreduce; no kernel waits on another rank
    one_gpu_check = os.environ.get("CQR_BENCH_ONE_GPU_RANKS") == "1"
    if one_gpu_check:
        local = 0
        os.environ["LOCAL_RANK"] = "0"
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu_check:
            dist.init_process_group("gloo")
        else:
            # NCCL's own INIT lines (ranks, NVLink / NVLS topology) on stderr so the
            # rank count can be checked from the run's log; stdout keeps the one JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        sys.stderr.write(f"[bench] rank {dist.get_rank()} of {dist.get_world_size()} on cuda:{local}, backend "
                         f"{dist.get_backend()}, nccl {'.'.join(map(str, torch.cuda.nccl.version()))}\n")
    import paper_2507_07788_b200 as cq
    from paper_2507_07788_b200 import _device
    from paper_2507_07788_b200.workloads import device_gaussian, device_svd_matrix

    cx = _device.ctx()
    cfg = CFG[ARGS.config]
    m, k = (ARGS.rows or cfg["m"]), cfg["k"]
    space = cq.VectorSpace(m)
    algo = getattr(cq, cfg["algo"])

    # ---- input resident in HBM (each rank builds the global matrix's own rows)
    def from_global(x_full):
        lo, hi = cx.row_range(m)
        return cq.CudaVectorArray.from_device_colmajor(space, x_full[lo:hi].T)

    if ARGS.config == 4:
        return run_update_chain(cq, cx, cfg, m, world, rank, local)
    data = "synthetic (seeded, built in HBM with torch)"
    if ARGS.config == 3 and world == 1 and not ARGS.rows:
        # the headline input: exactly the bits tests/test_gpu_fullsize.py checks
        # against the oracle (workloads.host_config, NumPy on the host)
        from paper_2507_07788_b200.workloads import host_config

        a = cq.CudaVectorArray.from_numpy(host_config(3, seed=SEED))
        data = "synthetic: workloads.host_config(3, seed=2025), NumPy on the host (the input tests/" \
               "test_gpu_fullsize.py checks against the oracle)"
    elif cfg["cond"] is not None:
        u_from = "householder" if ARGS.config == 1 else "cholqr2"
        a = device_svd_matrix(from_global, m, k, cfg["cond"], SEED, u_from=u_from)
    else:
        a = device_gaussian(cq.CudaVectorArray.zeros(space, k), SEED + rank)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=cx.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up
    res = None
    for _ in range(ARGS.warmup):
        res = None            # drop the previous Q before the next one is allocated (config 5: 61 GB each)
        res = algo(a)
    barrier()

    # ---- timed region (device-resident input): the headline, no per-call events
    launches0 = cx.launches
    with ClockSampler(local) as clocks:
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(ARGS.steps):
            res = None
            res = algo(a)
        e1.record()
        barrier()
    launches = (cx.launches - launches0) // ARGS.steps
    passes, attempts = res.iterations, list(res.shift_attempts)
    ms = max_over_ranks(e0.elapsed_time(e1) / ARGS.steps)
    value = m * k / (ms * 1e-3)
    # quality of the timed run's result (outside the timed region), the
    # reference's Frobenius measures (metrics.py:42-71)
    quality = {"loo_fro": cq.loss_of_orthogonality(res.q, norm="frobenius"),
               "rrr_fro": cq.reconstruction_residual(a, res.q, res.r, norm="frobenius"),
               "shift_attempts": attempts, "shifts": list(res.shifts_applied)}

    # ---- the same K steps again with CUDA events around every libcqr call on
    # the launching stream (KernelTimer): the per-kernel durations of the
    # roofline.  Kept out of the headline region because the per-call event
    # records cost host time that short calls (config 1) would otherwise see.
    cx.timer = _device.KernelTimer()
    barrier()
    k0 = torch.cuda.Event(enable_timing=True)
    k1 = torch.cuda.Event(enable_timing=True)
    k0.record()
    for _ in range(ARGS.steps):
        res = None
        res = algo(a)
    k1.record()
    barrier()
    ktimes = cx.timer.summary()
    cx.timer = None
    ms_timed = k0.elapsed_time(k1) / ARGS.steps

    # ---- dominant kernel roofline
    dom = "apply_gram" if "apply_gram" in ktimes else "gram"
    lm = [w[0] for w in ktimes[dom]["work"]]
    kms = ktimes[dom]["ms"]
    flops = [2.0 * rows * k * (k + 1) if dom == "apply_gram" else 1.0 * rows * k * (k + 1) for rows in lm]
    tfs = sum(flops) / (sum(kms) * 1e-3) / 1e12
    step_share = sum(kms) / ARGS.steps / ms_timed
    kernel_summary = {n: {"launches_per_step": len(v["ms"]) / ARGS.steps, "mean_ms": float(np.mean(v["ms"]))}
                      for n, v in ktimes.items()}

    # ---- e2e through the public API from pinned host memory
    e2e = None
    lo, hi = cx.row_range(m)
    # the streamed schedule holds the resident input, two staged inputs and two
    # calls' Q (plus their column-major copies): ~7 arrays; config 5 at N = 1
    # (61 GB each) cannot, so its line carries no e2e (said in the line)
    e2e_fits = 7 * (hi - lo) * k * 8 <= torch.cuda.get_device_properties(cx.device).total_memory
    if not ARGS.no_e2e and not e2e_fits:
        e2e = {"skipped": f"streamed e2e needs ~7 arrays of {(hi - lo) * k * 8 / 1e9:.1f} GB in HBM"}
    if not ARGS.no_e2e and e2e_fits:
        host = torch.empty((k, hi - lo), dtype=torch.float64, pin_memory=True)
        host.copy_(a.to_device_colmajor())
        qhost = torch.empty((k, hi - lo), dtype=torch.float64, pin_memory=True)
        torch.cuda.synchronize()

        def e2e_step():
            # host (pinned, column-major) -> HBM -> rs_chol_qr -> Q, R back to host
            arr = cq.CudaVectorArray.from_device_colmajor(space, host.to(cx.device, non_blocking=True))
            r = algo(arr)
            qhost.copy_(r.q.to_device_colmajor(), non_blocking=True)
            torch.cuda.synchronize()
            return r.r

        res = None
        e2e_step()
        barrier()
        n_ser = max(1, min(ARGS.steps, 3))
        t0 = time.perf_counter()
        for _ in range(n_ser):
            e2e_step()
        barrier()
        ser_ms = max_over_ranks((time.perf_counter() - t0) / n_ser * 1e3)

        # Streamed: K calls back to back, each with its own H2D of the input and
        # D2H of Q and R, as a loader would feed them: call i+1's input is copied
        # in on a copy stream and call i-1's Q copied out on another while call
        # i factors (PCIe is full duplex; the two copies and the FP64 work
        # overlap).  Every byte of every call still crosses PCIe inside the
        # timed region; per-call time = total / K.
        comp = torch.cuda.current_stream(cx.device)
        s_in, s_out = torch.cuda.Stream(cx.device), torch.cuda.Stream(cx.device)
        dev_in = [torch.empty((k, hi - lo), dtype=torch.float64, device=cx.device) for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        n_str = max(20, ARGS.steps)   # a loader's stream of calls: fill and drain amortised over >= 20

        def streamed():
            held = []             # (result, Q staging, copy-out event) of calls still copying out
            freed = torch.cuda.Event()
            freed.record(comp)
            with torch.cuda.stream(s_in):
                dev_in[0].copy_(host, non_blocking=True)
                ev_in[0].record(s_in)
            for i in range(n_str):
                b = i & 1
                comp.wait_event(ev_in[b])
                if i + 1 < n_str:
                    with torch.cuda.stream(s_in):
                        s_in.wait_event(freed)      # buffer b^1 was last read by call i-1
                        dev_in[b ^ 1].copy_(host, non_blocking=True)
                        ev_in[b ^ 1].record(s_in)
                arr = cq.CudaVectorArray.from_device_colmajor(space, dev_in[b])
                freed = torch.cuda.Event()
                freed.record(comp)                   # dev_in[b] consumed (packed into arr)
                r = algo(arr)                        # returns with R on the host
                done = torch.cuda.Event()
                done.record(comp)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(done)
                    qdev = r.q.to_device_colmajor()
                    qhost.copy_(qdev, non_blocking=True)
                    out_ev = torch.cuda.Event()
                    out_ev.record(s_out)
                # keep each call's Q alive until its copy-out has run (no host wait here:
                # the host goes straight on to enqueue the next call)
                held.append((r, qdev, out_ev))
                del arr, r, qdev
                while held and held[0][2].query():
                    held.pop(0)
            torch.cuda.synchronize()
            held.clear()

        streamed()
        barrier()
        t0 = time.perf_counter()
        streamed()
        barrier()
        e2e_ms = max_over_ranks((time.perf_counter() - t0) / n_str * 1e3)
        # the PCIe floor of this run: one H2D of the input and one D2H of Q at
        # once, through the same pinned buffers (the e2e step moves both)
        torch.cuda.synchronize()
        p0 = time.perf_counter()
        with torch.cuda.stream(s_in):
            dev_in[0].copy_(host, non_blocking=True)
        with torch.cuda.stream(s_out):
            qhost.copy_(dev_in[1], non_blocking=True)   # Q-sized device buffer (no extra allocation)
        torch.cuda.synchronize()
        floor_ms = (time.perf_counter() - p0) * 1e3
        h2d = (hi - lo) * k * 8
        e2e = {"value": m * k / (e2e_ms * 1e-3), "unit": "rows*cols/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": (h2d + k * k * 8) * world,
               "api": f"CudaVectorArray (H2D from pinned host) -> {cfg['algo']} -> Q, R to host",
               "schedule": f"{n_str} calls streamed: H2D of call i+1 and D2H of call i-1 overlap call i "
                           "(copy streams); ms_per_step = total / calls",
               "serial": {"value": m * k / (ser_ms * 1e-3), "ms_per_step": ser_ms,
                          "schedule": "one call at a time: H2D, run, D2H, synchronize"},
               "pcie_floor_ms_per_step": floor_ms,
               "pcie_floor_note": "one H2D of the input concurrent with one D2H of Q through the same pinned "
                                  "buffers, measured in this run: the bound of a streamed call"}

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not ARGS.no_cpu:
        try:
            sec, sample = _cpu_run(cfg, cfg["cpu_rows"], 1)
            cpu = {"value": cfg["cpu_rows"] * k / sec, "unit": "rows*cols/s", "cores": os.cpu_count(),
                   "kind": "port", "sample": sample + f", {os.cpu_count()} BLAS threads"}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "rows*cols/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc!r}"}

    if rank == 0:
        line = {
            "metric": _metric(), "value": value, "unit": "rows*cols/s", "n_gpus": world,
            "steps": ARGS.steps, "warmup": ARGS.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": data,
            "config": {"workload": cfg["workload"], "rows": m, "cols": k, "algo": cfg["algo"],
                       "passes": passes, "shift_attempts": attempts,
                       "parallelism": f"row-sharded dp{world}",
                       "collective": "per pass: all-gather of the k x k partials + in-order device sum "
                                     "(deterministic)" if world > 1 else None,
                       "l2": "inputs larger than L2 (%.1f GB)" % (m * k * 8 / 1e9)},
            "quality": quality,
            "roofline": {"bound": "tensor", "pipe": "FP64 DMMA.8x8x4 (tensor pipe)", "kernel": dom, "achieved": tfs, "peak": FP64_PEAK_TFS,
                         "unit": "TFLOP/s", "frac": tfs / FP64_PEAK_TFS,
                         "traffic": _traffic(ARGS.config, lm[0] if lm else 0, k),
                         "traffic_note": "DRAM bytes per launch, ncu --set full (profiles/r01_ncu_summary.json); "
                                         "algorithmic: read X + write Q (+ read Q again where TRMM and Gram "
                                         "are separate launches, k > 64) = 2-3 m k 8 B",
                         "peak_source": FP64_PEAK_SRC, "kernel_share_of_step": step_share,
                         "kernel_timing": "CUDA events around each launch on its stream, over a second run of "
                                          "the same K steps (the headline region has no per-call events)",
                         "flops_model": "TRMM k(k+1) + SYRK k(k+1) flops per row"},
            "kernels": kernel_summary,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_update_chain(cq, cx, cfg, m, world, rank, local):
    """Config 4: 31 chained chol_qr_update calls (16 -> 512 columns).  Each
    new block is A_j = Q_prev C_j + 1e-8 G_j built from the algorithm's own
    Q_prev (BASELINE.json config 4); the timed quantity is the sum of the
    update calls' CUDA-event times (block generation between calls is not
    part of the update path)."""
    import torch
    import torch.distributed as dist

    p, nblk = cfg["p"], cfg["blocks"]
    space = cq.VectorSpace(m)
    gen = torch.Generator(device="cuda").manual_seed(SEED + rank)
    from paper_2507_07788_b200 import _device
    from paper_2507_07788_b200.workloads import device_gaussian

    g0 = device_gaussian(cq.CudaVectorArray.zeros(space, p), SEED + 17 * rank)
    base = cq.rs_chol_qr(g0)
    q0 = cq.CudaVectorArray.zeros(space, 0, capacity=p * (nblk + 1))
    q0.append(base.q)
    r0 = base.r
    hgen = np.random.default_rng(SEED)

    def chain(timer_events):
        q, r = q0.copy(), r0
        q.reserve(p * (nblk + 1))
        passes = []
        for j in range(nblk):
            c = hgen.standard_normal((q.ncols, p))
            a = q.lincomb(c)
            noise = cq.CudaVectorArray.zeros(space, p)
            device_gaussian(noise, int(hgen.integers(1 << 30)) + rank)
            a.axpy(1e-8, noise)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            res = cq.chol_qr_update(q, r, a)
            e1.record()
            timer_events.append((e0, e1))
            passes.append({"iterations": res.iterations, "shift_attempts": list(res.shift_attempts)})
            q, r = res.q, res.r
        return q, r, passes

    for _ in range(max(1, ARGS.warmup)):
        ev = []
        chain(ev)
    torch.cuda.synchronize()
    cx.timer = _device.KernelTimer()
    launches0 = cx.launches
    totals = []
    with ClockSampler(local) as clocks:
        for _ in range(ARGS.steps):
            ev = []
            q, r, passes = chain(ev)
            torch.cuda.synchronize()
            totals.append(sum(a.elapsed_time(b) for a, b in ev))
    ktimes = cx.timer.summary()
    cx.timer = None
    launches = (cx.launches - launches0) // ARGS.steps
    ms = float(np.mean(totals))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=cx.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = m * 512 / (ms * 1e-3)
    loo = cq.loss_of_orthogonality(q, norm="frobenius")
    # dominant kernel: the fused update pass; flops per launch
    up = ktimes.get("update_pass", {"ms": [1.0], "work": [(0, 0, 0, 0)]})
    fl = 0.0
    for rows_, qq, pp, init in up["work"]:
        fl += (2.0 * rows_ * qq * pp + rows_ * pp * (pp + 1)) * (1 if init else 2)
    tfs = fl / (sum(up["ms"]) * 1e-3) / 1e12
    # per-pass bound: the slower of HBM bytes and FP64 flops for every launch (the
    # initial pass of an append has half an iteration's flops on the same bytes and
    # is HBM-bound), summed over the chain, against the kernels' measured time
    hbm = _hbm_peak_gbs()
    bound_ms = 0.0
    for rows_, qq, pp, init in up["work"]:
        f_ = (2.0 * rows_ * qq * pp + rows_ * pp * (pp + 1)) * (1 if init else 2)
        b_ = 8.0 * rows_ * (qq + pp * (1 if init else 2))
        bound_ms += max(f_ / (FP64_PEAK_TFS * 1e12), b_ / (hbm * 1e9)) * 1e3
    per_pass = {"bound_ms_per_step": bound_ms / ARGS.steps, "kernel_ms_per_step": sum(up["ms"]) / ARGS.steps,
                "frac": bound_ms / sum(up["ms"]), "hbm_peak_gbs": hbm,
                "note": "sum over update-pass launches of max(flops / FP64 peak, bytes / HBM peak): initial passes "
                        "(Bt = Q_in^T A, G = A^T A) are HBM-bound, iteration passes FP64-bound"}
    cpu = None
    if rank == 0 and world == 1 and not ARGS.no_cpu:
        rows = cfg["cpu_rows"]
        sec = _cpu_update_chain(rows, cfg["blocks"])
        cpu = {"value": rows * 512 / sec, "unit": "rows*cols/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"oracle: 31 chol_qr_update calls on {rows} rows (16 -> 512 columns), block "
                         f"generation excluded, {os.cpu_count()} BLAS threads"}
    if rank == 0:
        print(json.dumps({
            "metric": _metric(), "value": value, "unit": "rows*cols/s", "n_gpus": world, "steps": ARGS.steps,
            "warmup": ARGS.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, built in HBM)",
            "config": {"workload": cfg["workload"], "rows": m, "cols": 512, "block": p, "blocks": nblk,
                       "parallelism": f"row-sharded dp{world}", "timed": "sum of update-call event times",
                       "per_block": passes[:3] + ["..."] + passes[-2:], "final_loo_fro": loo},
            "roofline": {"bound": "tensor", "pipe": "FP64 DMMA.8x8x4 (tensor pipe)", "kernel": "update_pass", "achieved": tfs, "peak": FP64_PEAK_TFS,
                         "unit": "TFLOP/s", "frac": tfs / FP64_PEAK_TFS, "traffic": None,
                         "peak_source": FP64_PEAK_SRC,
                         "flops_model": "2 m q p (projection) + 2 m q p (cross Gram) + 2 m p (p+1) per pass",
                         "per_pass_bound": per_pass},
            "kernels": {n: {"launches_per_step": len(v["ms"]) / ARGS.steps, "mean_ms": float(np.mean(v["ms"]))}
                        for n, v in ktimes.items()},
            "gpu_launches": launches, "clocks": clocks.summary(), "e2e": None, "cpu_baseline": cpu}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    if ARGS.impl == "reference":
        run_reference()
    else:
        run_ours()
