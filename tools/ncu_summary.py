"""Summarise ncu captures (.ncu-rep) into one JSON for profiles/.

    python tools/ncu_summary.py gpurun_out/prof/*.ncu-rep > profiles/r01_ncu_summary.json

Per capture: kernel, duration, DRAM bytes read/written (the `traffic` term of
bench.py's roofline), FP64 tensor-pipe (DMMA) activity, occupancy, registers
and the top warp-stall reasons.
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),        # ns -> ms (converted below by unit)
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dmma_pipe_active_pct": ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", None),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", None),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "registers_per_thread": ("launch__registers_per_thread", None),
    "grid_size": ("launch__grid_size", None),
    "block_size": ("launch__block_size", None),
    "smem_dynamic_bytes": ("launch__shared_mem_per_block_dynamic", None),
    "shared_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", None),
}
UNITS = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def summarise(rep):
    h, u, v = raw(rep)
    col = {n: i for i, n in enumerate(h)}
    d = {"capture": os.path.basename(rep), "kernel": v[col["Kernel Name"]] if "Kernel Name" in col else None}
    for key, (name, _) in METRICS.items():
        if name not in col:
            continue
        x = num(v[col[name]])
        unit = u[col[name]]
        if x is not None and key == "duration_ms":
            x *= UNITS.get(unit, 1e-6)
        elif x is not None and key.endswith("_bytes") and key != "smem_dynamic_bytes":
            x *= UNITS.get(unit, 1)
        d[key] = x
    stalls = {}
    for n, i in col.items():
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
            x = num(v[i])
            if x:
                stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = x
    tot = sum(stalls.values()) or 1.0
    d["stall_pct"] = {k: round(100 * x / tot, 1) for k, x in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
    return d


if __name__ == "__main__":
    print(json.dumps([summarise(r) for r in sys.argv[1:]], indent=1))
