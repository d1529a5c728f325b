"""Build libcqr.so in-tree with nvcc for sm_100a (no torch JIT, no cache dir).

    python -m paper_2507_07788_b200.build        # or __graft_entry__.build()

Each csrc/*.cu compiles to its own object in parallel (the kernel files share
no device symbols), then one nvcc link makes the shared library.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libcqr.so")
OBJ = os.path.join(HERE, "build_obj")
SOURCES = ["cqr_abi.cu", "cqr_gram.cu", "cqr_gram_pairs.cu", "cqr_gemm.cu", "cqr_layout.cu", "cqr_fused.cu",
           "cqr_update.cu", "cqr_factor.cu", "cqr_small.cu", "cqr_device.cu", "cqr_metrics.cu",
           "cqr_schedule.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    *ARCH,
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "cqr.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, defines=(), objdir=OBJ):
    obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
    cmd = [NVCC, *FLAGS, *["-D" + d for d in defines], "-I", INCLUDE, "-c", "-o", obj, os.path.join(CSRC, src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return src, obj, res


def build(force=False, verbose=False, defines=(), out=None):
    """Compile every .cu of csrc/ (in parallel) and link one shared library.
    `defines` / `out`: a diagnostic variant (e.g. CQR_L2_HINTS=0) written to
    another path (the product library is always built without them)."""
    lib = out or LIB
    if not force and not defines and out is None and not _stale():
        return LIB
    objdir = OBJ if not defines else OBJ + "_" + "_".join(d.replace("=", "") for d in defines)
    os.makedirs(objdir, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as pool:
        results = list(pool.map(lambda src: _compile(src, defines, objdir), SOURCES))
    report = []
    failed = False
    for src, _obj, res in results:
        report.append(f"==== {src}\n{res.stdout}{res.stderr}")
        if res.returncode != 0:
            failed = True
            sys.stderr.write(f"nvcc failed on {src}:\n{res.stdout}{res.stderr}")
    if verbose and not failed:
        sys.stderr.write("".join(report))
    if failed:
        raise RuntimeError("nvcc failed building libcqr.so")
    link = [NVCC, *ARCH, "-shared", "-o", lib] + [obj for _src, obj, _res in results]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libcqr.so")
    if lib == LIB:
        with open(os.path.join(HERE, "ptxas_report.txt"), "w") as fh:
            fh.write("".join(report))
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
