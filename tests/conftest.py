"""Shared test setup.

Markers: `gpu` = needs a CUDA device (run on the B200 box with -m gpu);
everything else runs on the CPU build container.  The oracle (CPU restatement
of the reference, `oracle/`) is the checker for every parity test.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class Golden:
    """Golden vectors written by tests/golden/make_golden.py from the reference."""

    def __init__(self):
        with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
            self.meta = json.load(fh)
        self.arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
        self.cases = {c["name"]: c for c in self.meta["cases"]}

    def input(self, case):
        from oracle import matgen_oracle as mg

        if "spec" in case:
            m, n, x, seed, zero = case["spec"]
            blk = mg.generate(m, n, float(x), seed)
            return mg.with_zero_columns(blk, zero) if zero else blk
        return self.arrays[case["name"] + "__in"]

    def r(self, case):
        return self.arrays[case["name"] + "__r"]


@pytest.fixture(scope="session")
def golden():
    return Golden()


def oracle_cfg(case):
    from oracle import cholqr_oracle as co

    return co.default_cfg(**case.get("cfg", {}))


def algo_cfg(case):
    from paper_2507_07788_b200 import AlgoConfig

    return AlgoConfig(**case.get("cfg", {}))
