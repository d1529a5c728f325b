"""C ABI checks that need no GPU: libcqr.so loads, exports exactly the
functions include/cqr.h declares, and the ctypes struct layouts match the
header (so the status record is parsed correctly)."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "cqr.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cqr_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2507_07788_b200 import _lib
    from paper_2507_07788_b200.build import build

    build()
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    names = _declared()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n


def test_python_binding_covers_the_header():
    from paper_2507_07788_b200 import _lib

    assert sorted(_lib.SIGNATURES) == _declared()


def test_abi_version(lib):
    assert lib.cqr_abi_version() == 10


def test_struct_layouts_match_header(tmp_path):
    """Compile a probe against include/cqr.h with gcc and compare every
    field offset with the ctypes mirror."""
    import subprocess

    from paper_2507_07788_b200 import _lib

    lines = []
    for cname, cls in (("cqr_factor_status", _lib.FactorStatus), ("cqr_factor_config", _lib.FactorConfig),
                      ("cqr_fixed_plan", _lib.FixedPlan)):
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    src = tmp_path / "probe.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "cqr.h"\nint main(void){'
                   + "".join(lines) + "return 0;}\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    table = {}
    for line in out:
        if line:
            name, field, val = line.split()
            table[(name, field)] = int(val)
    for cname, cls in (("cqr_factor_status", _lib.FactorStatus), ("cqr_factor_config", _lib.FactorConfig),
                      ("cqr_fixed_plan", _lib.FixedPlan)):
        assert table[(cname, "size")] == ctypes.sizeof(cls)
        for f, _ in cls._fields_:
            assert table[(cname, f)] == getattr(cls, f).offset, (cname, f)


def test_workspace_queries_without_gpu(lib):
    # pure host planning functions
    assert lib.cqr_factor_workspace_bytes(64) >= 64 * 64 * 8
    assert lib.cqr_apply_gram_inplace_ok(64) == 1


def test_product_has_no_oracle_dependency():
    pkg = os.path.join(ROOT, "paper_2507_07788_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), f
