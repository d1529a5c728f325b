"""Matrix Market dense files for device arrays (reference varray.py:291-356).

Format contract (kept byte for byte): header `%%MatrixMarket matrix array real
general`, a size line `m k`, then the values column by column, one per line, as
Python's shortest round-trip `repr(float)`.  So a file written here is the file
the reference writes for the same values, and rewriting a loaded file is
byte-identical (reference tests/test_varray.py:226-232).

Device arrays are downloaded and written a column block at a time, and files
are parsed with NumPy's correctly rounded string conversion, then uploaded.
"""

from __future__ import annotations

import numpy as np

HEADER = "%%MatrixMarket matrix array real general"
_COLS_PER_BLOCK = 64


def to_dense_block(array):
    """m x k float64 block of any array (varray.py:291-301)."""
    if array.ncols == 0:
        return np.zeros((array.space.dim, 0))
    return np.asarray(array.to_numpy(), dtype=float)


def format_values(block):
    """The value lines of an m x k block (column-major), newline-terminated."""
    block = np.asarray(block, dtype=float)
    if block.size == 0:
        return ""
    return "\n".join(map(repr, block.ravel(order="F").tolist())) + "\n"


def write_block(fh, block):
    m, k = block.shape
    fh.write(f"{HEADER}\n{m} {k}\n")
    fh.write(format_values(block))


def save_matrix_market(array, path):
    """Write an array (or a NumPy block) as a dense real general Matrix Market file."""
    if isinstance(array, np.ndarray):
        with open(path, "w") as fh:
            write_block(fh, array)
        return
    m, k = array.space.dim, array.ncols
    with open(path, "w") as fh:
        fh.write(f"{HEADER}\n{m} {k}\n")
        if k == 0:
            return
        for j0 in range(0, k, _COLS_PER_BLOCK):
            j1 = min(k, j0 + _COLS_PER_BLOCK)
            part = array.copy(list(range(j0, j1))) if (j0, j1) != (0, k) else array
            fh.write(format_values(to_dense_block(part)))


def parse_matrix_market(path):
    """(m, k, column-major values) of a dense real general file; ValueError on bad input."""
    with open(path) as fh:
        header = fh.readline().strip()
        words = header.lower().split()
        if words[:1] != ["%%matrixmarket"] or words[1:] != ["matrix", "array", "real", "general"]:
            raise ValueError(f"unsupported Matrix Market header (need dense real general): {header!r}")
        size = None
        values = []
        for raw in fh:
            line = raw.strip()
            if not line or line.startswith("%"):
                continue
            if size is None:
                parts = line.split()
                if len(parts) != 2:
                    raise ValueError(f"malformed size line: {line!r}")
                size = (int(parts[0]), int(parts[1]))
                continue
            values.append(line)
    if size is None:
        raise ValueError("missing size line")
    m, k = size
    if len(values) != m * k:
        raise ValueError(f"expected {m * k} values, found {len(values)}")
    try:
        data = np.array(values, dtype=np.float64)
    except ValueError:
        data = np.array([float(v) for v in values], dtype=np.float64)   # Python's error for the bad token
    return m, k, data


def load_block(path):
    m, k, data = parse_matrix_market(path)
    return data.reshape((m, k), order="F")


def load_matrix_market(path, backend="cuda"):
    """Read a dense real general Matrix Market file into a device array."""
    from . import backend_class

    cls = backend_class(backend)
    return cls.from_numpy(load_block(path))
