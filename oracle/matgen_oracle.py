"""Seeded test matrices -- TEST INFRASTRUCTURE ONLY (see cholqr_oracle.py).

Restates the reference's generator (`matgen.py:27-96`) so tests on the GPU
box (where `/root/reference` does not exist) can rebuild the reference's test
inputs bit-for-bit: seed mixed by splitmix64 over (m, n, round(10 log10_cond))
XOR the user seed, Haar factors from sign-fixed Householder QR of Gaussian
blocks, singular values log-spaced from 10^c down to 1.  Pinned against the
reference by `tests/test_oracle_golden.py::test_matgen_matches_reference`.
"""

from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1


def _mix(z):
    # splitmix64 finalizer (`matgen.py:27-31`)
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def spec_seed(m, n, log10_cond, seed=0):
    """`effective_seed` (`matgen.py:50-55`)."""
    acc = 0
    for v in (m, n, int(round(10 * log10_cond))):
        acc = _mix((acc + v) & _M64)
    return (acc ^ seed) & _M64


def haar(rows, cols, rng):
    """Sign-fixed Householder Q of a Gaussian block (`matgen.py:58-70`)."""
    q, r = np.linalg.qr(rng.standard_normal((rows, cols)))
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s


def sigmas(n, log10_cond):
    """10^c ... 1, log-equidistant (`matgen.py:73-81`)."""
    if n == 1:
        return np.ones(1)
    return 10.0 ** np.linspace(0.0, log10_cond, n)[::-1]


def generate(m, n, log10_cond, seed=0):
    """Dense m x n block A = U diag(sigma) V (`matgen.py:84-96`)."""
    rng = np.random.default_rng(spec_seed(m, n, log10_cond, seed))
    s = sigmas(n, log10_cond)
    u = haar(m, n, rng)
    v = haar(n, n, rng)
    return np.asfortranarray((u * s) @ v)


def with_zero_columns(block, cols):
    """Copy with the named columns zeroed (`tests/conftest.py:24-28`)."""
    out = np.array(block, dtype=float, copy=True)
    out[:, list(cols)] = 0.0
    return out
