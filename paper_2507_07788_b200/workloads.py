"""Synthetic inputs of BASELINE.json's five configurations (seeded).

The reference benchmarks on synthetic matrices only; these builders follow
BASELINE.json's descriptions with singular values scaled
from 1 down to 10^-c.  `host_*` build NumPy blocks (used by the parity tests,
which feed the same bits to the CPU oracle); `device_*` build the large
bench inputs directly in HBM with torch (cuRAND / cuBLAS are input
generation here, outside every timed region).
"""

from __future__ import annotations

import numpy as np

CONFIGS = {
    1: dict(name="scholqr3_200000x64_k1e12", m=200_000, k=64, log10_cond=12.0, algo="s_chol_qr3"),
    2: dict(name="cholqr2_4000000x128_gauss", m=4_000_000, k=128, log10_cond=None, algo="chol_qr2"),
    3: dict(name="rscholqr_2000000x256_k1e15", m=2_000_000, k=256, log10_cond=15.0, algo="rs_chol_qr"),
    4: dict(name="update_8000000x(16+31x16)", m=8_000_000, k=16, blocks=31, algo="chol_qr_update"),
    5: dict(name="cholqr2_128000000x64_gauss", m=128_000_000, k=64, log10_cond=None, algo="chol_qr2"),
}


def _haar(rng, rows, cols):
    q, r = np.linalg.qr(rng.standard_normal((rows, cols)))
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s


def host_svd_matrix(m, k, log10_cond, seed, u_from="householder"):
    """X = U diag(sigma) V^T, sigma log-spaced 1 -> 10^-c (configs 1 and 3)."""
    rng = np.random.default_rng(seed)
    if u_from == "householder":
        u = _haar(rng, m, k)
    else:  # config 3: U = Q of CholeskyQR2 of Gaussian rows
        g = rng.standard_normal((m, k))
        for _ in range(2):
            r = np.linalg.cholesky(g.T @ g).T
            g = np.linalg.solve(r.T, g.T).T
        u = g
    v = _haar(rng, k, k)
    sigma = 10.0 ** np.linspace(0.0, -log10_cond, k)
    return np.asfortranarray((u * sigma) @ v.T)


def host_gaussian(m, k, seed):
    """i.i.d. N(0,1) (configs 2 and 5)."""
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((m, k)))


def host_config(cfg_id, m=None, seed=2025):
    c = CONFIGS[cfg_id]
    m = m or c["m"]
    if cfg_id == 1:
        return host_svd_matrix(m, c["k"], c["log10_cond"], seed)
    if cfg_id == 3:
        return host_svd_matrix(m, c["k"], c["log10_cond"], seed, u_from="cholqr2")
    if cfg_id in (2, 5):
        return host_gaussian(m, c["k"], seed)
    raise ValueError("config 4 is built block by block (update_blocks)")


def next_block(q_prev_host, rng, p=16, noise=1e-8):
    """Config 4: A_j = Q_prev C_j + 1e-8 G_j with C_j, G_j ~ N(0,1)."""
    m, q = q_prev_host.shape
    c = rng.standard_normal((q, p))
    g = rng.standard_normal((m, p))
    return np.asfortranarray(q_prev_host @ c + noise * g)


# ------------------------------------------------------------------ device builders (bench)
def device_svd_matrix(arr_factory, m, k, log10_cond, seed, u_from="householder"):
    """Same construction as host_svd_matrix, built in HBM with torch fp64."""
    import torch

    gen = torch.Generator(device="cuda").manual_seed(seed)
    g = torch.randn((m, k), generator=gen, dtype=torch.float64, device="cuda")
    if u_from == "householder":
        u, r = torch.linalg.qr(g)
        u = u * torch.sign(torch.diagonal(r))
    else:
        u = g
        for _ in range(2):
            r = torch.linalg.cholesky(u.T @ u).mH
            u = torch.linalg.solve_triangular(r, u, upper=True, left=False)
    v, rv = torch.linalg.qr(torch.randn((k, k), generator=gen, dtype=torch.float64, device="cuda"))
    v = v * torch.sign(torch.diagonal(rv))
    sigma = 10.0 ** torch.linspace(0.0, -log10_cond, k, dtype=torch.float64, device="cuda")
    x = (u * sigma) @ v.T
    return arr_factory(x)


def device_gaussian(arr, seed, chunk_quads=1 << 22):
    """Fill a device array (QI storage) with N(0,1), padding rows kept zero.
    The values are a function of the seed and the local shard only."""
    import torch

    gen = torch.Generator(device="cuda").manual_seed(seed)
    buf = arr._buf[:, : arr.ncols, :]
    nq = buf.shape[0]
    for q0 in range(0, nq, chunk_quads):
        buf[q0: q0 + chunk_quads].normal_(generator=gen)
    m = arr.m_local
    qa = m // 4
    if m % 4:
        buf[qa, :, m % 4:] = 0.0
        qa += 1
    buf[qa:] = 0.0
    return arr
