"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module is the ONLY code both the oracle side and the CUDA side are fed
from.  It holds no arithmetic of the method (no Gram, no coefficients, no
recurrence): it only draws matrices.  Recipes follow BASELINE.json ``configs``
with the readings listed in DESIGN.md §"Input recipe":
every draw uses ``numpy.random.default_rng(seed)`` (PCG64), seed 0 by default,
in the order the recipe lists, ``N()`` = ``rng.standard_normal``.

The paper's own data (the Bricks / Office-windows textures and the Laboratory
video) is not available; these synthetic workloads stand in
for it (DESIGN.md §"Input recipe").
"""

from __future__ import annotations

import numpy as np

# Kernel descriptions are plain dicts: {"kind", "tau", "tau_relative", "w_c", "w_shift", "w_eps"}.
SOFT_2 = {"kind": "soft", "tau": 2.0, "tau_relative": False}

CONFIGS = {
    # configs[0]: 64x48 fp64, rank-5 + 0.1 noise, soft tau = 2.0, K = 20, T = 30
    "c1": {"path": "dense", "m": 64, "n": 48, "dtype": "f64", "K": 20, "T": 30,
           "kernel": {"kind": "soft", "tau": 2.0, "tau_relative": False}},
    # configs[1]: 1024^2 fp64, rank-20 (var 1/sqrt 20) + 0.1 noise, soft tau = 0.05 sigma_max_hat, K = 30
    "c2": {"path": "dense", "m": 1024, "n": 1024, "dtype": "f64", "K": 30, "T": 300,
           "kernel": {"kind": "soft", "tau": 0.05, "tau_relative": True}},
    # configs[2]: 65536 x [64x64] fp32 patch groups, weighted soft w = 2.8*sqrt(64)/(sigma + 1e-6), K = 20
    "c3": {"path": "batched", "batch": 65536, "m": 64, "n": 64, "dtype": "f32", "K": 20, "T": 30,
           "kernel": {"kind": "wsoft", "w_c": 2.8 * 8.0, "w_shift": 0.0, "w_eps": 1e-6}},
    # configs[3]: CSR 20000 x 200000, 0.1% density, N(0,1), hard tau = 0.5 sigma_max_hat, K = 30
    "c4": {"path": "sparse", "m": 20000, "n": 200000, "nnz": 4_000_000, "dtype": "f64", "K": 30, "T": 300,
           "kernel": {"kind": "hard", "tau": 0.5, "tau_relative": True}},
    # configs[4]: 16384 x 65536 rank-50 (var 1/sqrt 50) + 0.01 noise, soft tau = 0.1 sigma_max_hat, K = 40
    "c5": {"path": "dense", "m": 16384, "n": 65536, "dtype": "f64", "K": 40, "T": 300,
           "kernel": {"kind": "soft", "tau": 0.1, "tau_relative": True}},
}


def lowrank_plus_noise(m: int, n: int, r: int, a_var: float, noise: float, seed: int = 0) -> np.ndarray:
    """X = A B^T + noise * E, A (m x r), B (n x r) with entries of variance a_var.

    Draw order A, B, E (reading R14).  'N(0, v)' in BASELINE is read as variance v
    (reading R11), so entries are scaled by a_var ** 0.5.
    """
    rng = np.random.default_rng(seed)
    sd = a_var ** 0.5
    A = rng.standard_normal((m, r)) * sd
    B = rng.standard_normal((n, r)) * sd
    E = rng.standard_normal((m, n))
    return A @ B.T + noise * E


def gen_c1(seed: int = 0) -> np.ndarray:
    """configs[0]: 64 x 48, rank-5 N(0,1) product + 0.1 N(0,1)."""
    return lowrank_plus_noise(64, 48, 5, 1.0, 0.1, seed)


def gen_c2(seed: int = 0, m: int = 1024, n: int = 1024) -> np.ndarray:
    """configs[1]: rank-20 product with factor variance 1/sqrt(20), + 0.1 N(0,1)."""
    return lowrank_plus_noise(m, n, 20, 20 ** -0.5, 0.1, seed)


def gen_c5(seed: int = 0, m: int = 16384, n: int = 65536, dtype=np.float64) -> np.ndarray:
    """configs[4]: rank-50 product with factor variance 1/sqrt(50), + 0.01 N(0,1).

    Generated in row blocks so the fp64 temporaries stay bounded; the stream of
    draws is A, B, then E row-major, identical to one big draw.
    """
    rng = np.random.default_rng(seed)
    sd = (50 ** -0.5) ** 0.5
    A = rng.standard_normal((m, 50)) * sd
    B = rng.standard_normal((n, 50)) * sd
    X = np.empty((m, n), dtype=dtype)
    blk = max(1, (1 << 26) // n)
    for i in range(0, m, blk):
        j = min(m, i + blk)
        E = rng.standard_normal((j - i, n))
        X[i:j] = A[i:j] @ B.T + 0.01 * E
    return X


def gen_c3(batch: int = 65536, seed: int = 0, m: int = 64, n: int = 64, rank: int = 3) -> np.ndarray:
    """configs[2]: per matrix a rank-3 N(0,1) product, min-max scaled to [0,1] per matrix,
    plus 0.05 N(0,1) noise; returned as float32 [batch, m, n] (reading R12)."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((batch, m, rank))
    B = rng.standard_normal((batch, n, rank))
    P = A @ B.transpose(0, 2, 1)
    lo = P.min(axis=(1, 2), keepdims=True)
    hi = P.max(axis=(1, 2), keepdims=True)
    P = (P - lo) / (hi - lo)
    out = np.empty((batch, m, n), dtype=np.float32)
    blk = 4096
    for i in range(0, batch, blk):
        j = min(batch, i + blk)
        E = rng.standard_normal((j - i, m, n))
        out[i:j] = (P[i:j] + 0.05 * E).astype(np.float32)
    return out


def gen_c4(seed: int = 0, m: int = 20000, n: int = 200000, nnz: int = 4_000_000):
    """configs[3]: CSR with exactly nnz distinct uniformly random positions, values N(0,1).

    Returns (row_ptr int64[m+1], col int32[nnz], val float64[nnz]) with column
    indices sorted within each row (reading R13).
    """
    rng = np.random.default_rng(seed)
    draw = int(nnz * 1.025) + 1024
    while True:
        pos = np.unique(rng.integers(0, m * n, draw, dtype=np.int64))
        if pos.size >= nnz:
            break
        draw *= 2
    keep = np.sort(pos[rng.choice(pos.size, nnz, replace=False)])
    rows, cols = np.divmod(keep, n)
    val = rng.standard_normal(nnz)
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return row_ptr, cols.astype(np.int32), val


def block_diag_D(N: int, nblocks: int, ncopies: int = 1) -> np.ndarray:
    """The paper's synthetic matrix D = J - blkdiag(0.5 1 1^T, n).

    N x N with nblocks diagonal blocks of size N/nblocks; ``ncopies`` > 1 returns
    the wide matrix [D D ... D] (N x ncopies*N, unscaled).
    """
    if N % nblocks:
        raise ValueError("nblocks must divide N")
    p = N // nblocks
    D = np.ones((N, N))
    for b in range(nblocks):
        D[b * p:(b + 1) * p, b * p:(b + 1) * p] -= 0.5
    if ncopies > 1:
        D = np.concatenate([D] * ncopies, axis=1)
    return D


def random_dense(m: int, n: int, seed: int = 0, dtype=np.float64) -> np.ndarray:
    """Plain N(0,1) matrix (odd-shape parity cases)."""
    return np.random.default_rng(seed).standard_normal((m, n)).astype(dtype)


def gen_pinpaint(seed: int = 0, m: int = 2560, n: int = 1920) -> np.ndarray:
    """Context shape (not a BASELINE config, SURVEY 8d 'p-inpaint'): a stand-in for one
    2560 x 1920 colour channel of the paper's texture images, values in
    [0, 1]: three separable 2-D cosines with random frequencies and phases (DCT-sparse and
    low rank), min-max scaled, plus N(0, 0.02^2).  Seeded; no arithmetic of the method."""
    rng = np.random.default_rng(seed)
    i = np.arange(m)[:, None]
    j = np.arange(n)[None, :]
    X = np.zeros((m, n))
    for _ in range(3):
        fi, fj = rng.uniform(0.002, 0.05, 2)
        pi, pj = rng.uniform(0, 2 * np.pi, 2)
        X += rng.uniform(0.5, 1.0) * np.cos(2 * np.pi * fi * i + pi) * np.cos(2 * np.pi * fj * j + pj)
    X = (X - X.min()) / (X.max() - X.min())
    return X + 0.02 * rng.standard_normal((m, n))


def gen_pvideo(seed: int = 0, h: int = 360, w: int = 240, frames: int = 5000, blocks: int = 173) -> np.ndarray:
    """Context shape (not a BASELINE config, SURVEY 8d 'p-video'): a stand-in for the paper's
    86400 x 5000 background-modeling matrix (pixels x frames, values in
    [0, 1]): a rank-1 static background (a smooth [0, 1] frame repeated in every column) plus
    `blocks` 5 x 5 foreground blocks per frame (~5% of the pixels) moving at constant
    velocities, set to random [0, 1] values.  Seeded; no arithmetic of the method."""
    rng = np.random.default_rng(seed)
    yy, xx = np.meshgrid(np.arange(h), np.arange(w), indexing="ij")
    bg = np.zeros((h, w))
    for _ in range(4):
        fy, fx = rng.uniform(0.002, 0.02, 2)
        bg += rng.uniform(0.5, 1.0) * np.cos(2 * np.pi * fy * yy + rng.uniform(0, 6.3)) * np.cos(
            2 * np.pi * fx * xx + rng.uniform(0, 6.3))
    bg = (bg - bg.min()) / (bg.max() - bg.min())
    X = np.repeat(bg.reshape(-1, 1), frames, axis=1)             # (h w) x frames, Fortran-free copy
    y0, x0 = rng.uniform(0, h, blocks), rng.uniform(0, w, blocks)
    vy, vx = rng.uniform(-0.5, 0.5, blocks), rng.uniform(-0.5, 0.5, blocks)
    dy, dx = np.meshgrid(np.arange(5), np.arange(5), indexing="ij")
    for t in range(frames):
        py = (np.floor(y0 + vy * t).astype(np.int64) % (h - 5))[:, None] + dy.reshape(1, -1)
        px = (np.floor(x0 + vx * t).astype(np.int64) % (w - 5))[:, None] + dx.reshape(1, -1)
        X[(py * w + px).ravel(), t] = rng.random(blocks * 25)
    return X


def synthetic_D(N: int, rank: int) -> np.ndarray:
    """The paper's synthetic data: D = J - blkdiag(0.5 1 1^T) with `rank`
    diagonal blocks of size N / rank.  Deterministic; no arithmetic of the method."""
    p = N // rank
    D = np.ones((N, N))
    for b in range(rank):
        D[b * p:(b + 1) * p, b * p:(b + 1) * p] -= 0.5
    return D


def gen_c3_closed_form(batch: int = 65536, seed: int = 0, n: int = 64, n_scales: int = 256):
    """Closed-form stand-ins for the c3 batch (full-scale checks without the oracle per matrix):
    matrix b has scale a = scales[b % n_scales] (uniform in [0.5, 20]);
      even b: X_b = a Q_b, Q_b a random orthogonal n x n matrix (QR of a Gaussian draw, signs fixed);
      odd b:  X_b = a diag(ratios) with the fixed ratios (1, then uniform in [0.05, 0.5]) -- a
              dominant first entry so the power iteration converges in a few steps.
    Returns (X float32 [batch, n, n], scales float64 [n_scales], ratios float64 [n]).  No arithmetic
    of the method; the expected outputs come from the oracle's series (tests)."""
    rng = np.random.default_rng(seed)
    scales = rng.uniform(0.5, 20.0, n_scales)
    ratios = np.concatenate([[1.0], rng.uniform(0.05, 0.5, n - 1)])
    X = np.zeros((batch, n, n), dtype=np.float32)
    ne = (batch + 1) // 2
    blk = 4096
    for i in range(0, ne, blk):
        j = min(ne, i + blk)
        q, r = np.linalg.qr(rng.standard_normal((j - i, n, n)))
        q = q * np.sign(np.diagonal(r, axis1=1, axis2=2))[:, None, :]
        b = 2 * np.arange(i, j)
        X[b] = (scales[b % n_scales][:, None, None] * q).astype(np.float32)
    b = np.arange(1, batch, 2)
    idx = np.arange(n)
    X[b[:, None], idx[None, :], idx[None, :]] = (scales[b % n_scales][:, None] * ratios[None, :]).astype(np.float32)
    return X, scales, ratios
