"""Seeded random sweep of shapes, orders, kernels and power-iteration lengths against the oracle.

Every case is drawn from a fixed seed (deterministic test ids): dense fp64 (both sides, ragged tile
counts, every dense form the automatic choice reaches: the single-block kernel, the two-chain and
one-chain persistent recurrences, line 12 folded or separate, the host pipeline), 3xTF32, the
batched tcgen05 kernel and the sparse SpMM pair -- each against the plain oracle at the north-star
bars (fp64 1e-10, fp32 1e-4 relative Frobenius).
"""

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu
KINDS = ("hard", "soft", "wsoft")


def _case(seed, smax, lmax):
    rng = np.random.default_rng(10_000 + seed)
    s = int(rng.integers(1, smax + 1))
    L = int(rng.integers(s, lmax + 1))
    m, n = (s, L) if rng.random() < 0.5 else (L, s)
    K = int(rng.choice([2, 3, 4, 5, 7, 12, 20, 31, 40]))
    T = int(rng.choice([20, 30, 100, 300]))   # (short iterations: tests of their own, divergence tests)
    kind = KINDS[int(rng.integers(0, 3))]
    kern = {"kind": kind, "tau": float(rng.uniform(0.05, 0.6)), "tau_relative": True,
            "w_c": float(rng.uniform(0.5, 4.0)), "w_shift": 0.0, "w_eps": 1e-6}
    rank = int(rng.integers(1, max(2, s // 2) + 1))
    A = rng.standard_normal((m, rank))
    B = rng.standard_normal((n, rank))
    X = A @ B.T / np.sqrt(rank) + 0.1 * rng.standard_normal((m, n))
    return X, kern, K, T


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_07112_b200 as P
    h = P.Handle(0)
    yield torch, P, h
    h.close()


def _check(Y, X, kern, K, T, tol, info=None):
    Yo, io = O.cpa_shrink(X, O.Kernel(**kern), K, T=T, return_info=True)
    err = O.rel_fro(Y, Yo)
    assert err <= tol, (X.shape, kern["kind"], K, T, err)
    if info is not None and not io["degenerate"]:
        assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-9 * io["lambda_hat"]


@pytest.mark.parametrize("seed", list(range(40)) + list(range(200, 260)))
def test_fuzz_dense_f64(env, seed):
    torch, P, h = env
    X, kern, K, T = _case(seed, 300 if seed < 200 else 760, 700 if seed < 200 else 1400)
    try:
        Y, info = h.apply(torch.from_numpy(X).cuda(), kern, K, T=T, info=True)
    except P.CpaSvtError as e:   # only acceptable where the oracle's series diverges as well
        assert e.status == 3
        Yo, io = O.cpa_shrink(X, O.Kernel(**kern), K, T=T, return_info=True)
        assert np.linalg.norm(Yo) > 1e3 * sum(abs(c) for c in io["coeffs"]) * np.linalg.norm(X)
        return
    _check(Y.cpu().numpy(), X, kern, K, T, 1e-10, info)


@pytest.mark.parametrize("seed", range(40, 52))
def test_fuzz_dense_f64_host_pipeline(env, seed):
    torch, P, h = env
    X, kern, K, T = _case(seed, 260, 600)
    Xh = torch.from_numpy(X).pin_memory()
    Yh = torch.empty_like(Xh).pin_memory()
    h.apply_host(Xh, Yh, kern, K, T=T)
    _check(Yh.numpy(), X, kern, K, T, 1e-10)


@pytest.mark.parametrize("seed", range(60, 76))
def test_fuzz_3xtf32(env, seed):
    torch, P, h = env
    X, kern, K, T = _case(seed, 200, 500)
    X32 = X.astype(np.float32)
    Y = h.apply(torch.from_numpy(X32).cuda(), kern, K, T=T, math="3xtf32")
    _check(Y.double().cpu().numpy(), X32.astype(np.float64), kern, K, T, 1e-4)


@pytest.mark.parametrize("seed", range(80, 92))
def test_fuzz_batched(env, seed):
    torch, P, h = env
    rng = np.random.default_rng(20_000 + seed)
    m, n = int(rng.integers(1, 65)), int(rng.integers(1, 65))
    K = int(rng.choice([2, 3, 5, 12, 20, 33]))
    T = int(rng.choice([1, 5, 8, 30]))
    kind = KINDS[int(rng.integers(0, 3))]
    kern = {"kind": kind, "tau": 0.3, "tau_relative": True, "w_c": 2.0, "w_shift": 0.0, "w_eps": 1e-6}
    Xb = rng.standard_normal((int(rng.integers(1, 300)), m, n)).astype(np.float32)
    Y = h.apply_batched(torch.from_numpy(Xb).cuda(), kern, K, T=T).cpu().numpy()
    idx = sorted(set([0, Xb.shape[0] - 1] + list(rng.choice(Xb.shape[0], min(12, Xb.shape[0]), replace=False))))
    Yo, _ = O.cpa_shrink_batched(Xb[idx].astype(np.float64), O.Kernel(**kern), K, T=T)
    assert O.rel_fro(Y[idx].astype(np.float64), Yo) <= 1e-4, (Xb.shape, kind, K, T)


@pytest.mark.parametrize("seed", range(100, 108))
def test_fuzz_sparse(env, seed):
    import scipy.sparse as sp
    torch, P, h = env
    rng = np.random.default_rng(30_000 + seed)
    m = int(rng.integers(2, 150))
    n = int(rng.integers(m, 3000))
    nnz = int(rng.integers(1, min(m * n, 6000) + 1))
    K = int(rng.choice([2, 3, 7, 12, 30]))
    kind = KINDS[int(rng.integers(0, 3))]
    kern = {"kind": kind, "tau": 0.4, "tau_relative": True, "w_c": 2.0, "w_shift": 0.0, "w_eps": 1e-6}
    rp, col, val = W.gen_c4(seed=seed, m=m, n=n, nnz=nnz)
    rb = int(rng.integers(0, m))
    re_ = int(rng.integers(rb, m + 1))
    Ys = h.apply_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda(), m, n,
                     kern, K, T=60, row_begin=rb, row_end=re_).cpu().numpy()
    Xs = sp.csr_matrix((val, col, rp), shape=(m, n))
    Yo, _ = O.cpa_shrink_sparse_rows(Xs, list(range(rb, re_)), O.Kernel(**kern), K, T=60)
    if re_ > rb:
        assert O.rel_fro(Ys, Yo) <= 1e-10, (m, n, nnz, kind, K, rb, re_)
