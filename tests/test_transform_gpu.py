"""Parity of the NEXT-2 transform variant (Alg. 1 with T = one-level Haar DWT of the Gram
index, high-frequency components of Phi set to 0, reading R22)
with the oracle's literal Alg. 1 (explicit T, Phi = T B^T B T^T, zeroed band, line 12
B T^T H_hat T).  Bar: fp64, relative Frobenius <= 1e-10."""

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu
TOL64 = 1e-10


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_07112_b200 as P
    h = P.Handle(0)
    h.set_transform("haar1")
    yield torch, P, h
    h.close()


@pytest.mark.parametrize("shape", [(64, 128), (128, 64), (65, 200), (200, 65), (1, 9), (2, 2), (3, 3), (257, 1000),
                                   (1000, 257), (1024, 1024)])
@pytest.mark.parametrize("kind,K", [("soft", 2), ("soft", 20), ("hard", 7), ("wsoft", 12)])
def test_transform_parity(env, shape, kind, K):
    torch, P, h = env
    X = W.gen_c2(m=shape[0], n=shape[1], seed=shape[0] + 7 * shape[1] + K)
    kern = {"kind": kind, "tau": 0.1, "tau_relative": True, "w_c": 2.0, "w_shift": 0.0, "w_eps": 1e-6}
    Y, info = h.apply(torch.from_numpy(X).cuda(), kern, K, T=200, info=True)
    Yo, io = O.cpa_shrink_transform(X, O.Kernel(**kern), K, T=200, return_info=True)
    assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-11 * max(io["lambda_hat"], 1e-300)
    assert O.rel_fro(Y.cpu().numpy(), Yo) <= TOL64, (shape, kind, K)


def test_transform_lowpass_matches_plain(env):
    """Pairwise-equal rows: no high band, the transform variant equals T = I (at a fixed
    Lambda; the power iterations start in different bases)."""
    torch, P, h = env
    base = np.random.default_rng(3).standard_normal((100, 300))
    X = np.repeat(base, 2, axis=0)
    kern = {"kind": "soft", "tau": 0.2, "tau_relative": True}
    lam = 1.01 * float(np.linalg.eigvalsh(X @ X.T)[-1])
    Yt = h.apply(torch.from_numpy(X).cuda(), kern, 15, lambda_max=lam).cpu().numpy()
    h2 = P.Handle(0)
    Yp = h2.apply(torch.from_numpy(X).cuda(), kern, 15, lambda_max=lam).cpu().numpy()
    h2.close()
    assert O.rel_fro(Yt, Yp) <= 1e-12


def test_transform_unsupported_paths(env):
    torch, P, h = env
    X = torch.zeros((8, 16), dtype=torch.float32, device="cuda")
    with pytest.raises(P.CpaSvtError) as e:
        h.apply(X, {"kind": "soft", "tau": 1.0}, 5, math="3xtf32")
    assert e.value.status == 7


# ---- DCT variant with component thresholding

def _gap_k(X, target, rel=1e-6, tmat=None):
    """A k near `target` where the k-th and (k+1)-th largest |Phi_ij| differ by more than `rel`
    relative: the kept set is then the same on both sides whatever the rounding of Phi."""
    m, n = X.shape
    B = X.T if m <= n else X
    Tm = (tmat or O.dct2_matrix)(B.shape[1])
    a = np.sort(np.abs(Tm @ (B.T @ B) @ Tm.T).ravel())[::-1]
    for d in range(0, a.size):
        for k in (target + d, target - d):
            if 1 <= k < a.size and a[k - 1] > a[k] * (1 + rel):
                return k
    raise AssertionError("no gap")


@pytest.fixture(scope="module")
def dct_env():
    import torch
    import paper_1705_07112_b200 as P
    h = P.Handle(0)
    h.set_transform("dct")
    yield torch, P, h
    h.close()


@pytest.mark.parametrize("shape", [(64, 128), (130, 70), (7, 9), (257, 300)])
@pytest.mark.parametrize("eps", [("none", 0), ("abs", 0.5), ("topk", 0.02), ("topk", 0.3)])
@pytest.mark.parametrize("kind,K", [("soft", 2), ("soft", 15), ("hard", 6)])
def test_dct_parity(dct_env, shape, eps, kind, K):
    torch, P, h = dct_env
    X = W.gen_c2(m=shape[0], n=shape[1], seed=shape[0] * 3 + shape[1] + K)
    mode, val = eps
    if mode == "topk":
        s = min(shape)
        val = _gap_k(X, max(1, int(val * s * s)))
    if mode == "abs":   # an absolute epsilon in a gap of |Phi|
        m, n = X.shape
        B = X.T if m <= n else X
        Tm = O.dct2_matrix(B.shape[1])
        a = np.sort(np.abs(Tm @ (B.T @ B) @ Tm.T).ravel())[::-1]
        k = _gap_k(X, max(1, a.size // 10))
        val = 0.5 * (a[k - 1] + a[k])
    h.set_epsilon(mode, val)
    kern = {"kind": kind, "tau": 0.1, "tau_relative": True}
    Y, info = h.apply(torch.from_numpy(X).cuda(), kern, K, T=200, info=True)
    Yo, io = O.cpa_shrink_transform(X, O.Kernel(**kern), K, T=200, return_info=True, transform="dct",
                                    eps_mode=None if mode == "none" else mode, eps=val)
    assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-11 * io["lambda_hat"]
    assert O.rel_fro(Y.cpu().numpy(), Yo) <= TOL64, (shape, eps, kind, K)


# ---- 8 x 8 block DCT (reading R24): ragged last blocks included

@pytest.fixture(scope="module")
def bdct_env():
    import torch
    import paper_1705_07112_b200 as P
    h = P.Handle(0)
    h.set_transform("dct8")
    yield torch, P, h
    h.close()


@pytest.mark.parametrize("shape", [(64, 128), (130, 70), (7, 9), (257, 300)])
@pytest.mark.parametrize("eps", [("none", 0), ("abs", 0.1), ("topk", 0.05)])
@pytest.mark.parametrize("kind,K", [("soft", 15), ("hard", 6)])
def test_block_dct_parity(bdct_env, shape, eps, kind, K):
    torch, P, h = bdct_env
    X = W.gen_c2(m=shape[0], n=shape[1], seed=shape[0] * 5 + shape[1] + K)
    mode, val = eps
    s = min(shape)
    if mode == "topk":
        val = _gap_k(X, max(1, int(val * s * s)), tmat=O.dct2_block_matrix)
    if mode == "abs":   # an absolute epsilon in a gap of |Phi|
        m, n = X.shape
        B = X.T if m <= n else X
        Tm = O.dct2_block_matrix(B.shape[1])
        a = np.sort(np.abs(Tm @ (B.T @ B) @ Tm.T).ravel())[::-1]
        k = _gap_k(X, max(1, int(val * a.size)), tmat=O.dct2_block_matrix)
        val = 0.5 * (a[k - 1] + a[k])
    h.set_epsilon(mode, val)
    kern = {"kind": kind, "tau": 0.1, "tau_relative": True}
    Y, info = h.apply(torch.from_numpy(X).cuda(), kern, K, T=200, info=True)
    Yo, io = O.cpa_shrink_transform(X, O.Kernel(**kern), K, T=200, return_info=True, transform="dct8",
                                    eps_mode=None if mode == "none" else mode, eps=val)
    assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-11 * io["lambda_hat"]
    assert O.rel_fro(Y.cpu().numpy(), Yo) <= TOL64, (shape, eps, kind, K)
