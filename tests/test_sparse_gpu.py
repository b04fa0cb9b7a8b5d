"""Parity of the sparse CSR CUDA path (SpMM pair X^T / X, Gram never formed) with the oracle.

The oracle runs Alg. 1 on the densified X (small cases) or the vector form on
sampled rows with scipy.sparse products (config-4 scale).  Bar: <= 1e-10 (fp64).
"""

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
    yield torch, P, h
    h.close()


def _dev(torch, row_ptr, col, val):
    return (torch.from_numpy(row_ptr).cuda(), torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda())


def _dense(row_ptr, col, val, m, n):
    X = np.zeros((m, n))
    for i in range(m):
        X[i, col[row_ptr[i]:row_ptr[i + 1]]] = val[row_ptr[i]:row_ptr[i + 1]]
    return X


@pytest.mark.parametrize("m,n,nnz,kind,K", [(40, 400, 800, "hard", 12), (100, 1000, 3000, "soft", 20),
                                            (33, 70, 500, "wsoft", 7), (1, 50, 10, "soft", 5),
                                            (64, 64, 400, "hard", 2), (70, 30, 300, "soft", 9)])
def test_sparse_vs_dense_oracle(env, m, n, nnz, kind, K):
    torch, P, h = env
    row_ptr, col, val = W.gen_c4(seed=m + n, m=m, n=n, nnz=nnz)
    kern = {"kind": kind, "tau": 0.4, "tau_relative": True, "w_c": 1.5, "w_shift": 0.0, "w_eps": 1e-6}
    Y, info = h.apply_csr(*_dev(torch, row_ptr, col, val), m, n, kern, K, T=60, info=True)
    X = _dense(row_ptr, col, val, m, n)
    if m > n:
        # the sparse path takes lambda on the m-side (X X^T), the dense oracle on the n-side: feed the same Lambda
        Yo = O.cpa_shrink(X, O.Kernel(**kern), K, lam=info["lambda_max"])
    else:
        Yo, io = O.cpa_shrink(X, O.Kernel(**kern), K, T=60, return_info=True)
        assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-12 * io["lambda_hat"]
    assert O.rel_fro(Y.cpu().numpy(), Yo) <= TOL64


def test_sparse_row_ranges_and_sampled_rows(env):
    import scipy.sparse as sp
    torch, P, h = env
    m, n, nnz = 2000, 20000, 40000
    row_ptr, col, val = W.gen_c4(seed=4, m=m, n=n, nnz=nnz)
    kern = W.CONFIGS["c4"]["kernel"]
    d = _dev(torch, row_ptr, col, val)
    Yfull, info = h.apply_csr(*d, m, n, kern, 30, T=300, info=True)
    Yfull = Yfull.cpu().numpy()
    Xs = sp.csr_matrix((val, col, row_ptr), shape=(m, n))
    rows = [0, 1, 31, 32, 777, 1999]
    Yo, io = O.cpa_shrink_sparse_rows(Xs, rows, O.Kernel(**kern), 30, T=300)
    assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-12 * io["lambda_hat"]
    assert O.rel_fro(Yfull[rows], Yo) <= TOL64
    # a rank's row range [r0, r1) equals the same rows of the full result (bitwise: same sums)
    r0, r1 = 37, 1001
    Ypart = h.apply_csr(*d, m, n, kern, 30, T=300, row_begin=r0, row_end=r1).cpu().numpy()
    assert np.array_equal(Ypart, Yfull[r0:r1])


def test_sparse_zero_and_deterministic(env):
    torch, P, h = env
    m, n = 50, 300
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    col = np.zeros(0, dtype=np.int32)
    val = np.zeros(0)
    Y, info = h.apply_csr(*_dev(torch, row_ptr, col, val), m, n, {"kind": "soft", "tau": 1.0}, 5, T=10, info=True)
    assert info["degenerate"] == 1 and not Y.cpu().numpy().any()
    row_ptr, col, val = W.gen_c4(seed=9, m=300, n=3000, nnz=9000)
    d = _dev(torch, row_ptr, col, val)
    a = h.apply_csr(*d, 300, 3000, {"kind": "soft", "tau": 0.2, "tau_relative": True}, 10, T=50).cpu().numpy()
    b = h.apply_csr(*d, 300, 3000, {"kind": "soft", "tau": 0.2, "tau_relative": True}, 10, T=50).cpu().numpy()
    assert np.array_equal(a, b)


@pytest.mark.slow
def test_config4_full_size_sampled(env):
    """BASELINE configs[3] at full size (20000 x 200000, nnz 4e6, K = 30, T = 300):
    64 sampled rows (seed-fixed, plus first and last) against the oracle's vector form."""
    import scipy.sparse as sp
    torch, P, h = env
    cfg = W.CONFIGS["c4"]
    m, n = cfg["m"], cfg["n"]
    row_ptr, col, val = W.gen_c4()
    Y, info = h.apply_csr(*_dev(torch, row_ptr, col, val), m, n, cfg["kernel"], cfg["K"], T=cfg["T"], info=True)
    rng = np.random.default_rng(0)
    rows = sorted(set([0, m - 1] + list(rng.choice(m, 62, replace=False))))
    Ys = Y[torch.tensor(rows, device=Y.device)].cpu().numpy()
    del Y
    Xs = sp.csr_matrix((val, col, row_ptr), shape=(m, n))
    Yo, io = O.cpa_shrink_sparse_rows(Xs, rows, O.Kernel(**cfg["kernel"]), cfg["K"], T=cfg["T"])
    assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-12 * io["lambda_hat"]
    assert O.rel_fro(Ys, Yo) <= TOL64


def test_raw_coefficients_sparse():
    """P8 on the sparse path: raw coefficients (2, 0, ...) give Y = X's rows, (Lambda, Lambda/2, 0, ...)
    give the rows of X X^T X (one SpMM pair), e_k gives X Psi_k(B_hat) (oracle)."""
    import scipy.sparse as sp
    import torch
    import paper_1705_07112_b200 as P
    m, n = 60, 500
    rp, col, val = W.gen_c4(m=m, n=n, nnz=1500, seed=5)
    Xs = sp.csr_matrix((val, col, rp), shape=(m, n))
    Xd = Xs.toarray()
    lam = 2.0 * float(np.linalg.norm(Xd, 2)) ** 2
    d = [torch.from_numpy(a).cuda() for a in (rp, col, val)]
    h = P.Handle(0)
    Y = h.apply_csr(*d, m, n, None, 4, lambda_max=lam, coeffs=[2.0, 0.0, 0.0, 0.0]).cpu().numpy()
    assert O.rel_fro(Y, Xd) <= 1e-14
    Y = h.apply_csr(*d, m, n, None, 4, lambda_max=lam, coeffs=[lam, lam / 2, 0.0, 0.0]).cpu().numpy()
    assert O.rel_fro(Y, Xd @ Xd.T @ Xd) <= 1e-13
    for kk in (2, 3, 5):
        c = [0.0] * 6
        c[kk] = 1.0
        Y = h.apply_csr(*d, m, n, None, 6, lambda_max=lam, coeffs=c).cpu().numpy()
        assert O.rel_fro(Y, O.cpa_shrink(Xd, None, 6, lam=lam, coeffs=c)) <= 1e-12
    h.close()


@pytest.mark.parametrize("K", [3, 4, 5, 6, 7, 8, 11, 13])
def test_sparse_grouped_y_updates(env, K):
    """Y += c_j W_j grouped over three steps (Y read and written every third step, the last step
    flushing the rest; reading R30) against the per-step updates (CPA_SVT_SP_YEVERY=1, Alg. 1's
    order) at rounding level and the oracle at the fp64 bar, for every residue of K."""
    import os
    torch, P, h = env
    m, n = 60, 500
    row_ptr, col, val = W.gen_c4(seed=K, m=m, n=n, nnz=1500)
    kern = {"kind": "soft", "tau": 0.3, "tau_relative": True}
    args = _dev(torch, row_ptr, col, val)
    Y = h.apply_csr(*args, m, n, kern, K, T=60).cpu().numpy()
    os.environ["CPA_SVT_SP_YEVERY"] = "1"
    try:
        Ye = h.apply_csr(*args, m, n, kern, K, T=60).cpu().numpy()
    finally:
        os.environ.pop("CPA_SVT_SP_YEVERY", None)
    Yo = O.cpa_shrink(_dense(row_ptr, col, val, m, n), O.Kernel(**kern), K, T=60)
    assert O.rel_fro(Y, Ye) <= 1e-13
    assert O.rel_fro(Y, Yo) <= TOL64
