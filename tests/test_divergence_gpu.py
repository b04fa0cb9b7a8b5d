"""Divergence detection (CPA_SVT_E_DIVERGED in include/cpa_svt.h).

The series is bounded only while the Gram spectrum lies in [0, Lambda_max]
(psi_k(x) = cos(k arccos x) on [-1, 1], cosh(k acosh x) beyond).
A Lambda_max override at a quarter of the true top eigenvalue puts B_hat's top
eigenvalue at 7, so ||Psi_K|| ~ 14^K and ||Y|| exceeds 1e3 sum|c_k| ||X||: every
path must report E_DIVERGED (status 3) when it synchronises, and stay silent on
healthy inputs and when the check is off.
"""

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
E_DIVERGED = 3


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_07112_b200 as P
    h = P.Handle(0)
    yield torch, P, h
    h.close()


def _lam_true(X):
    return float(np.linalg.norm(X, 2)) ** 2


@pytest.mark.parametrize("shape,dtype,math", [((300, 500), "f64", None), ((64, 48), "f64", None),
                                              ((700, 300), "f64", None), ((300, 500), "f32", "3xtf32"),
                                              ((300, 500), "f32", "tf32")])
def test_underestimated_lambda_diverges(env, shape, dtype, math):
    torch, P, h = env
    X = W.gen_c2(m=shape[0], n=shape[1], seed=1)
    Xd = torch.from_numpy(X.astype(np.float32) if dtype == "f32" else X).cuda()
    kern = {"kind": "soft", "tau": 0.1, "tau_relative": True}
    lam = 0.25 * _lam_true(X)
    with pytest.raises(P.CpaSvtError) as e:
        h.apply(Xd, kern, 20, lambda_max=lam, math=math, info=True)
    assert e.value.status == E_DIVERGED
    # healthy call on the same handle: the verdict is reset
    Y, info = h.apply(Xd, kern, 20, T=100, math=math, info=True)
    assert torch.isfinite(Y).all()
    # asynchronous call: no sync, no status; mode 'sync' reports it; 'off' never checks
    h.apply(Xd, kern, 20, lambda_max=lam, math=math)
    h.set_divergence("sync")
    try:
        with pytest.raises(P.CpaSvtError) as e:
            h.apply(Xd, kern, 20, lambda_max=lam, math=math)
        assert e.value.status == E_DIVERGED
        h.apply(Xd, kern, 20, T=100, math=math)
        h.set_divergence("off")
        h.apply(Xd, kern, 20, lambda_max=lam, math=math, info=True)
    finally:
        h.set_divergence("on")


def test_apply_host_reports_divergence(env):
    torch, P, h = env
    X = W.gen_c2(m=256, n=384, seed=2)
    Xh = torch.from_numpy(X).pin_memory()
    Yh = torch.empty_like(Xh).pin_memory()
    with pytest.raises(P.CpaSvtError) as e:
        h.apply_host(Xh, Yh, {"kind": "soft", "tau": 0.1, "tau_relative": True}, 20, lambda_max=0.2 * _lam_true(X))
    assert e.value.status == E_DIVERGED
    h.apply_host(Xh, Yh, {"kind": "soft", "tau": 0.1, "tau_relative": True}, 20, T=100)


def test_nonfinite_input_is_flagged(env):
    torch, P, h = env
    X = W.gen_c2(m=200, n=300, seed=3)
    X[5, 7] = np.nan
    with pytest.raises(P.CpaSvtError) as e:
        h.apply(torch.from_numpy(X).cuda(), {"kind": "soft", "tau": 0.1}, 10, lambda_max=1e4, info=True)
    assert e.value.status == E_DIVERGED


def test_csr_divergence(env):
    torch, P, h = env
    rp, col, val = W.gen_c4(m=300, n=3000, nnz=6000, seed=1)
    import scipy.sparse as sp
    lam_true = float(np.linalg.norm(sp.csr_matrix((val, col, rp), shape=(300, 3000)).toarray(), 2)) ** 2
    args = (torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda(), 300, 3000,
            {"kind": "hard", "tau": 0.5, "tau_relative": True}, 20)
    with pytest.raises(P.CpaSvtError) as e:
        h.apply_csr(*args, lambda_max=0.25 * lam_true, info=True)
    assert e.value.status == E_DIVERGED
    h.apply_csr(*args, T=300, info=True)
