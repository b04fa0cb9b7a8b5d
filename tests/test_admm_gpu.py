"""NEXT-3 parity: the device ADMM recovery (cpa_svt_admm_recover: DMMA DCT products, CPA
shrinkage prox, fused elementwise updates) against the oracle's ADMM (numpy, oracle CPA
shrinkage) on the paper's synthetic D, iterate for iterate (tol = 0,
fixed iteration count).  Bar: fp64, relative Frobenius <= 1e-9 after 25 iterations."""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_07112_b200 as P
    h = P.Handle(0)
    yield torch, P, h
    h.close()


@pytest.mark.parametrize("N,rank,frac,K", [(96, 4, 0.10, 12), (120, 10, 0.20, 20), (65, 5, 0.01, 8)])
def test_admm_matches_oracle(env, N, rank, frac, K):
    torch, P, h = env
    rng = np.random.default_rng(N + rank)
    D = O.synthetic_D(N - N % rank, rank)
    mask = (rng.random(D.shape) >= frac).astype(np.uint8)
    Dobs = D * mask
    rho, eta, T, iters = 1.0, 0.01, 30, 25
    L, info = h.admm_recover(torch.from_numpy(Dobs).cuda(), torch.from_numpy(mask).cuda(), K, rho, eta, T=T,
                             tol=0.0, max_iter=iters)
    assert info["iters"] == iters
    kern = O.Kernel(kind="soft", tau=1.0 / rho, tau_relative=False)
    Lo = O.admm_recover(Dobs, mask, kern, K, T, rho, eta, max_iter=iters, tol=0.0)
    assert O.rel_fro(L.cpu().numpy(), Lo) <= 1e-9
    # and the recovery is much closer to D than the corrupted observation
    assert O.rel_fro(L.cpu().numpy(), D) < 0.5 * O.rel_fro(Dobs, D)


def test_admm_stops_at_tolerance(env):
    torch, P, h = env
    D = O.synthetic_D(100, 10)
    mask = (np.random.default_rng(1).random(D.shape) >= 0.1).astype(np.uint8)
    L, info = h.admm_recover(torch.from_numpy(D * mask).cuda(), torch.from_numpy(mask).cuda(), 20, 1.0, 0.01,
                             tol=1e-4, max_iter=500)
    assert info["iters"] < 500 and info["last_rel"] < 1e-4


@pytest.mark.parametrize("transform", ["dct", "dct8"])
def test_admm_adaptive_eps_matches_oracle(transform):
    """The recommended epsilon(E_t) schedule: every shrinkage thresholds its
    transform-domain Gram at the top-k of the schedule for the previous iteration's error --
    device against the oracle's adaptive ADMM, iterate for iterate."""
    import torch
    import paper_1705_07112_b200 as P
    rng = np.random.default_rng(7)
    N = 160
    A = rng.random((N, 6)) @ rng.random((6, N)) / 6.0          # low-rank in [0, 1], distinct |Phi_ij|
    mask = (rng.random(A.shape) >= 0.1).astype(np.uint8)
    Dobs = A * mask
    rho, eta, T, K, iters = 1.0, 0.01, 30, 8, 6
    h = P.Handle(0)
    h.set_transform(transform)
    L, info = h.admm_recover(torch.from_numpy(Dobs).cuda(), torch.from_numpy(mask).cuda(), K, rho, eta, T=T,
                             tol=0.0, max_iter=iters, adaptive_eps=True)
    h.close()
    kern = O.Kernel(kind="soft", tau=1.0 / rho, tau_relative=False)
    Lo = O.admm_recover(Dobs, mask, kern, K, T, rho, eta, max_iter=iters, tol=0.0, transform=transform,
                        adaptive_eps=True)
    assert info["iters"] == iters
    assert O.rel_fro(L.cpu().numpy(), Lo) <= 1e-9


def test_admm_adaptive_eps_needs_a_dct_transform(env):
    torch, P, h = env
    D = torch.zeros((32, 32), dtype=torch.float64, device="cuda")
    mask = torch.ones((32, 32), dtype=torch.uint8, device="cuda")
    with pytest.raises(P.CpaSvtError):
        h.admm_recover(D, mask, 8, 1.0, 0.01, max_iter=2, adaptive_eps=True)
