"""NEXT-4: the exact EVD-based shrinkage baseline (paper_1705_07112_b200.exact, cuSOLVER) against
the oracle's exact shrinkage (one-sided Jacobi SVD, U g(Sigma) V^T), and CPA's own
approximation error against it falling with the order K (the P10 property)."""

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(64, 48), (48, 64), (120, 120), (300, 90)])
@pytest.mark.parametrize("kind", ["hard", "soft", "wsoft"])
def test_exact_baseline_matches_oracle(shape, kind):
    import torch
    from paper_1705_07112_b200 import exact as E
    X = W.gen_c1() if shape == (64, 48) else W.random_dense(*shape, seed=shape[0] + shape[1])
    kern = {"kind": kind, "tau": 2.0, "w_c": 6.0, "w_shift": 0.0, "w_eps": 1e-6}
    Y = E.exact_shrink(torch.from_numpy(X).cuda(), kern, tau=2.0).cpu().numpy()
    Yo = O.exact_shrink(X, O.Kernel(**kern), 2.0)
    assert O.rel_fro(Y, Yo) <= 1e-10


def test_cpa_error_against_exact_falls_with_K():
    import torch
    import paper_1705_07112_b200 as P
    from paper_1705_07112_b200 import exact as E
    X = W.gen_c2(m=512, n=768)
    Xd = torch.from_numpy(X).cuda()
    h = P.Handle(0)
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    errs = []
    for K in (5, 10, 20, 40):
        Y, info = h.apply(Xd, kern, K, T=300, info=True)
        Ye = E.exact_shrink(Xd, kern, tau=info["tau_used"])
        errs.append(float(torch.linalg.norm(Y - Ye) / torch.linalg.norm(Ye)))
    h.close()
    assert all(a > b for a, b in zip(errs, errs[1:])), errs
