"""Parity of the fp32 dense path on tcgen05 (TF32 with round-to-nearest operands,
and 3xTF32) with the fp64 oracle on the fp32-rounded inputs (reading R15).

Bar (north_star): relative Frobenius error <= 1e-4 on the fp32/TF32 path.  The
3xTF32 mode (the fp32 default, CPA_SVT_MATH_3XTF32) meets it with ~50x margin
(measured 1-3e-6) and is the fp32 path the north-star numbers are claimed on.
Single-pass TF32 (CPA_SVT_MATH_TF32, declared in include/cpa_svt.h as a
reduced-accuracy mode) lands at 0.5-1.5e-4 on the small shapes below: there it is
gated at TF32_REDUCED = 3e-4 and NOT claimed; the c5 full-size single-pass run
(the only single-pass number reported) is gated at the 1e-4 bar.
"""

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu
TOL32 = 1e-4
TF32_REDUCED = 3e-4   # single-pass TF32 on small shapes: reported, not claimed (see above)


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_07112_b200 as P
    h = P.Handle(0)
    yield torch, P, h
    h.close()


def _run(env, X, kern, K, math, T=30, **kw):
    torch, P, h = env
    Xd = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).cuda()
    Y, info = h.apply(Xd, kern, K, T=T, math=math, info=True, **kw)
    torch.cuda.synchronize()
    return Y.cpu().numpy().astype(np.float64), info


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("shape", [(128, 256), (200, 333), (333, 200), (64, 48), (1, 9), (257, 1030)])
def test_tf32_raw_gemm(env, math, shape):
    # coefficients (lam, lam/2) make Y = G X (left) / X G (right): one GEMM through the whole path
    X = W.random_dense(*shape, seed=shape[0] + shape[1]).astype(np.float32).astype(np.float64)
    lam = 2.0 * float(np.linalg.norm(X, 2)) ** 2
    Y, _ = _run(env, X, None, 4, math, lambda_max=lam, coeffs=[lam, lam / 2, 0.0, 0.0])
    want = X @ X.T @ X
    assert O.rel_fro(Y, want) <= (3e-5 if math == "3xtf32" else 2e-3)


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("shape,K", [((512, 2048), 40), ((300, 700), 20), ((700, 300), 12), ((64, 64), 5)])
def test_tf32_parity(env, math, shape, K):
    X = W.gen_c2(m=shape[0], n=shape[1], seed=5).astype(np.float32).astype(np.float64)
    kern = {"kind": "soft", "tau": 0.1, "tau_relative": True}
    Y, info = _run(env, X, kern, K, math, T=300)
    Yo, io = O.cpa_shrink(X, O.Kernel(**kern), K, T=300, return_info=True)
    # lambda_hat of an fp32 Gram: unconverged power iterations move by ~T * eps_G
    assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-4 * io["lambda_hat"]
    assert O.rel_fro(Y, Yo) <= (TOL32 if math == "3xtf32" else TF32_REDUCED), O.rel_fro(Y, Yo)


def test_tf32_config5_proxy(env):
    # configs[4] recipe (rank-50 + 0.01 noise, soft 0.1 sigma_max_hat, K = 40, T = 300) at 1024 x 4096
    cfg = W.CONFIGS["c5"]
    X = W.gen_c5(m=1024, n=4096).astype(np.float32).astype(np.float64)
    Yo = O.cpa_shrink(X, O.Kernel(**cfg["kernel"]), cfg["K"], T=cfg["T"])
    for math in ("tf32", "3xtf32"):
        Y, _ = _run(env, X, cfg["kernel"], cfg["K"], math, T=cfg["T"])
        assert O.rel_fro(Y, Yo) <= (TOL32 if math == "3xtf32" else TF32_REDUCED), (math, O.rel_fro(Y, Yo))


def test_tf32_gemm_engine(env):
    """The tcgen05 engine alone (unit hook): both operand majors, ragged M/N/K."""
    torch, P, h = env
    g = torch.Generator(device="cuda").manual_seed(1)
    r4 = lambda v: (v + 3) // 4 * 4  # TMA needs 16-byte row strides: pad ld, keep the logical shape ragged
    for (M, N, K) in [(128, 128, 32), (129, 130, 131), (300, 520, 1000), (1, 4, 4), (7, 9, 5)]:
        A = torch.randn(M, r4(K), device="cuda", generator=g)[:, :K]
        for b_mn in (True, False):
            B = (torch.randn(K, r4(N), device="cuda", generator=g)[:, :N] if b_mn
                 else torch.randn(N, r4(K), device="cuda", generator=g)[:, :K])
            ref = A.double() @ (B.double() if b_mn else B.double().T)
            for terms, tol in ((3, 2e-5), (1, 3e-3)):
                C = h.debug_gemm_tf32(A, B, b_mn, terms).double()
                assert float((C - ref).norm() / ref.norm()) <= tol, (M, N, K, b_mn, terms)


@pytest.mark.parametrize("shape,K", [((200, 700), 20), ((700, 200), 12), ((256, 256), 9), ((1000, 1300), 7),
                                     ((129, 400), 4), ((300, 300), 3)])
def test_tf32_both_forms(env, shape, K):
    """3xTF32 in the Alg. 1 s x s form and in the apply-to-X form, against the oracle."""
    torch, P, _ = env
    X = W.gen_c2(m=shape[0], n=shape[1], seed=2).astype(np.float32).astype(np.float64)
    kern = {"kind": "soft", "tau": 0.1, "tau_relative": True}
    ref = O.cpa_shrink(X, O.Kernel(**kern), K, T=100)
    for form in ("poly", "apply"):
        h2 = P.Handle(0)
        h2.set_form(form)
        Y = h2.apply(torch.from_numpy(X.astype(np.float32)).cuda(), kern, K, T=100, math="3xtf32")
        h2.close()
        assert O.rel_fro(Y.cpu().numpy().astype(np.float64), ref) <= TOL32, form


def test_config5_full_size_sampled_tf32(env):
    """configs[4] fp32 variant at full size (16384 x 65536): 3xTF32 and TF32 on 10 sampled
    columns (seed-fixed, plus first and last) against the oracle's vector form on the
    fp64-promoted fp32 input, at the oracle's own Lambda (power iteration on the numpy
    Gram); lambda_hat from the fp32 Gram agrees to ~1e-6."""
    import math as m_
    torch, P, h = env
    cfg = W.CONFIGS["c5"]
    X32 = W.gen_c5(dtype=np.float32)
    Xd = torch.from_numpy(X32).cuda()
    m, n = X32.shape
    rng = np.random.default_rng(0)
    cols = sorted(set([0, n - 1] + list(rng.choice(n, 8, replace=False))))
    got = {}
    for math in ("3xtf32", "tf32"):
        Yd, info = h.apply(Xd, cfg["kernel"], cfg["K"], T=cfg["T"], math=math, info=True)
        assert info["form"] == 2
        got[math] = (Yd[:, torch.tensor(cols, device=Yd.device)].cpu().numpy().astype(np.float64), info)
        del Yd
    del Xd
    torch.cuda.empty_cache()
    X = X32.astype(np.float64)
    G = O.gram(X.T)
    lam_hat = O.power_iteration(lambda v: G @ v, m, cfg["T"])[0]
    lam = 1.01 * lam_hat
    c = O.kernel_coefficients(O.Kernel(**cfg["kernel"]), cfg["K"], lam, m_.sqrt(lam_hat))
    Yo = O.cpa_apply_vectors(lambda V: G @ V, X[:, cols], c, lam)
    for math, tol in (("3xtf32", TOL32), ("tf32", TOL32)):
        Ys, info = got[math]
        print(math, "lambda rel err", info["lambda_hat"] / lam_hat - 1, "Y rel err", O.rel_fro(Ys, Yo))
    for math, tol in (("3xtf32", TOL32), ("tf32", TOL32)):
        Ys, info = got[math]
        assert abs(info["lambda_hat"] - lam_hat) <= 1e-5 * lam_hat, math
        assert O.rel_fro(Ys, Yo) <= tol, (math, O.rel_fro(Ys, Yo))
