"""Parity of the fp64 dense CUDA path (DMMA Gram + fused recurrence) with the oracle.

Bar (north_star): relative Frobenius error <= 1e-10 on the fp64 path.  Inputs are
the seeded workloads; the oracle runs Alg. 1 literally (H_hat formed s x s, then
one product), the GPU runs the apply-to-X recurrence, so agreement checks the
arithmetic, not a shared code path.
"""

import math

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu
TOL64 = 1e-10


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_1705_07112_b200 as P
    h = P.Handle(0)
    yield torch, P, h
    h.close()


def _run(env, X, kernel, K, T=30, **kw):
    torch, P, h = env
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    out = h.apply(Xd, kernel, K, T=T, info=True, **kw)
    Y, info = out
    torch.cuda.synchronize()
    return Y.cpu().numpy(), info


def test_config1_parity_and_exact(env):
    cfg = W.CONFIGS["c1"]
    X = W.gen_c1()
    Y, info = _run(env, X, cfg["kernel"], cfg["K"], T=cfg["T"])
    k = O.Kernel(**cfg["kernel"])
    Yo, io = O.cpa_shrink(X, k, cfg["K"], T=cfg["T"], return_info=True)
    assert info["side"] == 1 and io["side"] == "right"
    assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-13 * io["lambda_hat"]
    assert O.rel_fro(Y, Yo) <= TOL64
    # and the method's own error vs exact Jacobi-SVD shrinkage (P10 at K = 20)
    assert O.rel_fro(Y, O.exact_shrink(X, k, 2.0)) <= 2e-2


def test_config2_parity(env):
    cfg = W.CONFIGS["c2"]
    X = W.gen_c2()
    Y, info = _run(env, X, cfg["kernel"], cfg["K"], T=cfg["T"])
    Yo, io = O.cpa_shrink(X, O.Kernel(**cfg["kernel"]), cfg["K"], T=cfg["T"], return_info=True)
    assert info["side"] == 0
    assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-12 * io["lambda_hat"]
    assert abs(info["tau_used"] - io["tau"]) <= 1e-12 * io["tau"]
    assert O.rel_fro(Y, Yo) <= TOL64


SHAPES = [(1, 1), (1, 7), (7, 1), (7, 33), (33, 7), (64, 64), (100, 257), (257, 100), (130, 130), (65, 200)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("kind,K", [("soft", 2), ("hard", 3), ("wsoft", 5), ("soft", 20)])
def test_odd_shapes(env, shape, kind, K):
    X = W.random_dense(*shape, seed=shape[0] * 1000 + shape[1] + K)
    kern = {"kind": kind, "tau": 0.3, "tau_relative": True, "w_c": 2.0, "w_shift": 0.0, "w_eps": 1e-6}
    Y, info = _run(env, X, kern, K, T=40)
    Yo, io = O.cpa_shrink(X, O.Kernel(**kern), K, T=40, return_info=True)
    assert info["side"] == (0 if shape[0] <= shape[1] else 1)
    assert O.rel_fro(Y, Yo) <= TOL64, (shape, kind, K)


@pytest.mark.parametrize("shape", [(40, 70), (70, 40)])
def test_raw_coefficients(env, shape):
    torch, P, h = env
    X = W.random_dense(*shape, seed=3)
    lam = 2.0 * float(np.linalg.norm(X, 2)) ** 2
    Y, _ = _run(env, X, None, 4, lambda_max=lam, coeffs=[2.0, 0.0, 0.0, 0.0])
    assert O.rel_fro(Y, X) <= 1e-14
    Y, _ = _run(env, X, None, 4, lambda_max=lam, coeffs=[lam, lam / 2, 0.0, 0.0])
    assert O.rel_fro(Y, X @ X.T @ X) <= 1e-13
    for kk in (2, 3, 5):
        c = [0.0] * 6
        c[kk] = 1.0
        Y, _ = _run(env, X, None, 6, lambda_max=lam, coeffs=c)
        assert O.rel_fro(Y, O.cpa_shrink(X, None, 6, lam=lam, coeffs=c)) <= 1e-12


def test_degenerate_zero(env):
    Y, info = _run(env, np.zeros((33, 20)), {"kind": "soft", "tau": 1.0}, 10)
    assert info["degenerate"] == 1 and not Y.any()


def test_deterministic_and_pow2(env):
    X = W.gen_c2(m=300, n=500)
    k1 = {"kind": "soft", "tau": 1.0}
    a, _ = _run(env, X, k1, 12)
    b, _ = _run(env, X, k1, 12)
    assert np.array_equal(a, b)
    c, _ = _run(env, 2 * X, {"kind": "soft", "tau": 2.0}, 12)
    assert np.array_equal(2 * a, c)


def test_hard_zero_tau_identity(env):
    X = W.random_dense(90, 150, seed=11)
    Y, _ = _run(env, X, {"kind": "hard", "tau": 0.0}, 25)
    assert O.rel_fro(Y, X) <= 1e-13


def test_block_diagonal_closed_form(env):
    # P17 at a larger, wide shape: the paper's D repeated 4x
    N, nb, copies = 1024, 16, 4
    D = W.block_diag_D(N, nb, copies)
    p = N // nb
    s1, s2 = math.sqrt(copies) * (N - p / 2), math.sqrt(copies) * (p / 2)
    kern = {"kind": "soft", "tau": 0.3, "tau_relative": True}
    Y, info = _run(env, D, kern, 24, T=30)
    lam, c = info["lambda_max"], O.kernel_coefficients(O.Kernel(**kern), 24, info["lambda_max"],
                                                        info["sigma_max_hat"])
    assert abs(info["lambda_hat"] - s1 ** 2) <= 1e-12 * s1 ** 2
    f1 = s1 * O.series_eval(c, lam, s1 ** 2)
    f2 = s2 * O.series_eval(c, lam, s2 ** 2)
    q = np.ones(N) / math.sqrt(N)
    Pb = np.kron(np.eye(nb), np.ones((p, p)) / p)
    R = np.concatenate([np.eye(N)] * copies, axis=1) / math.sqrt(copies)
    want = (f1 * np.outer(q, q) - f2 * (Pb - np.outer(q, q))) @ R
    assert O.rel_fro(Y, want) <= 1e-12


@pytest.mark.parametrize("shape", [(256, 384), (300, 1000), (1100, 300), (1024, 1024)])
def test_apply_host_matches_device(env, shape):
    """cpa_svt_apply_host: with the host pipeline (X copied in four k-chunks, each starting
    its unit of the split-K Gram; Y copied out in four chunks of line 12) it matches the
    device-resident call to rounding (different split-K order) and the oracle; without it
    (CPA_SVT_HOST_NOPIPE) bitwise."""
    import os
    torch, P, h = env
    X = W.gen_c2(m=shape[0], n=shape[1])
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    Yd, _ = _run(env, X, kern, 15, T=100)
    Xh = torch.from_numpy(X).pin_memory()
    Yh = torch.full_like(Xh, float("nan")).pin_memory()
    h.apply_host(Xh, Yh, kern, 15, T=100)
    assert O.rel_fro(Yh.numpy(), Yd) <= 1e-12
    assert O.rel_fro(Yh.numpy(), O.cpa_shrink(X, O.Kernel(**kern), 15, T=100)) <= TOL64
    os.environ["CPA_SVT_HOST_NOPIPE"] = "1"
    try:
        Yh.fill_(float("nan"))
        h.apply_host(Xh, Yh, kern, 15, T=100)
    finally:
        del os.environ["CPA_SVT_HOST_NOPIPE"]
    assert np.array_equal(Yh.numpy(), Yd)


def test_strided_inputs(env):
    torch, P, h = env
    X = W.random_dense(70, 90, seed=5)
    big = torch.zeros((70, 101), dtype=torch.float64, device="cuda")
    big[:, :90] = torch.from_numpy(X).cuda()
    Xv = big[:, :90]
    Yv = torch.full((70, 97), 7.0, dtype=torch.float64, device="cuda")[:, :90]
    kern = {"kind": "soft", "tau": 0.2, "tau_relative": True}
    h.apply(Xv, kern, 9, T=50, Y=Yv)
    assert O.rel_fro(Yv.cpu().numpy(), O.cpa_shrink(X, O.Kernel(**kern), 9, T=50)) <= TOL64


def test_bad_arguments(env):
    torch, P, h = env
    X = torch.zeros((4, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(P.CpaSvtError) as e:
        h.apply(X, {"kind": "soft", "tau": 1.0}, 1)
    assert e.value.status == 1
    with pytest.raises(P.CpaSvtError) as e:
        h.apply(X, {"kind": "soft", "tau": -1.0}, 5)
    assert e.value.status == 2
    with pytest.raises(P.CpaSvtError) as e:
        h.apply(X, {"kind": "soft", "tau": 1.0}, 5, Y=X)
    assert e.value.status == 1


@pytest.mark.parametrize("shape,K", [((1024, 1024), 30), ((300, 70), 9), ((65, 200), 7), ((129, 1000), 5)])
def test_flow_kernel_matches_per_step(env, shape, K):
    """The persistent dataflow recurrence (split-K when a step has few tiles) and
    the one-launch-per-step path differ only in the order of the k-sums."""
    import os
    torch, P, _ = env
    X = W.gen_c2(m=shape[0], n=shape[1], seed=7)
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    Xd = torch.from_numpy(X).cuda()
    out = {}
    for flow in ("1", "0"):
        os.environ["CPA_SVT_FLOW"] = flow
        try:
            h2 = P.Handle(0)
            out[flow] = h2.apply(Xd, kern, K, T=50).cpu().numpy()
            h2.close()
        finally:
            os.environ.pop("CPA_SVT_FLOW", None)
    assert O.rel_fro(out["1"], out["0"]) <= 1e-13
    ref = O.cpa_shrink(X, O.Kernel(**kern), K, T=50)
    assert O.rel_fro(out["1"], ref) <= TOL64 and O.rel_fro(out["0"], ref) <= TOL64


@pytest.mark.parametrize("shape,K", [((100, 257), 12), ((257, 100), 9), ((64, 48), 20), ((300, 1000), 30),
                                     ((129, 129), 5), ((1, 7), 3)])
def test_both_forms_match_oracle(env, shape, K):
    """Alg. 1 literal s x s form (H_hat formed, then Y = H_hat X) and the apply-to-X
    form agree with the oracle and with each other (NEXT-1)."""
    torch, P, _ = env
    X = W.gen_c2(m=shape[0], n=shape[1], seed=11)
    kern = {"kind": "soft", "tau": 0.1, "tau_relative": True}
    ref = O.cpa_shrink(X, O.Kernel(**kern), K, T=80)
    out = {}
    for form in ("poly", "apply", "poly_full"):
        h2 = P.Handle(0)
        h2.set_form(form)
        out[form] = h2.apply(torch.from_numpy(X).cuda(), kern, K, T=80).cpu().numpy()
        h2.close()
        assert O.rel_fro(out[form], ref) <= TOL64, form
    assert O.rel_fro(out["poly"], out["apply"]) <= 1e-12
    assert O.rel_fro(out["poly"], out["poly_full"]) <= 1e-12


@pytest.mark.parametrize("s,K,split", [(1024, 30, 0), (1024, 30, 1), (1024, 30, 2), (1024, 30, 3), (1024, 30, 4),
                                       (200, 9, 3), (1000, 12, 0), (64, 3, 0), (65, 4, 2), (1537, 6, 0), (130, 20, 4),
                                       (300, 5, 0)])
def test_symmetric_form_splits(env, s, K, split):
    """Symmetric s x s form (lower-triangle tiles, mirrored W_k, column-major dataflow
    over three W buffers, `split` k-splits per tile summed in fixed order) against the
    oracle, deterministic run to run; H_hat exactly symmetric shows up as Y = H_hat X
    for X = I being exactly symmetric."""
    import os
    torch, P, _ = env
    X = W.gen_c2(m=s, n=s + 37, seed=s + K)
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    if split:
        os.environ["CPA_SVT_FLOW_SPLIT"] = str(split)
    try:
        h2 = P.Handle(0)
        h2.set_form("poly")
        Y = h2.apply(torch.from_numpy(X).cuda(), kern, K, T=120).cpu().numpy()
        Y2 = h2.apply(torch.from_numpy(X).cuda(), kern, K, T=120).cpu().numpy()
        Hx = h2.apply(torch.eye(s, dtype=torch.float64, device="cuda"), kern, K, T=60).cpu().numpy()
        h2.close()
    finally:
        os.environ.pop("CPA_SVT_FLOW_SPLIT", None)
    assert O.rel_fro(Y, O.cpa_shrink(X, O.Kernel(**kern), K, T=120)) <= TOL64
    assert np.array_equal(Y, Y2)
    assert np.array_equal(Hx, Hx.T)


def test_config5_full_size_sampled(env):
    """BASELINE configs[4] at full size (16384 x 65536 fp64, rank-50 + 0.01 noise, soft
    tau = 0.1 sigma_max_hat, K = 40, T = 300) in the launch configuration the config
    measurement uses: the GPU's lambda_hat against the oracle's power iteration on the
    numpy Gram, and 10 sampled columns (seed-fixed, plus first and last) against the
    oracle's vector form at the oracle's own Lambda."""
    torch, P, h = env
    cfg = W.CONFIGS["c5"]
    X = W.gen_c5()
    Xd = torch.from_numpy(X).cuda()
    Yd, info = h.apply(Xd, cfg["kernel"], cfg["K"], T=cfg["T"], info=True)
    assert info["form"] == 2
    m, n = X.shape
    rng = np.random.default_rng(0)
    cols = sorted(set([0, n - 1] + list(rng.choice(n, 8, replace=False))))
    Ys = Yd[:, torch.tensor(cols, device=Yd.device)].cpu().numpy()
    del Yd, Xd
    torch.cuda.empty_cache()
    G = O.gram(X.T)                       # X X^T: the left Gram, one library product
    lam_hat = O.power_iteration(lambda v: G @ v, m, cfg["T"])[0]
    assert abs(info["lambda_hat"] - lam_hat) <= 1e-12 * lam_hat
    lam = 1.01 * lam_hat
    c = O.kernel_coefficients(O.Kernel(**cfg["kernel"]), cfg["K"], lam, math.sqrt(lam_hat))
    Yo = O.cpa_apply_vectors(lambda V: G @ V, X[:, cols], c, lam)
    err = O.rel_fro(Ys, Yo)
    print(f"c5 full size: lambda_hat rel diff {abs(info['lambda_hat'] - lam_hat) / lam_hat:.3e}, Y rel err {err:.3e}")
    assert err <= TOL64


@pytest.mark.parametrize("shape,K", [((100, 257), 12), ((258, 130), 9), ((1024, 1100), 30), ((66, 66), 5)])
def test_tma_kernels_against_cp_async_and_oracle(env, shape, K):
    """The TMA-fed kernels (k_cheb_sym_tma, k_dmma_gemm_tma: default for 16-byte aligned
    rows) against the cp.async kernels they replace (CPA_SVT_SYM_NOTMA / CPA_SVT_GEMM_NOTMA)
    on even, ragged s (TMA zero-fills the out-of-range box elements) and against the
    oracle.  The two kernels sum the 16 k of a slab in different orders, so they agree to
    rounding (amplified by the power iteration), not bitwise."""
    import os
    X = W.gen_c2(seed=11, m=shape[0], n=shape[1])
    kern = {"kind": "soft", "tau": 0.1, "tau_relative": True}
    Y_tma, i_tma = _run(env, X, kern, K, T=60)
    os.environ["CPA_SVT_SYM_NOTMA"] = "1"
    os.environ["CPA_SVT_GEMM_NOTMA"] = "1"
    try:
        Y_cpa, i_cpa = _run(env, X, kern, K, T=60)
    finally:
        del os.environ["CPA_SVT_SYM_NOTMA"], os.environ["CPA_SVT_GEMM_NOTMA"]
    assert i_tma["form"] == 2 and i_cpa["form"] == 2
    # (the squared power iteration amplifies the Gram's last-bit differences: 1.7e-13 measured)
    assert abs(i_tma["lambda_hat"] - i_cpa["lambda_hat"]) <= 1e-11 * i_cpa["lambda_hat"]
    assert O.rel_fro(Y_tma, Y_cpa) <= 1e-11
    Yo = O.cpa_shrink(X, O.Kernel(**kern), K, T=60)
    assert O.rel_fro(Y_tma, Yo) <= TOL64


@pytest.mark.parametrize("shape", [(1, 1), (7, 33), (33, 7), (64, 48), (48, 64), (64, 64), (40, 128), (128, 40)])
def test_small_kernel_against_grid_path_and_oracle(env, shape):
    """Small problems (s <= 64, L <= 128) run all of Alg. 1 in one thread block (form 4);
    the grid path (CPA_SVT_NO_SMALL) and the oracle must agree with it."""
    import os
    X = W.random_dense(*shape, seed=3)
    kern = {"kind": "soft", "tau": 0.2, "tau_relative": True}
    Y1, i1 = _run(env, X, kern, 12, T=30)
    os.environ["CPA_SVT_NO_SMALL"] = "1"
    try:
        Y2, i2 = _run(env, X, kern, 12, T=30)
    finally:
        del os.environ["CPA_SVT_NO_SMALL"]
    assert i1["form"] == 4 and i2["form"] != 4
    assert abs(i1["lambda_hat"] - i2["lambda_hat"]) <= 1e-12 * i2["lambda_hat"]
    assert O.rel_fro(Y1, Y2) <= 1e-12
    Yo, io = O.cpa_shrink(X, O.Kernel(**kern), 12, T=30, return_info=True)
    assert abs(i1["lambda_hat"] - io["lambda_hat"]) <= 1e-12 * io["lambda_hat"]
    assert O.rel_fro(Y1, Yo) <= TOL64


@pytest.mark.parametrize("shape,K", [((48, 64), 4), ((48, 64), 5), ((64, 128), 12), ((33, 7), 13), ((5, 9), 30)])
def test_small_kernel_two_chains(env, shape, K):
    """The single-block kernel's two-chain recurrence (R28) with Psi_2 from the first squaring (R29)
    against its one-chain recurrence (CPA_SVT_SMALL_CHAIN=0) and the oracle; K even and odd (the last
    pair single), K = 4 (one pair); 64 x 128 has no room for the extra buffer (one chain both ways)."""
    import os
    X = W.random_dense(*shape, seed=K)
    kern = {"kind": "soft", "tau": 0.2, "tau_relative": True}
    Y1, i1 = _run(env, X, kern, K, T=30)
    os.environ["CPA_SVT_SMALL_CHAIN"] = "0"
    try:
        Y2, i2 = _run(env, X, kern, K, T=30)
    finally:
        del os.environ["CPA_SVT_SMALL_CHAIN"]
    assert i1["form"] == 4 and i2["form"] == 4
    # (the extra buffer fits beside the line-12 operand for L <= 64: 64 x 128 keeps one chain)
    assert i1["rec_products"] == (K - 3 if max(shape) <= 64 else K - 2) and i2["rec_products"] == K - 2
    assert i1["lambda_hat"] == i2["lambda_hat"]
    assert O.rel_fro(Y1, Y2) <= 1e-12
    Yo = O.cpa_shrink(X, O.Kernel(**kern), K, T=30)
    assert O.rel_fro(Y1, Yo) <= TOL64


@pytest.mark.parametrize("shape", [(40, 56), (150, 90), (90, 150)])
def test_max_order(env, shape):
    """K = CPA_SVT_KMAX (512) on the single-block path (40 x 56) and the grid path (150 x 90; 90 x 150:
    the two-chain launch with line 12 inside): the coefficients of the 512-point rule and 510
    recurrence steps against the oracle."""
    X = W.random_dense(*shape, seed=21)
    kern = {"kind": "soft", "tau": 0.25, "tau_relative": True}
    Y, info = _run(env, X, kern, 512, T=60)
    Yo, io = O.cpa_shrink(X, O.Kernel(**kern), 512, T=60, return_info=True)
    assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-12 * io["lambda_hat"]
    assert O.rel_fro(Y, Yo) <= TOL64


@pytest.mark.parametrize("s,L,K,split", [(1024, 1024, 30, 0), (1024, 1100, 12, 1), (1024, 1024, 9, 3), (256, 300, 5, 2),
                                         (130, 300, 7, 0), (64, 200, 3, 0), (4096, 4200, 5, 0), (1538, 1600, 6, 5)])
def test_warp_specialized_recurrence_bitwise(env, s, L, K, split):
    """k_cheb_sym_ws (MMA warps hand the accumulators to epilogue warps through shared memory)
    performs the same sums in the same order as k_cheb_sym_tma: bitwise-equal outputs, and the
    oracle bar."""
    import os
    torch, P, _ = env
    X = W.gen_c2(m=s, n=L, seed=s + K)
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    Xd = torch.from_numpy(X).cuda()
    out = {}
    if split:
        os.environ["CPA_SVT_FLOW_SPLIT"] = str(split)
    os.environ["CPA_SVT_SYM_CHAIN"] = "0"   # (the one-chain kernel is the bitwise reference)
    try:
        for ws in ("0", "1"):
            os.environ["CPA_SVT_SYM_WS"] = ws
            h2 = P.Handle(0)
            out[ws] = h2.apply(Xd, kern, K, T=100).cpu().numpy()
            h2.close()
    finally:
        os.environ.pop("CPA_SVT_SYM_WS", None)
        os.environ.pop("CPA_SVT_FLOW_SPLIT", None)
        os.environ.pop("CPA_SVT_SYM_CHAIN", None)
    assert np.array_equal(out["0"], out["1"])
    if s <= 1100:
        assert O.rel_fro(out["1"], O.cpa_shrink(X, O.Kernel(**kern), K, T=100)) <= TOL64


@pytest.mark.parametrize("s,L,K,split", [(1024, 1024, 30, 0), (1024, 1100, 12, 1), (1024, 1024, 9, 3), (256, 300, 5, 2),
                                         (130, 300, 7, 0), (64, 200, 3, 0), (4096, 4200, 5, 0), (1538, 1600, 6, 5)])
def test_eight_warp_recurrence_bitwise(env, s, L, K, split):
    """k_cheb_sym_tma with eight 32 x 16 warp tiles per CTA (CPA_SVT_SYM_NW=8) against the four
    32 x 32 warp tiles: every output element sees the same DMMA k-order and the same split-K sums,
    so the outputs are bitwise equal; and the oracle bar."""
    import os
    torch, P, _ = env
    X = W.gen_c2(m=s, n=L, seed=s + K + 1)
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    Xd = torch.from_numpy(X).cuda()
    out = {}
    if split:
        os.environ["CPA_SVT_FLOW_SPLIT"] = str(split)
    os.environ["CPA_SVT_SYM_CHAIN"] = "0"   # (the one-chain kernel is the bitwise reference)
    try:
        for nw in ("4", "8"):
            os.environ["CPA_SVT_SYM_NW"] = nw
            h2 = P.Handle(0)
            out[nw] = h2.apply(Xd, kern, K, T=100).cpu().numpy()
            h2.close()
    finally:
        os.environ.pop("CPA_SVT_SYM_NW", None)
        os.environ.pop("CPA_SVT_FLOW_SPLIT", None)
        os.environ.pop("CPA_SVT_SYM_CHAIN", None)
    assert np.array_equal(out["4"], out["8"])
    if s <= 1100:
        assert O.rel_fro(out["8"], O.cpa_shrink(X, O.Kernel(**kern), K, T=100)) <= TOL64


@pytest.mark.parametrize("m", [2, 3])
@pytest.mark.parametrize("s,L,K,split", [(1024, 1024, 30, 0), (1024, 1100, 31, 0), (1024, 1024, 6, 2), (1024, 1030, 7, 3),
                                         (256, 300, 8, 1), (256, 260, 9, 2), (130, 300, 10, 0), (130, 140, 11, 5),
                                         (64, 200, 12, 1), (1538, 1600, 13, 4), (2048, 2100, 20, 0), (512, 520, 40, 6),
                                         (200, 210, 14, 2), (320, 330, 15, 3), (1024, 1024, 29, 2)])
def test_two_chain_recurrence(env, m, s, L, K, split):
    """m-chain symmetric recurrence (Psi_k = 2 Psi_m Psi_{k-m} - Psi_{|k-2m|}: the Chebyshev terms of
    each residue k mod m as an independent chain, reading R28) against the oracle's one-chain Alg. 1
     at the fp64 bar, against the one-chain kernel at rounding level, run-to-run
    deterministic, and H_hat exactly symmetric; every residue of K - 1 (which chain's product sums
    H), every k-split count, and K below 2m + 2 (the library falls back to one chain)."""
    import os
    torch, P, _ = env
    X = W.gen_c2(m=s, n=L, seed=s + K + 7)
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    Xd = torch.from_numpy(X).cuda()
    out = {}
    if split:
        os.environ["CPA_SVT_CHAIN_SPLIT"] = str(split)
    try:
        for ch in (str(m), "0"):
            os.environ["CPA_SVT_SYM_CHAIN"] = ch
            h2 = P.Handle(0)
            h2.set_form("poly")
            out[ch] = h2.apply(Xd, kern, K, T=100).cpu().numpy()
            if ch != "0":
                out["again"] = h2.apply(Xd, kern, K, T=100).cpu().numpy()
                out["eye"] = h2.apply(torch.eye(s, dtype=torch.float64, device="cuda"), kern, K, T=60).cpu().numpy()
                os.environ["CPA_SVT_NO_PSI2_SQ"] = "1"   # Psi_2 by the recurrence's own k = 2 product
                out["nosq"] = h2.apply(Xd, kern, K, T=100).cpu().numpy()
                os.environ.pop("CPA_SVT_NO_PSI2_SQ", None)
            h2.close()
    finally:
        os.environ.pop("CPA_SVT_SYM_CHAIN", None)
        os.environ.pop("CPA_SVT_CHAIN_SPLIT", None)
        os.environ.pop("CPA_SVT_NO_PSI2_SQ", None)
    Ym = out[str(m)]
    assert np.array_equal(Ym, out["again"])
    assert np.array_equal(out["eye"], out["eye"].T)
    assert O.rel_fro(Ym, out["0"]) <= 1e-12
    assert O.rel_fro(out["nosq"], out["0"]) <= 1e-12
    if s <= 1100:
        assert O.rel_fro(Ym, O.cpa_shrink(X, O.Kernel(**kern), K, T=100)) <= TOL64


@pytest.mark.parametrize("m,s,L,K,split", [(2, 1024, 1024, 30, 3), (2, 1024, 1100, 31, 2), (3, 1024, 1024, 30, 2),
                                           (2, 256, 300, 9, 1), (3, 320, 330, 15, 3), (2, 130, 140, 11, 5)])
def test_pingpong_recurrence_bitwise(env, m, s, L, K, split):
    """k_cheb_sym_pp (one CTA per SM: two MMA warp groups and an epilogue group, split-K by last
    arrival; opt-in CPA_SVT_SYM_PP=1) sums each tile's partials in the order of k_cheb_sym_tma's
    reducer: bitwise-equal outputs, and the oracle bar."""
    import os
    torch, P, _ = env
    X = W.gen_c2(m=s, n=L, seed=s + K + 3)
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    Xd = torch.from_numpy(X).cuda()
    out = {}
    os.environ["CPA_SVT_SYM_CHAIN"] = str(m)
    os.environ["CPA_SVT_CHAIN_SPLIT"] = str(split)
    try:
        for pp in ("0", "1"):
            os.environ["CPA_SVT_SYM_PP"] = pp
            h2 = P.Handle(0)
            h2.set_form("poly")
            out[pp] = h2.apply(Xd, kern, K, T=100).cpu().numpy()
            h2.close()
    finally:
        for v in ("CPA_SVT_SYM_PP", "CPA_SVT_SYM_CHAIN", "CPA_SVT_CHAIN_SPLIT"):
            os.environ.pop(v, None)
    assert np.array_equal(out["0"], out["1"])
    if s <= 1100:
        assert O.rel_fro(out["1"], O.cpa_shrink(X, O.Kernel(**kern), K, T=100)) <= TOL64


@pytest.mark.parametrize("case", ["left", "left_odd_ld", "right"])
def test_chain_line12_fold_variants(env, case):
    """Line 12 inside the m-chain launch (left side, 16-byte X rows) against the separate line-12
    product (CPA_SVT_NO_L12_FOLD) and the oracle; an odd leading dimension of X and the right side
    fall back to the separate product (info.line12_in_recurrence = 0) and meet the same bar."""
    import os
    torch, P, _ = env
    if case == "right":
        X = W.gen_c2(m=1100, n=1024, seed=5)
        Xd = torch.from_numpy(X).cuda()
    else:
        X = W.gen_c2(m=1024, n=1100, seed=6)
        if case == "left_odd_ld":
            buf = torch.zeros((1024, 1101), dtype=torch.float64, device="cuda")
            buf[:, :1100] = torch.from_numpy(X).cuda()
            Xd = buf[:, :1100]
        else:
            Xd = torch.from_numpy(X).cuda()
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    h2 = P.Handle(0)
    Y, info = h2.apply(Xd, kern, 30, T=300, info=True)
    os.environ["CPA_SVT_NO_L12_FOLD"] = "1"
    try:
        Ysep = h2.apply(Xd, kern, 30, T=300)
    finally:
        os.environ.pop("CPA_SVT_NO_L12_FOLD", None)
    h2.close()
    Y, Ysep = Y.cpu().numpy(), Ysep.cpu().numpy()
    assert info["line12_in_recurrence"] == (1 if case == "left" else 0)
    assert info["rec_products"] == 27   # Psi_2 from the power iteration's squaring (R29)
    assert O.rel_fro(Y, Ysep) <= 1e-12
    assert O.rel_fro(Y, O.cpa_shrink(X, O.Kernel(**kern), 30, T=300)) <= TOL64


def test_binding_rejects_mismatched_buffers(env):
    """The binding checks every buffer the library writes through (ValueError, not assert): an
    apply_host Y of another dtype would take m*n*8 bytes into a 4-byte-per-element host buffer."""
    torch, P, h = env
    kern = {"kind": "soft", "tau": 0.5}
    X = torch.zeros((8, 8), dtype=torch.float64)
    with pytest.raises(ValueError):
        h.apply_host(X, torch.zeros((8, 8), dtype=torch.float32), kern, 5)
    with pytest.raises(ValueError):
        h.apply_host(X, torch.zeros((8, 4), dtype=torch.float64), kern, 5)
    Xd = X.cuda()
    with pytest.raises(ValueError):
        h.apply(Xd, kern, 5, Y=torch.zeros((8, 8), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        h.apply(Xd.cpu(), kern, 5)


def test_enum_arguments(env):
    """Bad enums are E_ARG; a valid but unbuilt combination (fp32 data, MATH_NATIVE) is
    E_UNSUPPORTED -- also for an empty X (header: cpa_svt_status)."""
    import ctypes
    torch, P, h = env
    k = P.kernel_from_dict({"kind": "soft", "tau": 0.5})
    lam = P.Lambda(10, 0, 1.01, 0.0, 0.0)
    X = torch.zeros((8, 8), dtype=torch.float64, device="cuda")
    Y = torch.zeros_like(X)
    call = lambda dt, math, m=8: P.lib.cpa_svt_apply(h._h, dt, math, m, 8, 0, 0, X.data_ptr(), 8, Y.data_ptr(), 8,
                                                     ctypes.byref(k), 5, None, ctypes.byref(lam), None)
    assert call(2, 0) == 1 and call(0, 3) == 1 and call(-1, 0) == 1
    assert call(1, 0) == 7 and call(1, 0, m=0) == 7
    assert call(0, 0) == 0

