"""Parity of the batched fp32 CUDA path (one CTA per matrix, whole Alg. 1 on chip)
with the fp64 oracle run per matrix on the fp32-rounded inputs (reading R15).

Bar (north_star): relative Frobenius error <= 1e-4 on the fp32 path, whole batch.
"""

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu
TOL32 = 1e-4


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_07112_b200 as P
    h = P.Handle(0)
    yield torch, P, h
    h.close()


def _run(env, Xb, kern, K, T=30, **kw):
    torch, P, h = env
    Xd = torch.from_numpy(np.ascontiguousarray(Xb, dtype=np.float32)).cuda()
    lam = torch.empty(Xb.shape[0], dtype=torch.float32, device="cuda")
    Y = h.apply_batched(Xd, kern, K, T=T, lambda_out=lam, **kw)
    torch.cuda.synchronize()
    return Y.cpu().numpy().astype(np.float64), lam.cpu().numpy()


def test_config3_parity(env):
    cfg = W.CONFIGS["c3"]
    Xb = W.gen_c3(batch=512)
    Y, lam = _run(env, Xb, cfg["kernel"], cfg["K"], T=cfg["T"])
    Yo, lo = O.cpa_shrink_batched(Xb.astype(np.float64), O.Kernel(**cfg["kernel"]), cfg["K"], T=cfg["T"])
    err = O.rel_fro(Y, Yo)
    per = max(O.rel_fro(Y[b], Yo[b]) for b in range(Xb.shape[0]))
    assert err <= TOL32, (err, per)
    assert np.max(np.abs(lam - lo) / lo) < 1e-5


def test_config3_full_batch_sampled(env):
    """BASELINE configs[2] at full size (65536 matrices): 256 sampled matrices (seed-fixed,
    plus first and last) against the oracle, whole-sample Frobenius bar."""
    cfg = W.CONFIGS["c3"]
    Xb = W.gen_c3()
    assert Xb.shape[0] == 65536
    Y, lam = _run(env, Xb, cfg["kernel"], cfg["K"], T=cfg["T"])
    rng = np.random.default_rng(0)
    idx = sorted(set([0, Xb.shape[0] - 1] + list(rng.choice(Xb.shape[0], 254, replace=False))))
    Yo, lo = O.cpa_shrink_batched(Xb[idx].astype(np.float64), O.Kernel(**cfg["kernel"]), cfg["K"], T=cfg["T"])
    assert O.rel_fro(Y[idx], Yo) <= TOL32
    assert np.max(np.abs(lam[idx] - lo) / lo) < 1e-5


@pytest.mark.parametrize("shape", [(64, 48), (48, 64), (7, 33), (33, 7), (1, 1), (64, 64), (17, 17), (64, 1)])
@pytest.mark.parametrize("kind,K", [("soft", 2), ("soft", 20), ("hard", 7), ("wsoft", 12)])
def test_batched_shapes(env, shape, kind, K):
    rng = np.random.default_rng(shape[0] * 100 + shape[1] + K)
    Xb = rng.standard_normal((37,) + shape).astype(np.float32)
    kern = {"kind": kind, "tau": 0.3, "tau_relative": True, "w_c": 2.0, "w_shift": 0.0, "w_eps": 1e-6}
    Y, _ = _run(env, Xb, kern, K, T=30)
    Yo, _ = O.cpa_shrink_batched(Xb.astype(np.float64), O.Kernel(**kern), K, T=30)
    assert O.rel_fro(Y, Yo) <= TOL32


def test_batched_lambda_override_and_zero(env):
    Xb = np.zeros((5, 20, 30), dtype=np.float32)
    Xb[1] = np.random.default_rng(1).standard_normal((20, 30))
    Y, lam = _run(env, Xb, {"kind": "soft", "tau": 0.5}, 10)
    assert not Y[0].any() and not Y[2:].any() and Y[1].any()
    Y2, lam2 = _run(env, Xb[1:2], {"kind": "soft", "tau": 0.5}, 10, lambda_max=500.0)
    Yo = O.cpa_shrink(Xb[1].astype(np.float64), O.Kernel("soft", tau=0.5), 10, lam=500.0)
    assert O.rel_fro(Y2[0], Yo) <= TOL32 and abs(lam2[0] - 500.0) < 1e-3


def test_batched_deterministic(env):
    Xb = W.gen_c3(batch=300, seed=3)
    cfg = W.CONFIGS["c3"]
    a, _ = _run(env, Xb, cfg["kernel"], cfg["K"])
    b, _ = _run(env, Xb, cfg["kernel"], cfg["K"])
    assert np.array_equal(a, b)


@pytest.mark.parametrize("T", [1, 2, 5, 7, 8, 9])
def test_batched_short_power_iterations(env, T):
    """T < 8 runs the power iteration without the squared Gram (qsq = 0); T = 8, 9 the first
    squared cases.  The oracle runs the same T plain products (reading R6)."""
    cfg = W.CONFIGS["c3"]
    Xb = W.gen_c3(batch=64, seed=T)
    Y, lam = _run(env, Xb, cfg["kernel"], cfg["K"], T=T)
    Yo, lo = O.cpa_shrink_batched(Xb.astype(np.float64), O.Kernel(**cfg["kernel"]), cfg["K"], T=T)
    assert O.rel_fro(Y, Yo) <= TOL32
    assert np.max(np.abs(lam - lo) / lo) < 1e-5


def test_batched_256_thread_instance(env):
    """The 8-warp CTA instance (CPA_SVT_BTC_NT=256, 3 CTAs per SM) against the oracle and
    against the default 128-thread instance."""
    import os
    cfg = W.CONFIGS["c3"]
    Xb = W.gen_c3(batch=1000, seed=9)
    Y128, _ = _run(env, Xb, cfg["kernel"], cfg["K"], T=cfg["T"])
    os.environ["CPA_SVT_BTC_NT"] = "256"
    try:
        Y256, lam = _run(env, Xb, cfg["kernel"], cfg["K"], T=cfg["T"])
    finally:
        del os.environ["CPA_SVT_BTC_NT"]
    Yo, lo = O.cpa_shrink_batched(Xb.astype(np.float64), O.Kernel(**cfg["kernel"]), cfg["K"], T=cfg["T"])
    assert O.rel_fro(Y256, Yo) <= TOL32 and O.rel_fro(Y128, Yo) <= TOL32
    assert O.rel_fro(Y256, Y128) <= 1e-5


def test_batched_argument_checks(env):
    torch, P, h = env
    X = torch.zeros((4, 8, 8), dtype=torch.float32, device="cuda")
    kern = {"kind": "soft", "tau": 0.5}
    with pytest.raises(ValueError):
        h.apply_batched(X, kern, 5, Y=torch.zeros((3, 8, 8), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        h.apply_batched(X, kern, 5, Y=torch.zeros((4, 8, 8), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        h.apply_batched(X, kern, 5, lambda_out=torch.zeros(3, dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        h.apply_batched(X, kern, 5, lambda_out=torch.zeros(4, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("K,T", [(20, 30), (4, 30), (5, 8), (12, 7)])
def test_batched_psi2_from_squaring(env, K, T):
    """Psi_2 formed from the power iteration's first squaring (reading R29: c^2 G^2 kept in the H
    buffer, the steps start at k = 3) against the k = 2 product (CPA_SVT_NO_PSI2_SQ=1) at fp32
    rounding level and the oracle at the 1e-4 bar; T < 8 (no squaring) and K = 4 included."""
    import os
    torch, P, h = env
    Xb = W.gen_c3(batch=257, seed=K + T)
    cfg = W.CONFIGS["c3"]
    Y, lam = _run(env, Xb, cfg["kernel"], K, T=T)
    os.environ["CPA_SVT_NO_PSI2_SQ"] = "1"
    try:
        Y0, lam0 = _run(env, Xb, cfg["kernel"], K, T=T)
    finally:
        os.environ.pop("CPA_SVT_NO_PSI2_SQ", None)
    Yo, _ = O.cpa_shrink_batched(Xb.astype(np.float64), O.Kernel(**cfg["kernel"]), K, T=T)
    assert np.array_equal(lam, lam0)
    assert O.rel_fro(Y.astype(np.float64), Y0.astype(np.float64)) <= 1e-5
    assert O.rel_fro(Y.astype(np.float64), Yo) <= 1e-4


def test_batched_size_limits(env):
    """The header's contract: m, n <= 64 and K <= 128, else CPA_SVT_E_UNSUPPORTED (a valid request
    this build does not implement); negative sizes are argument errors."""
    torch, P, h = env
    kern = {"kind": "soft", "tau": 0.5}
    for shape, K in (((2, 65, 8), 5), ((2, 8, 65), 5), ((2, 8, 8), 129)):
        X = torch.zeros(shape, dtype=torch.float32, device="cuda")
        with pytest.raises(P.CpaSvtError) as e:
            h.apply_batched(X, kern, K)
        assert e.value.status == 7, (shape, K)

