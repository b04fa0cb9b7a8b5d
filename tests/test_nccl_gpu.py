"""The shipped multi-GPU exchange on one B200: a one-rank NCCL communicator.

cpa_svt_init with an ncclUniqueId creates a communicator at any world size, and the
sharded calls (SHARD_COLS for a wide X, SHARD_ROWS for a tall one) then run the real
collectives -- ncclAllReduce of the partial Gram (G = sum_p X_p X_p^T, PAPER.md:278-307,
eq. sing_shrink_from_eig_shrink) and ncclBroadcast of the series parameters -- on the
handle's stream.  At world 1 the all-reduce is the identity, so the result must equal the
unsharded call bitwise (fp64) and match the oracle at the north-star bars.
"""

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu
TOL64, TOL32 = 1e-10, 1e-4


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_07112_b200 as P
    from paper_1705_07112_b200 import dist as D
    h_comm = D.make_handle(0)            # world 1, library-owned NCCL communicator
    assert h_comm.has_comm and h_comm.comm_info() == (1, 0)
    h_plain = P.Handle(0)
    assert h_plain.comm_info() == (0, -1)
    yield torch, P, D, h_comm, h_plain
    h_comm.close()
    h_plain.close()


CASES = [((200, 900), "cols"), ((1024, 4096), "cols"), ((900, 200), "rows"), ((3000, 256), "rows"),
         ((64, 48), "rows"), ((33, 40), "cols")]


@pytest.mark.parametrize("shape,side", CASES)
@pytest.mark.parametrize("form", ["auto", "apply"])
def test_sharded_f64_one_rank(env, shape, side, form):
    torch, P, D, hc, hp = env
    m, n = shape
    X = W.gen_c2(m=m, n=n, seed=11)
    kern = {"kind": "soft", "tau": 0.1, "tau_relative": True}
    Xd = torch.from_numpy(X).cuda()
    assert D.shard_args(m, n, True)["shard"] == side
    hc.set_form(form)
    hp.set_form(form)
    try:
        Ys, info = D.apply_sharded(hc, Xd, m, n, kern, 12, T=100, info=True)
        Yn, _ = hp.apply(Xd, kern, 12, T=100, info=True)
    finally:
        hc.set_form("auto")
        hp.set_form("auto")
    Ys, Yn = Ys.cpu().numpy(), Yn.cpu().numpy()
    if min(m, n) > 64 or max(m, n) > 128:
        assert np.array_equal(Ys, Yn)
    else:   # (unsharded, the single-block kernel runs: same arithmetic, another summation order)
        assert O.rel_fro(Ys, Yn) <= 1e-12
    assert O.rel_fro(Ys, O.cpa_shrink(X, O.Kernel(**kern), 12, T=100)) <= TOL64
    if min(m, n) > 64 or max(m, n) > 128:       # (the single-block kernel has no exchange)
        assert info["ms_allreduce"] > 0.0


@pytest.mark.parametrize("shape", [(300, 1200), (1100, 260)])
@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
def test_sharded_tf32_one_rank(env, shape, math):
    torch, P, D, hc, hp = env
    m, n = shape
    X = W.gen_c2(m=m, n=n, seed=12).astype(np.float32)
    kern = {"kind": "soft", "tau": 0.1, "tau_relative": True}
    Xd = torch.from_numpy(X).cuda()
    Ys, info = D.apply_sharded(hc, Xd, m, n, kern, 15, T=200, math=math, info=True)
    Yn = hp.apply(Xd, kern, 15, T=200, math=math)
    assert info["ms_allreduce"] > 0.0
    Ys, Yn = Ys.cpu().numpy().astype(np.float64), Yn.cpu().numpy().astype(np.float64)
    # the all-reduce of a one-rank communicator copies G; the fp32 split copies are rebuilt from it
    assert O.rel_fro(Ys, Yn) <= 1e-6
    Yo = O.cpa_shrink(X.astype(np.float64), O.Kernel(**kern), 15, T=200)
    assert O.rel_fro(Ys, Yo) <= (TOL32 if math == "3xtf32" else 3e-4)


def test_sharded_block_diagonal_closed_form(env):
    """The paper's synthetic D through the NCCL path, against its closed form."""
    import math
    torch, P, D, hc, hp = env
    N, nb, copies = 512, 8, 4
    Dm = W.block_diag_D(N, nb, copies)
    p = N // nb
    s1, s2 = math.sqrt(copies) * (N - p / 2), math.sqrt(copies) * (p / 2)
    kern = {"kind": "soft", "tau": 0.3, "tau_relative": True}
    Y, info = D.apply_sharded(hc, torch.from_numpy(Dm).cuda(), N, N * copies, kern, 24, T=30, info=True)
    lam = info["lambda_max"]
    c = O.kernel_coefficients(O.Kernel(**kern), 24, lam, info["sigma_max_hat"])
    f1, f2 = s1 * O.series_eval(c, lam, s1 ** 2), s2 * O.series_eval(c, lam, s2 ** 2)
    q = np.ones(N) / math.sqrt(N)
    Pb = np.kron(np.eye(nb), np.ones((p, p)) / p)
    R = np.concatenate([np.eye(N)] * copies, axis=1) / math.sqrt(copies)
    want = (f1 * np.outer(q, q) - f2 * (Pb - np.outer(q, q))) @ R
    assert O.rel_fro(Y.cpu().numpy(), want) <= 1e-12


def test_unsharded_call_on_comm_handle(env):
    """SHARD_NONE on a handle with a communicator runs no collective and equals the plain handle."""
    torch, P, D, hc, hp = env
    X = W.gen_c2(m=256, n=384, seed=3)
    Xd = torch.from_numpy(X).cuda()
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    hc.profile(True)
    Ya = hc.apply(Xd, kern, 10, T=60)
    prof = hc.profile_read()
    hc.profile(False)
    Yb = hp.apply(Xd, kern, 10, T=60)
    assert prof["allreduce"][1] == 0 and prof["exchange"][1] == 0
    assert torch.equal(Ya, Yb)


@pytest.mark.parametrize("s_,L_,K", [(1024, 2048, 30), (768, 800, 12), (257, 600, 9), (130, 3000, 5), (64, 700, 3),
                                     (2048, 2100, 7)])
@pytest.mark.parametrize("mode", ["sim2", "sim3", "sim8", "nccl1"])
def test_panel_sharded_recurrence(env, s_, L_, K, mode):
    """Multi-GPU s x s recurrence: each rank computes a contiguous 1/P of the lower tiles of every
    step, packs them into its all-gather slot, and every rank unpacks all slots into the full
    Psi_k (and H_hat after the last step).  simP: P virtual ranks' panels on this GPU one after
    the other (the slot layout a P-rank all-gather produces); nccl1: the real in-place
    ncclAllGather of a one-rank communicator.  Against the oracle and the persistent one-launch
    recurrence (another k-split, so agreement to rounding).  The power iteration is row-sharded in
    this mode as well (rank p computes rows [s p / P, s (p+1) / P) of every product)."""
    import os
    torch, P, D, hc, hp = env
    X = W.gen_c2(m=s_, n=L_, seed=s_ + K)
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    Xd = torch.from_numpy(X).cuda()
    env_var = ("CPA_SVT_PANEL_SIM", mode[3:]) if mode.startswith("sim") else ("CPA_SVT_PANELS", "1")
    os.environ[env_var[0]] = env_var[1]
    try:
        hc.profile(True)
        Yp, info = D.apply_sharded(hc, Xd, s_, L_, kern, K, T=80, info=True)
        prof = hc.profile_read()
        hc.profile(False)
    finally:
        del os.environ[env_var[0]]
    Yn = hp.apply(Xd, kern, K, T=80)
    assert info["form"] == 2
    nsteps = max(K - 2, 0)
    per = int(mode[3:]) if mode.startswith("sim") else 1
    assert prof["step"][1] == nsteps * per and prof["exchange"][1] == nsteps
    Yp, Yn = Yp.cpu().numpy(), Yn.cpu().numpy()
    assert O.rel_fro(Yp, Yn) <= 1e-12
    Yo, io = O.cpa_shrink(X, O.Kernel(**kern), K, T=80, return_info=True)
    # the power iteration runs row-sharded too (one all-gather of u per product)
    assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-12 * io["lambda_hat"]
    assert prof["power"][1] >= 1
    assert O.rel_fro(Yp, Yo) <= TOL64



@pytest.mark.parametrize("shape,K", [((300, 1200), 15), ((1100, 260), 9), ((520, 600), 3)])
@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("mode", ["sim3", "nccl1"])
def test_panel_sharded_tf32(env, shape, K, math, mode):
    """The tcgen05 s x s recurrence by tile panels (each rank 1/P of the lower-triangle tile list
    of every step, packed slots all-gathered, unpacked into the fp32 lower triangle and the TF32
    hi / lo operand copies) and the row-sharded power iteration on the fp32 Gram."""
    import os
    torch, P, D, hc, hp = env
    m, n = shape
    X = W.gen_c2(m=m, n=n, seed=21).astype(np.float32)
    kern = {"kind": "soft", "tau": 0.1, "tau_relative": True}
    Xd = torch.from_numpy(X).cuda()
    env_var = ("CPA_SVT_PANEL_SIM", mode[3:]) if mode.startswith("sim") else ("CPA_SVT_PANELS", "1")
    os.environ[env_var[0]] = env_var[1]
    try:
        hc.profile(True)
        Yp, info = D.apply_sharded(hc, Xd, m, n, kern, K, T=200, math=math, info=True)
        prof = hc.profile_read()
        hc.profile(False)
    finally:
        del os.environ[env_var[0]]
    Yn = hp.apply(Xd, kern, K, T=200, math=math)
    per = int(mode[3:]) if mode.startswith("sim") else 1
    assert prof["step"][1] == (K - 2) * per and prof["exchange"][1] == K - 2
    Yp, Yn = Yp.cpu().numpy().astype(np.float64), Yn.cpu().numpy().astype(np.float64)
    assert O.rel_fro(Yp, Yn) <= 1e-5
    Yo, io = O.cpa_shrink(X.astype(np.float64), O.Kernel(**kern), K, T=200, return_info=True)
    assert abs(info["lambda_hat"] - io["lambda_hat"]) <= 1e-5 * io["lambda_hat"]
    assert O.rel_fro(Yp, Yo) <= (TOL32 if math == "3xtf32" else 3e-4)
