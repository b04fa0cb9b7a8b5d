"""Empty inputs on every entry point (the header's contract: dims < 0 are argument errors, an
empty X has an empty Y and needs no device work).

Sharded calls: a rank whose block of the long dimension is empty (long extent below the world
size, dist.shard_range) takes part in every collective with a zero partial Gram and writes no
output.  On one GPU the one-rank communicator runs that path with the whole (empty) block: a zero
Gram through the real ncclAllReduce, Lambda = 0, a degenerate (empty) result.
"""

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import paper_1705_07112_b200 as P
    from paper_1705_07112_b200 import dist as D
    h = P.Handle(0)
    hc = D.make_handle(0)
    yield torch, P, D, h, hc
    h.close()
    hc.close()


KERN = {"kind": "soft", "tau": 0.3, "tau_relative": True}


@pytest.mark.parametrize("shape", [(0, 5), (5, 0), (0, 0), (0, 200), (300, 0)])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_dense_empty(env, shape, dtype):
    torch, P, D, h, hc = env
    dt = torch.float64 if dtype == "f64" else torch.float32
    X = torch.empty(shape, dtype=dt, device="cuda")
    n0 = h.launches
    Y, info = h.apply(X, KERN, 12, T=20, info=True)
    assert Y.shape == X.shape and info["degenerate"] == 1
    assert h.launches == n0          # no device work
    # argument errors are still argument errors on an empty X
    with pytest.raises(P.CpaSvtError) as e:
        h.apply(X, KERN, 1)
    assert e.value.status == 1
    with pytest.raises(P.CpaSvtError) as e:
        h.apply(X, {"kind": "soft", "tau": -1.0}, 5)
    assert e.value.status == 2


def test_apply_host_empty(env):
    torch, P, D, h, hc = env
    for shape in [(0, 7), (7, 0)]:
        X = torch.empty(shape, dtype=torch.float64)
        Y = torch.empty_like(X)
        info = h.apply_host(X, Y, KERN, 10, T=20, info=True)
        assert info["degenerate"] == 1


def test_batched_empty(env):
    torch, P, D, h, hc = env
    for shape in [(0, 64, 64), (3, 0, 64), (3, 64, 0), (0, 1, 1)]:
        X = torch.empty(shape, dtype=torch.float32, device="cuda")
        Y = h.apply_batched(X, KERN, 12, T=20)
        assert Y.shape == X.shape


def test_csr_empty_row_range_and_empty_matrix(env):
    torch, P, D, h, hc = env
    row_ptr, col, val = W.gen_c4(m=40, n=300, nnz=600)
    rp = torch.from_numpy(row_ptr).cuda()
    cl = torch.from_numpy(col).cuda()
    vl = torch.from_numpy(val).cuda()
    # rows [7, 7): an empty block of a non-empty X (a rank of a row split with no rows)
    Y = h.apply_csr(rp, cl, vl, 40, 300, {"kind": "hard", "tau": 0.5, "tau_relative": True}, 10, T=50,
                    row_begin=7, row_end=7)
    assert Y.shape == (0, 300)
    # and the rows around it still match the oracle
    import scipy.sparse as sp
    Xs = sp.csr_matrix((val, col, row_ptr), shape=(40, 300))
    Ys = h.apply_csr(rp, cl, vl, 40, 300, {"kind": "hard", "tau": 0.5, "tau_relative": True}, 10, T=50,
                     row_begin=5, row_end=9)
    Yo, _ = O.cpa_shrink_sparse_rows(Xs, [5, 6, 7, 8], O.Kernel("hard", tau=0.5, tau_relative=True), 10, T=50)
    assert O.rel_fro(Ys.cpu().numpy(), Yo) <= 1e-10
    # an empty sparse X (no rows): row_ptr = [0]
    Y0 = h.apply_csr(torch.zeros(1, dtype=torch.int64, device="cuda"), cl[:0], vl[:0], 0, 300, KERN, 10, T=20)
    assert Y0.shape == (0, 300)


@pytest.mark.parametrize("dtype,math", [("f64", "native"), ("f32", "3xtf32")])
@pytest.mark.parametrize("side", ["cols", "rows"])
def test_sharded_empty_block(env, dtype, math, side):
    """One-rank communicator, a block with no columns (cols) / rows (rows) of a global X whose
    long extent is 7: the zero partial Gram goes through the real all-reduce, Lambda = 0, the call
    returns OK with nothing written -- what a rank of a long extent below the world size does
    (its peers' collectives are the same calls)."""
    torch, P, D, h, hc = env
    dt = torch.float64 if dtype == "f64" else torch.float32
    s = 4
    X = torch.empty((s, 0) if side == "cols" else (0, s), dtype=dt, device="cuda")
    Y, info = hc.apply(X, KERN, 9, T=20, math=math, shard=side, long_global=7, info=True)
    assert Y.shape == X.shape and info["degenerate"] == 1 and info["lambda_hat"] == 0.0
    assert info["side"] == (0 if side == "cols" else 1)
    # the same handle right after: a non-empty sharded call is unaffected
    Xf = torch.from_numpy(W.random_dense(*((s, 7) if side == "cols" else (7, s)), seed=3)).to(dt).cuda()
    Yf = hc.apply(Xf, KERN, 9, T=20, math=math, shard=side, long_global=7)
    Yo = O.cpa_shrink(Xf.double().cpu().numpy(), O.Kernel(**KERN), 9, T=20)
    assert O.rel_fro(Yf.double().cpu().numpy(), Yo) <= (1e-10 if dtype == "f64" else 1e-4)


def test_sharded_empty_short_dimension_is_an_error(env):
    torch, P, D, h, hc = env
    X = torch.empty((0, 5), dtype=torch.float64, device="cuda")
    with pytest.raises(P.CpaSvtError) as e:
        hc.apply(X, KERN, 9, T=20, shard="cols", long_global=5)
    assert e.value.status == 1


def test_admm_empty(env):
    torch, P, D, h, hc = env
    for shape in [(0, 6), (6, 0)]:
        Dm = torch.empty(shape, dtype=torch.float64, device="cuda")
        mask = torch.empty(shape, dtype=torch.uint8, device="cuda")
        L, st = h.admm_recover(Dm, mask, K=8, rho=1.0, eta=0.01)
        assert L.shape == shape and st["iters"] == 0

