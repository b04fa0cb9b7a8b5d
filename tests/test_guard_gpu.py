"""Memory-safety checks standing in for compute-sanitizer (closed on this GPU pool: runs under it
have left GPUs needing a reset).

1. tools/sanitize_run.py -- one small call through every kernel family, each checked against the
   oracle -- run in a subprocess on the CHECKED build of the library (build.py variant
   CPA_SVT_CHECKED=1: device bounds checks on every data-dependent index -- CSR / CSC gathers, the
   CSC build's scatter, tile decodes, all-gather slots, split-K slots -- that trap on failure) with
   CPA_SVT_GUARD=1 (every workspace allocation carries a guard band from the end of what the call
   uses, checked after every public call).
2. Caller-buffer canaries: outputs with padded leading dimensions and trailing rows filled with a
   sentinel; only the output region may change.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _checked_lib():
    import importlib.util
    spec = importlib.util.spec_from_file_location("cpa_build", os.path.join(ROOT, "paper_1705_07112_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    lib = os.path.join(ROOT, "paper_1705_07112_b200", "libcpasvt_checked.so")
    return mod.build(defines=("CPA_SVT_CHECKED=1",), lib=lib, tag="_checked")


def test_every_kernel_family_checked_build_with_guard_bands():
    lib = _checked_lib()
    env = dict(os.environ, CPA_SVT_LIB=lib, CPA_SVT_GUARD="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], env=env,
                       capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    print(out[-3000:])
    assert r.returncode == 0, out[-3000:]
    assert "CPA_DCHECK failed" not in out and "guard band" not in out
    assert "sanitize_run done" in out


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_1705_07112_b200 as P
    h = P.Handle(0)
    yield torch, P, h
    h.close()


SENT = -7.77e7


def _canvas(torch, rows, cols, ld_pad, extra_rows, dtype):
    big = torch.full((rows + extra_rows, cols + ld_pad), SENT, dtype=dtype, device="cuda")
    return big, big[:rows, :cols]


@pytest.mark.parametrize("shape,math", [((200, 330), None), ((330, 200), None), ((64, 48), None),
                                        ((300, 500), "3xtf32"), ((500, 300), "tf32")])
def test_dense_output_canary(env, shape, math):
    torch, P, h = env
    m, n = shape
    dt = torch.float64 if math is None else torch.float32
    X = torch.from_numpy(W.gen_c2(m=m, n=n, seed=5)).to(dt).cuda()
    big, Y = _canvas(torch, m, n, 13, 3, dt)
    h.apply(X, {"kind": "soft", "tau": 0.1, "tau_relative": True}, 9, T=50, Y=Y, math=math)
    torch.cuda.synchronize()
    mask = torch.ones_like(big, dtype=torch.bool)
    mask[:m, :n] = False
    assert bool((big[mask] == SENT).all())
    assert bool(torch.isfinite(Y).all())


def test_csr_output_canary(env):
    torch, P, h = env
    m, n = 90, 1000
    rp, col, val = W.gen_c4(m=m, n=n, nnz=3000, seed=2)
    big, Y = _canvas(torch, 40, n, 9, 2, torch.float64)
    d = [torch.from_numpy(a).cuda() for a in (rp, col, val)]
    h.apply_csr(*d, m, n, {"kind": "hard", "tau": 0.5, "tau_relative": True}, 7, T=40, row_begin=30, row_end=70, Y=Y)
    torch.cuda.synchronize()
    mask = torch.ones_like(big, dtype=torch.bool)
    mask[:40, :n] = False
    assert bool((big[mask] == SENT).all())
    import scipy.sparse as sp
    Yo, _ = O.cpa_shrink_sparse_rows(sp.csr_matrix((val, col, rp), shape=(m, n)), list(range(30, 70)),
                                     O.Kernel("hard", tau=0.5, tau_relative=True), 7, T=40)
    assert O.rel_fro(Y.cpu().numpy(), Yo) <= 1e-10


def test_batched_output_canary(env):
    torch, P, h = env
    Xb = torch.from_numpy(W.gen_c3(batch=70, seed=3)).cuda()
    buf = torch.full((72 * 64 * 64,), SENT, dtype=torch.float32, device="cuda")
    Y = buf[64 * 64: 64 * 64 * 71].view(70, 64, 64)
    lam = torch.full((72,), SENT, dtype=torch.float32, device="cuda")
    h.apply_batched(Xb, W.CONFIGS["c3"]["kernel"], 20, T=30, Y=Y, lambda_out=lam[1:71])
    torch.cuda.synchronize()
    assert bool((buf[:64 * 64] == SENT).all()) and bool((buf[64 * 64 * 71:] == SENT).all())
    assert float(lam[0]) == SENT and float(lam[71]) == SENT


@pytest.mark.parametrize("split", ["1", "2", "3", "5"])
def test_dataflow_repeatability_stress(env, split):
    """Races in the spin-wait dataflow kernels (tickets, cross counters, split-K slots, the
    power iteration's LL exchange) would show up as run-to-run differences: 25 runs bitwise equal."""
    torch, P, h = env
    X = torch.from_numpy(W.gen_c2(m=640, n=700, seed=int(split))).cuda()
    kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
    os.environ["CPA_SVT_FLOW_SPLIT"] = split
    try:
        ref = h.apply(X, kern, 12, T=120)
        for _ in range(24):
            assert torch.equal(h.apply(X, kern, 12, T=120), ref)
    finally:
        del os.environ["CPA_SVT_FLOW_SPLIT"]


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_bench_config_repeatability_stress(env, name):
    """The configurations bench.py / smoke() time, exactly as they run there (c2: the two-chain launch
    with line 12 inside it; c1: the single-block two-chain kernel): 40 runs bitwise equal."""
    torch, P, h = env
    cfg = W.CONFIGS[name]
    X = torch.from_numpy(W.gen_c1() if name == "c1" else W.gen_c2()).cuda()
    Y = torch.empty_like(X)
    ref = h.apply(X, cfg["kernel"], cfg["K"], T=cfg["T"]).clone()
    for _ in range(40):
        h.apply(X, cfg["kernel"], cfg["K"], T=cfg["T"], Y=Y)
        assert torch.equal(Y, ref)
