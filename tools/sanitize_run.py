"""One small call through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): `compute-sanitizer --tool memcheck python tools/sanitize_run.py`.
Shapes are reduced (several tiles and a ragged tail each) so the instrumented run finishes in
minutes; each call is also checked against the oracle so a silent corruption shows up."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

only = set(sys.argv[1:])
h = P.Handle(0)
soft = {"kind": "soft", "tau": 0.1, "tau_relative": True}


def check(name, Y, Yo, tol):
    err = O.rel_fro(np.asarray(Y, dtype=np.float64), Yo)
    print(f"{name}: rel err {err:.2e}", flush=True)
    assert err <= tol, name


def run(name):
    return not only or name in only


def with_env(var, val, fn):
    os.environ[var] = val
    try:
        return fn()
    finally:
        del os.environ[var]


if run("sym"):   # k_cheb_sym_tma (even s), k_dmma_gemm_tma (Gram, squarings, line 12), k_power_warp, k_sym_init
    X = W.gen_c2(m=256, n=328, seed=1)
    Yo = O.cpa_shrink(X, O.Kernel(**soft), 8, T=40)
    for split in ("1", "2", "4"):
        Y = with_env("CPA_SVT_FLOW_SPLIT", split, lambda: h.apply(torch.from_numpy(X).cuda(), soft, 8, T=40).cpu())
        check(f"sym split {split}", Y, Yo, 1e-10)
if run("sym_odd"):   # k_cheb_sym (cp.async), k_dmma_gemm (cp.async)
    X = W.gen_c2(m=193, n=250, seed=2)
    check("sym odd s", h.apply(torch.from_numpy(X).cuda(), soft, 7, T=40).cpu(),
          O.cpa_shrink(X, O.Kernel(**soft), 7, T=40), 1e-10)
if run("flow"):   # k_cheb_flow (apply-to-X dataflow)
    X = W.gen_c2(m=130, n=300, seed=3)
    h.set_form("apply")
    check("apply form", h.apply(torch.from_numpy(X).cuda(), soft, 6, T=40).cpu(),
          O.cpa_shrink(X, O.Kernel(**soft), 6, T=40), 1e-10)
    h.set_form("auto")
if run("power"):   # k_power_dense (rows in shared memory), k_power_stream (G streamed)
    X = W.gen_c2(m=300, n=400, seed=4)
    Yo = O.cpa_shrink(X, O.Kernel(**soft), 5, T=60)
    check("power smem", with_env("CPA_SVT_POWER_SMEM", "1",
                                 lambda: h.apply(torch.from_numpy(X).cuda(), soft, 5, T=60).cpu()), Yo, 1e-10)
    X = W.gen_c2(m=1100, n=1200, seed=5)
    check("power stream", h.apply(torch.from_numpy(X).cuda(), soft, 4, T=20).cpu(),
          O.cpa_shrink(X, O.Kernel(**soft), 4, T=20), 1e-10)
if run("small"):   # k_small_f64
    X = W.gen_c1()
    check("small", h.apply(torch.from_numpy(X).cuda(), {"kind": "soft", "tau": 2.0}, 20, T=30).cpu(),
          O.cpa_shrink(X, O.Kernel("soft", tau=2.0), 20, T=30), 1e-10)
if run("tf32"):   # k_tc_gemm (Gram sym, steps sym, line 12), tf32 prep/finish, k_power_dense_f32
    X = W.gen_c2(m=200, n=420, seed=6).astype(np.float32)
    Yo = O.cpa_shrink(X.astype(np.float64), O.Kernel(**soft), 8, T=60)
    for math in ("3xtf32", "tf32"):
        check(f"tcgen05 {math}", h.apply(torch.from_numpy(X).cuda(), soft, 8, T=60, math=math).cpu(), Yo,
              1e-4 if math == "3xtf32" else 3e-4)
    h.set_form("apply")
    check("tcgen05 apply form", h.apply(torch.from_numpy(X).cuda(), soft, 8, T=60).cpu(), Yo, 1e-4)
    h.set_form("auto")
if run("batched"):   # k_batched_tc, k_batched_f32
    Xb = W.gen_c3(batch=300, seed=7)
    cfg = W.CONFIGS["c3"]
    Yo, _ = O.cpa_shrink_batched(Xb.astype(np.float64), O.Kernel(**cfg["kernel"]), cfg["K"], T=cfg["T"])
    for eng in ("tc", "ffma"):
        h.set_batched_engine(eng)
        check(f"batched {eng}", h.apply_batched(torch.from_numpy(Xb).cuda(), cfg["kernel"], cfg["K"],
                                                T=cfg["T"]).cpu(), Yo, 1e-4)
    h.set_batched_engine("auto")
if run("sparse"):   # CSC build, SpMV pair, k_spmm_wxt / k_spmm_zx, k_unblock
    import scipy.sparse as sp
    m, n = 70, 900
    rp, col, val = W.gen_c4(m=m, n=n, nnz=2500, seed=8)
    kern = {"kind": "hard", "tau": 0.5, "tau_relative": True}
    Y = h.apply_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda(),
                    m, n, kern, 6, T=50).cpu()
    Xs = sp.csr_matrix((val, col, rp), shape=(m, n))
    Yo, _ = O.cpa_shrink_sparse_rows(Xs, list(range(m)), O.Kernel(**kern), 6, T=50)
    check("sparse", Y, Yo, 1e-10)
if run("panels"):   # multi-GPU s x s recurrence: panel kernels, unpack (3 virtual ranks)
    from paper_1705_07112_b200 import dist as D
    X = W.gen_c2(m=320, n=500, seed=9)
    hc = D.make_handle(0)
    Y = with_env("CPA_SVT_PANEL_SIM", "3", lambda: D.apply_sharded(hc, torch.from_numpy(X).cuda(), 320, 500, soft,
                                                                    6, T=40).cpu())
    check("panels sim3", Y, O.cpa_shrink(X, O.Kernel(**soft), 6, T=40), 1e-10)
    hc.close()
if run("check"):   # divergence check kernel
    X = W.gen_c2(m=128, n=200, seed=10)
    try:
        h.apply(torch.from_numpy(X).cuda(), soft, 12, lambda_max=0.2 * float(np.linalg.norm(X, 2)) ** 2, info=True)
        raise SystemExit("divergence not detected")
    except P.CpaSvtError as e:
        assert e.status == 3
        print("check: E_DIVERGED ok", flush=True)
h.close()
torch.cuda.synchronize()
print("sanitize_run done", flush=True)
