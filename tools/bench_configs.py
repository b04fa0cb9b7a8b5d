"""Measure every BASELINE config on one B200 (device-resident inputs, CUDA events).

Not the driver's bench line (bench.py is): this records the per-config numbers
kept under profiles/ -- GFLOP/s, ms per SVT, roofline fraction of the dominant
phase, HBM GB/s where that is the bound.  Usage: python tools/bench_configs.py c1 c3 c4 [--reps N]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

PEAKS = json.load(open(os.path.join(ROOT, "profiles", "r01_peaks.json")))
HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def oracle_time(kind, budget_s=10.0, **kw):
    """The CPU oracle timed on this host on a bounded sample of the config (reported, not tuned)."""
    import oracle as O
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"] or [1])
    except Exception:
        cores = os.cpu_count()
    t0 = time.perf_counter()
    units, n = 0, 0
    while time.perf_counter() - t0 < budget_s and n < 20:
        units += kw["fn"]()
        n += 1
    el = time.perf_counter() - t0
    return {"kind": "oracle", "cores": cores, "seconds": el, "sample": kw["sample"], "units_per_s": units / el}


def timed(fn, reps, h):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    h.profile(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    prof = h.profile_read()
    h.profile(False)
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    return ms[len(ms) // 2], {k: (v[0] / reps, v[1] / reps) for k, v in prof.items() if v[1]}


def dense(name, h, reps, m=None, n=None, K=None, dtype="f64", math="native"):
    cfg = dict(W.CONFIGS[name])
    m = m or cfg["m"]
    n = n or cfg["n"]
    K = K or cfg["K"]
    gen = {"c1": lambda: W.gen_c1(), "c2": lambda: W.gen_c2(m=m, n=n), "c5": lambda: W.gen_c5(m=m, n=n)}[name]
    X = torch.from_numpy(gen()).cuda()
    if dtype == "f32":
        X = X.float()
    Y = torch.empty_like(X)
    T = cfg["T"]
    ms, ph = timed(lambda: h.apply(X, cfg["kernel"], K, T=T, Y=Y, math=math), reps, h)
    info = h.apply(X, cfg["kernel"], K, T=T, Y=Y, math=math, info=True)[1]
    form = info["form"]
    s, L = min(m, n), max(m, n)
    # recurrence flops of the form that ran: 1 apply-to-X (K-1) 2 s^2 L; 2 symmetric s x s (K-2) s^2 (s+1)
    # (+ final 2 s^2 L); 3 s x s on full tiles (K-2) 2 s^3 (+ final)
    # 4: the whole SVT in one thread block (s <= 64, L <= 128): full s x s products, the step
    #    phase is the whole kernel
    nprod = info.get("rec_products") or (K - 2)   # (K - 3 when Psi_2 came from the squaring, R29)
    rec = {1: (K - 1) * 2 * s * s * L, 2: nprod * s * s * (s + 1), 3: (K - 2) * 2 * s ** 3,
           4: nprod * 2 * s ** 3}[form]
    if info.get("line12_in_recurrence"):   # line 12 ran inside the step launch (m-chain mode)
        rec += 2 * s * s * L
    F_exec = s * (s + 1) * L + rec + (0 if form == 1 or info.get("line12_in_recurrence") else 2 * s * s * L)
    F_eff = s * (s + 1) * L + (K - 1) * 2 * s * s * L   # bench.py's fixed per-workload count
    step_ms = ph.get("step", (0, 0))[0] + (ph.get("init", (0, 0))[0] if form == 1 else 0)
    r = {"config": name, "shape": [m, n], "K": K, "T": T, "dtype": dtype, "math": math,
         "form": {1: "apply-to-X", 2: "s x s symmetric", 3: "s x s full tiles", 4: "s x s, one thread block"}[form],
         "ms_per_svt": ms,
         "gflops_effective": F_eff / ms / 1e6, "gflops_executed": F_exec / ms / 1e6,
         "phases_ms": {k: v[0] for k, v in ph.items()},
         "recurrence_tflops": rec / step_ms / 1e9 if step_ms else None}
    if dtype == "f64":
        r["recurrence_frac_of_dmma_peak"] = rec / step_ms / 1e9 / PEAKS["fp64_dmma_tflops"] if step_ms else None
    else:
        terms = 3 if math == "3xtf32" else 1
        # tf32 dense peak = measured bf16 burst / 2 (nominal ratio); 3xTF32 issues 3 MMAs per product
        tf32_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] / 2
        r["tensor_tflops_issued"] = terms * rec / step_ms / 1e9 if step_ms else None
        r["tensor_frac_of_tf32_peak"] = terms * rec / step_ms / 1e9 / tf32_peak if step_ms else None
    return r


def batched(h, reps, batch=65536):
    cfg = W.CONFIGS["c3"]
    t0 = time.time()
    Xb = torch.from_numpy(W.gen_c3(batch=batch)).cuda()
    gen_s = time.time() - t0
    Y = torch.empty_like(Xb)
    ms, ph = timed(lambda: h.apply_batched(Xb, cfg["kernel"], cfg["K"], T=cfg["T"], Y=Y), reps, h)
    s = L = 64
    K, T = cfg["K"], cfg["T"]
    per = s * (s + 1) * L + (K - 1) * 2 * s * s * L
    F = per * batch
    byt = 2 * batch * 64 * 64 * 4
    # tcgen05 engine (default): Gram, 2 squarings, K-2 steps, line 12 = K + 1 products of 64^3,
    # each 3 TF32 MMAs (3xTF32); TF32 dense peak = MEASURED_PEAKS bf16 / 2, halved at M = 64
    # (one MMA of M64 N64 K8 per 64 cycles per SM)
    # (K - 3 steps when Psi_2 comes from the first squaring: reading R29, T >= 8, K > 3)
    psi2 = T >= 8 and K > 3 and not os.environ.get("CPA_SVT_NO_PSI2_SQ")
    products = (2 if T >= 8 else 0) + 1 + (K - 3 if psi2 else K - 2) + 1
    tensor_flops = batch * products * 3 * 2 * s * s * L
    tf32_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] / 2
    return {"config": "c3", "batch": batch, "engine": "tcgen05 3xTF32 (M=N=64, A in TMEM)", "ms_per_svt_batch": ms,
            "gflops": F / ms / 1e6, "tensor_tflops_issued": tensor_flops / ms / 1e9,
            "tensor_frac_of_tf32_peak": tensor_flops / ms / 1e9 / tf32_peak,
            "tensor_frac_of_m64_ceiling": tensor_flops / ms / 1e9 / (tf32_peak / 2),
            "fp32_frac": F / ms / 1e9 / PEAKS["fp32_ffma_tflops"], "hbm_gbs": byt / ms / 1e6,
            "hbm_frac": byt / ms / 1e6 / HBM, "gen_s": gen_s}


def sparse(h, reps, m=20000, n=200000, nnz=4_000_000):
    cfg = W.CONFIGS["c4"]
    row_ptr, col, val = W.gen_c4(m=m, n=n, nnz=nnz)
    d = [torch.from_numpy(a).cuda() for a in (row_ptr, col, val)]
    Y = torch.empty((m, n), dtype=torch.float64, device="cuda")
    ms, ph = timed(lambda: h.apply_csr(*d, m, n, cfg["kernel"], cfg["K"], T=cfg["T"], Y=Y), reps, h)
    K = cfg["K"]
    F = (K - 1) * 4 * m * nnz
    byt = (K - 1) * (5 * 8 * m * n + 2 * 8 * m * m)
    zx = ph.get("sparse_w", (0, 0))[0]
    zw = ph.get("sparse_z", (0, 0))[0]
    # L2 roofline of the SpMM pair (DESIGN.md §6 "Sparse roofline"): per step each SpMM gathers
    # m * nnz * 8 B (a 512-byte 64-row segment per nonzero and block) through L2, plus the dense W / Y
    # streams (W_{k-1}, W_{k-2}, W_k every step, Y read and written every third: reading R30) and one
    # read of the CSR / CSC structure per 64-row block; ceiling = the measured 512-byte random-gather
    # rate of tools/probes/l2_gather512.cu on this pool's B200 (19.2-20.1 TB/s)
    nblk = (m + 63) // 64
    l2_step = 2 * m * nnz * 8 + ((3 + 2 / 3) * 8 * m * n + 2 * 8 * m * m) + 2 * nblk * nnz * 12
    L2_CEIL = 19500.0
    pair = (zx + zw) / (K - 1)
    return {"config": "c4", "shape": [m, n, nnz], "ms_per_svt": ms, "gflops": F / ms / 1e6,
            "algorithmic_GB": byt / 1e9, "hbm_gbs_alg": byt / ms / 1e6, "hbm_frac": byt / ms / 1e6 / HBM,
            "phases_ms": {k: v[0] for k, v in ph.items()},
            "spmm_pair_ms_per_step": pair,
            "l2_bytes_per_step_GB": l2_step / 1e9, "l2_gbs": l2_step / pair / 1e6 if pair else None,
            "l2_gather_ceiling_gbs": L2_CEIL, "l2_frac": l2_step / pair / 1e6 / L2_CEIL if pair else None}


def oracle_leg(name, r):
    """Attach the oracle's host timing (bounded sample, extrapolated by algorithmic work)."""
    import oracle as O
    import scipy.sparse as sp
    cfg = W.CONFIGS[name]
    k = O.Kernel(**cfg["kernel"])
    if name in ("c1", "c2"):
        X = W.gen_c1() if name == "c1" else W.gen_c2()
        o = oracle_time("dense", fn=lambda: (O.cpa_shrink(X, k, cfg["K"], T=cfg["T"]), 1)[1],
                        sample=f"full {name} SVTs (numpy fp64, Alg. 1 literal)")
        r["oracle_ms_per_svt"] = 1e3 / o["units_per_s"]
    elif name == "c3":
        Xb = W.gen_c3(batch=256)
        o = oracle_time("batched", fn=lambda: (O.cpa_shrink_batched(Xb[:64], k, cfg["K"], T=cfg["T"]), 64)[1],
                        sample="64-matrix slices of the c3 recipe, extrapolated to 65536 matrices")
        r["oracle_ms_per_svt_batch"] = 65536 * 1e3 / o["units_per_s"]
    elif name == "c4":
        m, n, nnz = 20000, 200000, 4_000_000
        rp, col, val = W.gen_c4()
        Xs = sp.csr_matrix((val, col, rp), shape=(m, n))
        t0 = time.perf_counter()
        lam = 1.01 * O.sparse_power_iteration(Xs, 10)[0]
        t_pow = (time.perf_counter() - t0) / 10 * cfg["T"]
        rows = list(range(16))
        o = oracle_time("sparse", fn=lambda: (O.cpa_shrink_sparse_rows(Xs, rows, k, cfg["K"], lam=lam), 16)[1],
                        sample="16 rows per call (vector form, scipy.sparse), extrapolated to 20000 rows "
                               "+ T=300 power steps timed on 10")
        r["oracle_ms_per_svt"] = (t_pow + m / o["units_per_s"]) * 1e3
    elif name == "c5":
        X = W.gen_c5(m=1024, n=4096)
        o = oracle_time("dense", fn=lambda: (O.cpa_shrink(X, k, cfg["K"], T=cfg["T"]), 1)[1],
                        sample="full SVTs at 1024 x 4096 (c5 recipe), extrapolated to 16384 x 65536 by flops")
        s0, L0, s1, L1 = 1024, 4096, 16384, 65536
        f = lambda s_, L_: s_ * s_ * L_ + (cfg["K"] - 2) * 2 * s_ ** 3 + 2 * s_ * s_ * L_
        r["oracle_ms_per_svt"] = 1e3 / o["units_per_s"] * f(s1, L1) / f(s0, L0)
    else:
        return r
    r["oracle"] = o
    return r


if __name__ == "__main__":
    reps = 3
    args = [a for a in sys.argv[1:] if a != "--oracle"]
    if "--reps" in args:
        i = args.index("--reps")
        reps = int(args[i + 1])
        del args[i:i + 2]
    h = P.Handle(0)
    out = []
    for a in args:
        if a == "c1":
            r = dense("c1", h, reps)
        elif a == "c2":
            r = dense("c2", h, reps)
        elif a.startswith("c5t"):         # fp32 tensor-core variant: c5t:MxN:math
            parts = a.split(":")
            mm, nn = map(int, parts[1].split("x")) if len(parts) > 1 else (16384, 65536)
            r = dense("c5", h, reps, m=mm, n=nn, dtype="f32", math=parts[2] if len(parts) > 2 else "3xtf32")
        elif a.startswith("c5"):          # c5 or c5:KxM scaled, e.g. c5:8192x32768
            if ":" in a:
                mm, nn = map(int, a.split(":")[1].split("x"))
                r = dense("c5", h, reps, m=mm, n=nn)
            else:
                r = dense("c5", h, reps)
        elif a.startswith("c3"):
            r = batched(h, reps, int(a.split(":")[1]) if ":" in a else 65536)
        elif a.startswith("c4"):
            if ":" in a:
                mm, nn, zz = map(int, a.split(":")[1].split("x"))
                r = sparse(h, reps, mm, nn, zz)
            else:
                r = sparse(h, reps)
        else:
            raise SystemExit(f"unknown config {a}")
        if "--oracle" in sys.argv:
            r = oracle_leg(a.split(":")[0].replace("c5t", "c5"), r)
        print(json.dumps(r), flush=True)
        out.append(r)
        torch.cuda.empty_cache()
