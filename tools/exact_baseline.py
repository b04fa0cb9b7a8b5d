"""NEXT-4: the paper's exact EVD-based shrinkage timed on the
same B200 beside CPA, as the paper's Tables I-II compare them on a CPU.

EVD-based (library baseline, cuBLAS + cuSOLVER through torch -- a comparison system, not the
product path): G = X X^T (left) or X^T X, (lambda, V) = eigh(G), Y = V diag(h(lambda)) V^T X
(or X V diag(h) V^T) with the same response h as CPA (soft: h = max(sqrt(l) - tau, 0)/sqrt(l)).
CPA: cpa_svt_apply (this library).  Reports ms of each, the speed-up and the relative Frobenius
difference of CPA against the exact shrinkage (the approximation error of the method itself).
Usage: python tools/exact_baseline.py c2 c5 [--reps N]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402


def exact_evd(X, tau):
    from paper_1705_07112_b200 import exact as E
    return E.exact_shrink(X, {"kind": "soft"}, tau=tau)


def timed(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    out = None
    for a, b in ev:
        a.record()
        out = fn()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    return ms[len(ms) // 2], out


def main():
    reps = 5
    args = sys.argv[1:]
    if "--reps" in args:
        i = args.index("--reps")
        reps = int(args[i + 1])
        del args[i:i + 2]
    h = P.Handle(0)
    for name in args or ["c2"]:
        cfg = W.CONFIGS[name]
        X = torch.from_numpy({"c2": W.gen_c2, "c5": W.gen_c5, "c1": W.gen_c1}[name]()).cuda()
        kern = cfg["kernel"]
        assert kern["kind"] == "soft"
        Y = torch.empty_like(X)
        ms_cpa, _ = timed(lambda: h.apply(X, kern, cfg["K"], T=cfg["T"], Y=Y), reps)
        _, info = h.apply(X, kern, cfg["K"], T=cfg["T"], Y=Y, info=True)
        tau = info["tau_used"]
        ms_evd, Ye = timed(lambda: exact_evd(X, tau), max(1, reps // 2))
        err = float(torch.linalg.norm(Y - Ye) / torch.linalg.norm(Ye))
        r = {"config": name, "shape": list(X.shape), "K": cfg["K"], "T": cfg["T"], "ms_cpa": ms_cpa,
             "ms_evd_exact": ms_evd, "speedup_cpa_vs_evd": ms_evd / ms_cpa, "cpa_vs_exact_rel_fro": err,
             "evd": "torch.linalg.eigh (cuSOLVER syevd) + cuBLAS products, fp64, the tau CPA used"}
        print(json.dumps(r), flush=True)
        del X, Y, Ye
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
