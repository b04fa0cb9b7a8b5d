"""Diagnostic: GPU vs oracle vs closed form on the paper's D at N = 1024 / 2048, K = 24 / 40."""
import math
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import oracle as O
import paper_1705_07112_b200 as P
import workloads as W

h = P.Handle(0)
for N, K, T, tau in [(1024, 24, 30, 0.3), (1024, 40, 30, 0.3), (1024, 40, 300, 0.3), (1024, 40, 30, 0.1),
                     (2048, 40, 30, 0.3)]:
    nb, copies = 16, 4
    p = N // nb
    D = W.block_diag_D(N, nb, copies)
    kern = {"kind": "soft", "tau": tau, "tau_relative": True}
    Yg, info = h.apply(torch.from_numpy(D).cuda(), kern, K, T=T, info=True)
    Yg = Yg.cpu().numpy()
    Yo, io = O.cpa_shrink(D, O.Kernel(**kern), K, T=T, return_info=True)
    s1 = math.sqrt(copies) * (N - p / 2)
    s2 = math.sqrt(copies) * (p / 2)
    lam = io["lambda_max"]
    c = io["coeffs"]
    f1 = s1 * O.series_eval(c, lam, s1 ** 2)
    f2 = s2 * O.series_eval(c, lam, s2 ** 2)
    q = np.ones(N) / math.sqrt(N)
    Pb = np.kron(np.eye(nb), np.ones((p, p)) / p)
    R = np.concatenate([np.eye(N)] * copies, axis=1) / math.sqrt(copies)
    want = (f1 * np.outer(q, q) - f2 * (Pb - np.outer(q, q))) @ R
    print(f"N={N} K={K} T={T} tau={tau}: gpu-oracle {O.rel_fro(Yg, Yo):.3e} oracle-closed {O.rel_fro(Yo, want):.3e} "
          f"gpu-closed {O.rel_fro(Yg, want):.3e} lam gpu/or {info['lambda_hat'] / io['lambda_hat'] - 1:.2e} "
          f"tau gpu/or {info['tau_used'] / io['tau'] - 1:.2e} form {info['form']}", flush=True)
