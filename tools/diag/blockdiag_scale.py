"""Diagnostic: the paper's block-diagonal D tiled 4x at growing N, fp64,
every form; relative error against the closed form and the error's projection on the
closed form itself (a pure scale error shows up as |proj| ~ rel)."""
import math
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import oracle as O
import paper_1705_07112_b200 as P

h = P.Handle(0)
kern = {"kind": "soft", "tau": 0.3, "tau_relative": True}
K, T, copies = 40, 30, 4
for N in [int(a) for a in sys.argv[1:]] or [1024, 4096, 8192, 16384]:
    nb = 16
    p = N // nb
    r = torch.arange(N, device="cuda")[:, None] // p
    c = (torch.arange(N * copies, device="cuda")[None, :] % N) // p
    X = (1.0 - 0.5 * (r == c).double())
    s1 = math.sqrt(copies) * (N - p / 2)
    s2 = math.sqrt(copies) * (p / 2)
    lam = 1.01 * s1 * s1
    cf = O.kernel_coefficients(O.Kernel(**kern), K, lam, s1)
    f1 = s1 * O.series_eval(cf, lam, s1 * s1)
    f2 = s2 * O.series_eval(cf, lam, s2 * s2)
    same = (f1 / N - f2 * (1.0 / p - 1.0 / N)) / math.sqrt(copies)
    diff = (f1 / N + f2 / N) / math.sqrt(copies)
    want = torch.where(r == c, torch.tensor(same, dtype=torch.float64, device="cuda"),
                       torch.tensor(diff, dtype=torch.float64, device="cuda"))
    for form in ("poly", "apply", "poly_full"):
        if form == "poly_full" and N > 8192:
            continue
        h.set_form(form)
        Y, info = h.apply(X, kern, K, T=T, info=True)
        d = Y - want
        rel = float(d.norm() / want.norm())
        proj = float((d * want).sum() / (want * want).sum())
        resid = d - proj * want
        print(f"N={N} form={form}: lam_hat rel {info['lambda_hat'] / (s1 * s1) - 1:.2e} rel {rel:.3e} "
              f"scale-part {proj:.3e} rest {float(resid.norm() / want.norm()):.3e} "
              f"rowmean-dev {float(d.mean(dim=1).abs().max()):.3e} f2={f2:.3e}", flush=True)
        del Y, d, resid
    h.set_form("auto")
    del X, want, c
    torch.cuda.empty_cache()
