"""Diagnostic: TMA-fed symmetric recurrence (default) against the cp.async kernel (CPA_SVT_SYM_NOTMA=1)
on the same input, repeated; a correct kernel differs only by summation order (~1e-15)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

m, n = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4096x16384").split("x"))
X = torch.from_numpy(W.gen_c5(m=m, n=n)).cuda()
h = P.Handle(0)
kern = W.CONFIGS["c5"]["kernel"]
os.environ["CPA_SVT_SYM_NOTMA"] = "1"
Y0 = h.apply(X, kern, 40, T=300)
os.environ.pop("CPA_SVT_SYM_NOTMA")
for r in range(4):
    Y1 = h.apply(X, kern, 40, T=300)
    d = (torch.linalg.norm(Y1 - Y0) / torch.linalg.norm(Y0)).item()
    print(f"{m}x{n} rep {r}: rel diff TMA vs cp.async {d:.3e}", flush=True)
