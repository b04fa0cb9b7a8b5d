"""Phase clocks of k_small_f64 (variant build with CPA_SMALL_TRACE: stamps land in Y[0..])."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_07112_b200 as P, workloads as W
X = torch.from_numpy(W.gen_c1()).cuda()
h = P.Handle(0)
cfg = W.CONFIGS["c1"]
for _ in range(3):
    Y = h.apply(X, cfg["kernel"], cfg["K"], T=cfg["T"])
torch.cuda.synchronize()
st = Y.flatten()[:6].cpu().numpy()
names = ["gram", "power", "series", "recurrence", "line12"]
print({n: round(float(st[i + 1] - st[i]) / 1965.0, 2) for i, n in enumerate(names)}, "us")
