"""NEXT-2 measurement on the paper's own inpainting shape (context, not a BASELINE config):
2560 x 1920 fp64 stand-in (workloads.gen_pinpaint), soft threshold 1/rho = 6,
K = 20: plain CPA (T = I), CPA with the one-level Haar DWT (high band of Phi zeroed,
PAPER.md:628-630), and the exact EVD-based shrinkage, on one B200.  The paper's CPU times
(Table I): 2.00 s (alpha = 20, DWT) and 2.48 s (EVD)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402
import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from exact_baseline import exact_evd, timed  # noqa: E402

X = torch.from_numpy(W.gen_pinpaint()).cuda()
kern = {"kind": "soft", "tau": 6.0, "tau_relative": False}
K, T = 20, 300
out = {"shape": list(X.shape), "K": K, "T": T, "tau": 6.0}
for tr in ("none", "haar1"):
    h = P.Handle(0)
    h.set_transform(tr)
    Y = torch.empty_like(X)
    ms, _ = timed(lambda: h.apply(X, kern, K, T=T, Y=Y), 5)
    out[f"ms_cpa_{tr}"] = ms
    out[f"Y_{tr}"] = Y.clone()
    h.close()
ms_e, Ye = timed(lambda: exact_evd(X, 6.0), 3)
out["ms_evd_exact"] = ms_e
for tr in ("none", "haar1"):
    Y = out.pop(f"Y_{tr}")
    out[f"rel_fro_vs_exact_{tr}"] = float(torch.linalg.norm(Y - Ye) / torch.linalg.norm(Ye))
out["paper_cpu_s"] = {"cpa_alpha20_dwt": 2.00, "evd": 2.48, "source": "PAPER.md:750 (Table I), Xeon E5-2667, MATLAB"}
print(json.dumps(out))
