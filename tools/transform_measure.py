"""NEXT-2 measurement on the paper's own inpainting shape (context, not a BASELINE config):
2560 x 1920 fp64 stand-in (workloads.gen_pinpaint), soft threshold 1/rho = 6,
K = 20: plain CPA (T = I), CPA with the one-level Haar DWT (high band of Phi zeroed,
PAPER.md:628-630), with the DCT and the 8 x 8 block DCT (keep-all and top-k thresholds), and the
exact EVD-based shrinkage, on one B200.  The paper's CPU times
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
s_ = min(X.shape)
variants = [("none", None, 0), ("haar1", None, 0), ("dct", None, 0)]
# the paper's top-k thresholds k1..k3 = (0.5e-4, 1.5e-4, 0.5e-3) n^2, n = Gram side
for name, frac in (("k1", 0.5e-4), ("k2", 1.5e-4), ("k3", 0.5e-3)):
    variants.append((f"dct_{name}", "topk", max(1, int(frac * s_ * s_))))
# the 8 x 8 block DCT, keep-all and the same top-k thresholds
variants.append(("dct8", None, 0))
for name, frac in (("k1", 0.5e-4), ("k2", 1.5e-4), ("k3", 0.5e-3)):
    variants.append((f"dct8_{name}", "topk", max(1, int(frac * s_ * s_))))
Ys = {}
for name, mode, val in variants:
    h = P.Handle(0)
    h.set_transform(name.split("_")[0])
    if mode:
        h.set_epsilon(mode, val)
    Y = torch.empty_like(X)
    ms, _ = timed(lambda: h.apply(X, kern, K, T=T, Y=Y), 5)
    out[f"ms_cpa_{name}"] = ms
    Ys[name] = Y.clone()
    h.close()
ms_e, Ye = timed(lambda: exact_evd(X, 6.0), 3)
out["ms_evd_exact"] = ms_e
for name, Y in Ys.items():
    out[f"rel_fro_vs_exact_{name}"] = float(torch.linalg.norm(Y - Ye) / torch.linalg.norm(Ye))
out["paper_cpu_s"] = {"cpa_alpha20_dwt": 2.00, "evd": 2.48, "source": "PAPER.md:750 (Table I), Xeon E5-2667, MATLAB"}
print(json.dumps(out))
