"""Context run on the paper's background-modeling shape (SURVEY 8d 'p-video', not a BASELINE
config): 86400 x 5000 fp64 stand-in (workloads.gen_pvideo), soft 1/rho = 480,
K = 20 (the paper's alpha = 20), T = 300: plain CPA (T = I), CPA with the one-level Haar DWT
(the paper's variant), and the exact EVD-based shrinkage, on one B200.
Paper (Table II; MATLAB on a Xeon E5-2667): 22.20 s (CPA, alpha = 20),
30.77 s (EVD) per shrink."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402
import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from exact_baseline import exact_evd, timed  # noqa: E402

t0 = time.time()
X = torch.from_numpy(W.gen_pvideo()).cuda()
gen_s = time.time() - t0
kern = {"kind": "soft", "tau": 480.0, "tau_relative": False}
K, T = 20, 300
out = {"shape": list(X.shape), "K": K, "T": T, "tau": 480.0, "gen_s": gen_s}
Ys = {}
for name in ("none", "haar1"):
    h = P.Handle(0)
    h.set_transform(name)
    Y = torch.empty_like(X)
    ms, _ = timed(lambda: h.apply(X, kern, K, T=T, Y=Y), 5)
    out[f"ms_cpa_{name}"] = ms
    Ys[name] = Y.clone()
    h.close()
ms_e, Ye = timed(lambda: exact_evd(X, 480.0), 3)
out["ms_evd_exact"] = ms_e
for name, Y in Ys.items():
    out[f"rel_fro_vs_exact_{name}"] = float(torch.linalg.norm(Y - Ye) / torch.linalg.norm(Ye))
out["paper_cpu_s"] = {"cpa_alpha20_dwt": 22.20, "evd": 30.77, "source": "PAPER.md:883, 887 (Table II), Xeon E5-2667, MATLAB"}
print(json.dumps(out))
