"""NEXT-2 + NEXT-3: the ADMM of the synthetic experiment (settings of
tools/admm_measure.py) with the shrinkage's Gram in the DCT / block-DCT domain, thresholded at
fixed top-k (k1..k3, k4 = keep all) and at the adaptive epsilon(E_t) of
eq. recommendation_epsilon -- the paper's Table IV comparison (there on
images; here on the synthetic D, rank 10, 10% of entries zeroed)."""
import json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

N, rank, frac = 1000, 10, 0.10
D = W.synthetic_D(N, rank)
rng = np.random.default_rng(rank * 100 + int(frac * 100))
mask = (rng.random(D.shape) >= frac).astype(np.uint8)
Dobs = D * mask
Dd, Md = torch.from_numpy(Dobs).cuda(), torch.from_numpy(mask).cuda()
runs = [("none", None, None, False)]
for tr in ("dct", "dct8"):
    for name, k in (("k1", 0.5e-4), ("k2", 1.5e-4), ("k3", 0.5e-3), ("k4", None)):
        runs.append((tr, name, k, False))
    runs.append((tr, "adaptive", None, True))
for tr, name, k, adaptive in runs:
    h = P.Handle(0)
    if tr != "none":
        h.set_transform(tr)
        h.set_epsilon("topk", max(1, int(k * N * N))) if k else h.set_epsilon("none", 0.0)
    h.admm_recover(Dd, Md, 20, 1.0, 0.01, T=30, tol=1e-4, max_iter=3, adaptive_eps=adaptive)   # warm-up
    torch.cuda.synchronize()
    L, info = h.admm_recover(Dd, Md, 20, 1.0, 0.01, T=30, tol=1e-4, max_iter=1000, adaptive_eps=adaptive)
    Lh = L.cpu().numpy()
    h.close()
    print(json.dumps({"transform": tr, "epsilon": name, "iters": info["iters"], "ms_total": info["ms_total"],
                      "ms_per_shrink": info["ms_shrink"] / max(info["iters"], 1),
                      "err_recovered": float(np.linalg.norm(Lh - D) / np.linalg.norm(D)),
                      "err_corrupted": float(np.linalg.norm(Dobs - D) / np.linalg.norm(D))}), flush=True)
