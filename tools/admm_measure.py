"""NEXT-3 measurement: the paper's synthetic recovery experiment on one
B200 -- D 1000 x 1000 of rank n in {10, 100, 200, 500}, x% of entries zeroed at random
(x in {1, 10, 20}), recovered by cpa_svt_admm_recover (CPA shrinkage as the nuclear prox,
1/rho = 1, eta = 0.01, K = 20, T = 30, tol 1e-4: DESIGN.md reading R23).  Reports iterations,
time, average time per shrink and the recovery error ||L - D||_F / ||D||_F next to the
corrupted input's error."""
import json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

h = P.Handle(0)
for rank in (10, 100, 200, 500):
    D = W.synthetic_D(1000, rank)
    for frac in (0.01, 0.10, 0.20):
        rng = np.random.default_rng(rank * 100 + int(frac * 100))
        mask = (rng.random(D.shape) >= frac).astype(np.uint8)
        Dobs = D * mask
        Dd, Md = torch.from_numpy(Dobs).cuda(), torch.from_numpy(mask).cuda()
        h.admm_recover(Dd, Md, 20, 1.0, 0.01, T=30, tol=1e-4, max_iter=3)   # warm-up
        torch.cuda.synchronize()
        L, info = h.admm_recover(Dd, Md, 20, 1.0, 0.01, T=30, tol=1e-4, max_iter=1000)
        Lh = L.cpu().numpy()
        r = {"N": 1000, "rank": rank, "corrupted": frac, "iters": info["iters"], "last_rel": info["last_rel"],
             "ms_total": info["ms_total"], "ms_per_shrink": info["ms_shrink"] / max(info["iters"], 1),
             "err_recovered": float(np.linalg.norm(Lh - D) / np.linalg.norm(D)),
             "err_corrupted": float(np.linalg.norm(Dobs - D) / np.linalg.norm(D))}
        print(json.dumps(r), flush=True)
