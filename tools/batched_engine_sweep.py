import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1705_07112_b200 as P, workloads as W, oracle as O
Xb = W.gen_c3(batch=64)
Xd = torch.from_numpy(Xb).cuda()
for kern in [{"kind": "wsoft", "w_c": 22.4, "w_shift": 0.0, "w_eps": 1e-6}, {"kind": "soft", "tau": 0.1, "tau_relative": True}]:
  for K in [2, 3, 4, 5, 8, 20]:
    out = {}
    for eng in ("ffma", "tc"):
        h = P.Handle(0); h.set_batched_engine(eng)
        out[eng] = h.apply_batched(Xd, kern, K, T=30).cpu().numpy().astype(np.float64)
        h.close()
    Yo, _ = O.cpa_shrink_batched(Xb.astype(np.float64), O.Kernel(**kern), K, T=30)
    print(kern["kind"], K, "ffma vs oracle %.2e" % O.rel_fro(out["ffma"], Yo), "tc vs oracle %.2e" % O.rel_fro(out["tc"], Yo))
# lambda fixed
h = P.Handle(0); h.set_batched_engine("tc")
Y = h.apply_batched(Xd, {"kind": "soft", "tau": 0.1, "tau_relative": True}, 5, T=30, lambda_max=2000.0).cpu().numpy().astype(np.float64)
Yo, _ = O.cpa_shrink_batched(Xb.astype(np.float64), O.Kernel(kind="soft", tau=0.1, tau_relative=True), 5, T=30)
