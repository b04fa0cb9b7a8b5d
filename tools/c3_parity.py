"""c3 parity figures of the batched engines (whole-batch and worst per-matrix relative
Frobenius error against the fp64 oracle, 512 matrices of the c3 recipe)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_07112_b200 as P, workloads as W
from oracle import cpa_oracle as O

cfg = W.CONFIGS["c3"]
Xb = W.gen_c3(batch=512)
Yo, lo = O.cpa_shrink_batched(Xb.astype(np.float64), O.Kernel(**cfg["kernel"]), cfg["K"], T=cfg["T"])
h = P.Handle(0)
Y = h.apply_batched(torch.from_numpy(np.ascontiguousarray(Xb, dtype=np.float32)).cuda(), cfg["kernel"], cfg["K"], T=cfg["T"])
Y = Y.cpu().numpy().astype(np.float64)
print("c3 parity: batch %.3e, worst matrix %.3e (NT=%s)" % (O.rel_fro(Y, Yo), max(O.rel_fro(Y[b], Yo[b]) for b in range(len(Xb))),
                                                       os.environ.get("CPA_SVT_BTC_NT", "128")))
