"""Per-step times of the sparse (c4) SpMM pair on the c4 recipe (BASELINE configs[3] shape) with
a given Lambda (no power iteration) and a small K: python tools/sparse_step.py [K] [reps].
Prints ms per step of Z = W X^T (sparse_z) and W_k = (4/L) Z X - ... (sparse_w)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1705_07112_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
m, n = 20000, 200000
rp, col, val = W.gen_c4()
rp, col, val = (torch.from_numpy(a).cuda() for a in (rp, col, val))
h = P.Handle(0)
kern = {"kind": "hard", "tau": 0.5, "tau_relative": True}
Y = torch.empty((m, n), dtype=torch.float64, device="cuda")
lam = 50.0
h.apply_csr(rp, col, val, m, n, kern, K, lambda_max=lam, Y=Y)
torch.cuda.synchronize()
h.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    h.apply_csr(rp, col, val, m, n, kern, K, lambda_max=lam, Y=Y)
e1.record()
torch.cuda.synchronize()
prof = h.profile_read()
steps = (K - 1) * reps
out = {"K": K, "ms_per_call": e0.elapsed_time(e1) / reps,
       "sparse_z_ms_per_step": prof["sparse_z"][0] / steps, "sparse_w_ms_per_step": prof["sparse_w"][0] / steps,
       "gram_ms": prof["gram"][0] / reps, "checksum": float(Y[::997, ::991].abs().sum())}
print(json.dumps(out))
