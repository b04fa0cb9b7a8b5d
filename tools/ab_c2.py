"""A/B timing of the c2 SVT between two builds of the library (device-resident, L2 flushed, CUDA
events, the bench's loop): python tools/ab_c2.py <package-parent-dir> [reps]."""
import os
import sys

sys.path.insert(0, sys.argv[1])
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_07112_b200 as P  # noqa: E402

sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402

reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
X = torch.from_numpy(W.gen_c2()).cuda()
Y = torch.empty_like(X)
h = P.Handle(0)
kern = {"kind": "soft", "tau": 0.05, "tau_relative": True}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    h.apply(X, kern, 30, T=300, Y=Y)
h.profile(True)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
for i in range(reps):
    flush.fill_(i & 255)
    ev[i][0].record()
    h.apply(X, kern, 30, T=300, Y=Y)
    ev[i][1].record()
torch.cuda.synchronize()
prof = h.profile_read()
ms = sorted(a.elapsed_time(b) for a, b in ev)
print(sys.argv[1], "median", round(ms[len(ms) // 2], 4), "mean", round(sum(ms) / len(ms), 4),
      {k: round(v[0] / reps, 4) for k, v in prof.items() if v[1]})
